#!/usr/bin/env python
"""Benchmark of the B200 batched-dice path (BASELINE.json metric: bounded rolls/sec and
shuffled elements/sec per GPU and box-wide vs roofline).

Headline workload = BASELINE.json configs[1] ("C2"): 2^25 batches of k=2 bounded rolls
per GPU, bounds iid U[2, 2^16) drawn from seed 7 (2 + roll_single(pcg64(7), 65534),
generated on the device by our own k=1 roll kernel), roll words from
pcg64(array_seed(7, 1)).  One step = one bulk roll_batches over the resident bounds (2^26
rolls).  Inputs (256 MiB bounds) and outputs (256 MiB rolls + 32 MiB words) exceed the
126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config c2|c3|c4|c1]

Under torchrun (N > 1) every rank rolls its own 2^25-batch section of ONE global stream
(jump-ahead by rank * 2^25 words; weak scaling); the only exchange is an all-gather of the
per-rank rejection counts.  Secondary lines for the shuffle configs are
reported under "secondary" (C3 2^20 x 64 u32, C4 65,536 x 4096 u32, C1 one 10,000-element
stream).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NB_C2 = 1 << 25
BYTES_PER_BATCH_C2 = 17  # 8 B bounds in + 8 B rolls out + 1 B words out (8.5 B/roll)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_profile(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as fh:
            return json.load(fh)
    except Exception:
        return None


# 7 partial products (IMAD.WIDE.U32) per C2 roll: 2 per die + a PCG64 step
# (10) per k = 2 batch.  Peak: tools/micro/opcost.cu on B200 (profiles/opcost_r1.json).
INT_PP_PER_ROLL = 7
# smem bytes per element of a shared-memory-staged shuffle (algorithmic): stage in (4 B),
# each step reads and writes z[i] and z[j] (16 B), stage out (4 B); u32 payload.
SMEM_BYTES_PER_ELEM_U32 = 24
# the index-permutation kernel (u16 indices): identity written (2 B), each step reads and
# writes two u16 (8 B), payload staged in (4 B), gather reads index and payload (6 B)
SMEM_BYTES_PER_ELEM_IDX_U32 = 20


def int_roofline(rolls_per_s):
    p = load_profile("opcost_r1.json")
    if not p:
        return None
    peak = p["imad_wide_per_s"] / 1e12
    achieved = rolls_per_s * INT_PP_PER_ROLL / 1e12
    return {"bound": "int", "achieved": achieved, "peak": peak, "unit": "T IMAD.WIDE.U32/s", "frac": achieved / peak,
            "per_roll": INT_PP_PER_ROLL, "peak_source": "measured: profiles/opcost_r1.json (tools/micro/opcost.cu)"}


def smem_roofline(elems_per_s, kernel=""):
    p = load_profile("smem_r1.json")
    if not p:
        return None
    peak = min(p["lds32_gbs"], p["sts32_gbs"])
    per = SMEM_BYTES_PER_ELEM_IDX_U32 if "idx" in kernel else SMEM_BYTES_PER_ELEM_U32
    achieved = elems_per_s * per / 1e9
    return {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "bytes_per_element": per,
            "peak_source": "measured: profiles/smem_r1.json (tools/micro/smem_bw.cu)"}


def random_roofline(steps_per_s, footprint_mb):
    """HBM-resident arrays: every Fisher-Yates step reads z[j] at a random position and writes
    it back.  Peak = the measured random 8-byte read-modify-write rate over a buffer of the same
    footprint (tools/micro/randgather.cu rmw, profiles/randaccess_r1.jsonl).  The kernel can
    exceed it: targets j are uniform on [0, i], so the low positions of each array are hit
    often and stay in L2."""
    try:
        with open(os.path.join(ROOT, "profiles", "randaccess_r1.jsonl")) as fh:
            rows = [json.loads(x) for x in fh if x.strip()]
    except Exception:
        return None
    big = [r for r in rows if r["buffer_mb"] >= footprint_mb]
    if not big:
        return None
    r = min(big, key=lambda r: r["buffer_mb"])
    peak = r["rmw_per_s"] / 1e9
    achieved = steps_per_s / 1e9
    return {"bound": "hbm_random", "achieved": achieved, "peak": peak, "unit": "G random RMW/s",
            "frac": achieved / peak, "per_element": "one random 8-byte read + write of z[j]",
            "peak_source": f"measured: random RMW over {r['buffer_mb']} MB (tools/micro/randgather.cu, "
                           "profiles/randaccess_r1.jsonl)"}


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


_SAMPLER_SRC = r"""
import sys, time, pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), get_r(h)  # warm the query path
print("ready", nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM), flush=True)
while True:
    print(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), int(get_r(h)), flush=True)
    time.sleep(0.0002)
"""


class ClockSampler:
    """SM clock and throttle reasons sampled by NVML (~0.2 ms period) while the timed region
    runs, in a separate process so the samples keep coming while this one holds the GIL or
    waits in a device synchronisation; also records the reasons nvidia-smi would show
    (hw_slowdown, thermal, power cap)."""

    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self.max_sm = None
        self.proc = None

    def __enter__(self):
        import subprocess

        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER_SRC, str(self._nvml_index())],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            head = self.proc.stdout.readline().split()  # blocks until NVML answers
            if head and head[0] == "ready":
                self.max_sm = int(head[1])
                # the loop is running once its first sample is out; later ones fall in the region
                first = self.proc.stdout.readline().split()
                if len(first) != 2:
                    self._kill()
            else:
                self._kill()
        except Exception:
            self._kill()
        return self

    def _nvml_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[self.dev])
            except (ValueError, IndexError):
                pass
        return self.dev

    def _kill(self):
        if self.proc is not None:
            self.proc.kill()
            self.proc.wait()
            self.proc = None

    def __exit__(self, *a):
        if self.proc is None:
            return
        self.proc.kill()
        out, _ = self.proc.communicate()
        self.proc = None
        for line in out.splitlines():
            try:
                c, r = line.split()
                self.samples.append((int(c), int(r)))
            except ValueError:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": [], "samples": 0}
        reasons = sorted({k for _, r in self.samples for k, b in self.BITS.items() if r & b})
        return {"sm_mhz": statistics.median(c for c, _ in self.samples), "sm_max_mhz": self.max_sm,
                "reasons": reasons, "samples": len(self.samples)}


def soak(torch, fn, seconds=0.3):
    """Run the step back to back until the clocks have ramped (part of the warm-up)."""
    if os.environ.get("BENCH_NO_SOAK"):
        return
    t = time.perf_counter()
    while time.perf_counter() - t < seconds:
        for _ in range(8):
            fn()
        torch.cuda.synchronize()


# ------------------------------------------------------------------------------ helpers
def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(torch, value, ws):
    if ws == 1:
        return value
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(torch, ws):
    torch.cuda.synchronize()
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------------------ C2 (rolls)
def setup_c2(torch, B, rank, nb, generator="pcg64"):
    import numpy as np

    from paper_2408_06213_b200 import _native as N

    # bounds: 2 + roll_single(pcg64(7), 65534), this rank's section of the global sequence
    st = N.Pcg64State()
    N.lib().br_pcg64_seed(7, C.byref(st))
    N.lib().br_pcg64_advance(C.byref(st), rank * 2 * nb)
    gen = B.DeviceStream.from_struct(st)
    spans = torch.full((2 * nb,), 65534, dtype=torch.int32, device="cuda")
    r = B.roll_batches(gen, spans, 1)
    bounds = (r.rolls + 2).contiguous()
    del spans, r
    # roll stream: make_source(generator, array_seed(7, 1)) advanced to this rank's first batch
    seed = N.lib().br_array_seed(7, 1)
    if generator == "chacha":
        st = N.ChachaState()
        N.lib().br_chacha_seed(seed, C.byref(st))
    else:
        st = N.Pcg64State()
        (N.lib().br_lehmer_seed if generator == "lehmer" else N.lib().br_pcg64_seed)(seed, C.byref(st))
    N.lib().br_pcg64_advance(C.byref(st), rank * nb)
    stream = B.DeviceStream.from_struct(st)
    rolls = torch.empty(2 * nb, dtype=torch.int32, device="cuda")
    words = torch.empty(nb, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    return bounds, stream, rolls, words


def bench_c2(args, torch, B, ws, rank):
    from paper_2408_06213_b200 import _native as N

    L = N.lib()
    nb = NB_C2
    bounds, stream, rolls, words = setup_c2(torch, B, rank, nb, args.generator)
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    ptrs = [C.c_void_p(x.data_ptr()) for x in (bounds, stream.state, rolls, words)]
    wsp = C.c_void_p(stream.workspace.data_ptr())
    extras = torch.zeros(ws, dtype=torch.int64, device="cuda")

    def step():  # production call: main kernel + PDL-launched fixup (br_roll_batches)
        N.check(L.br_roll_batches_phase(ptrs[0], 2, nb, ptrs[1], ptrs[2], ptrs[3], None, None, wsp, 3, sp), "roll")

    for _ in range(args.warmup):
        step()
    soak(torch, step)
    barrier(torch, ws)
    K = args.steps
    with ClockSampler(torch.cuda.current_device()) as clk:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record()
        for i in range(K):
            step()
        end.record()
        torch.cuda.synchronize()
    total_ms = start.elapsed_time(end)
    # dominant kernel alone: the same K steps issued as two phases with CUDA events around
    # the main kernel (roll_fast_kernel) on the launching stream
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    for i in range(K):
        e0[i].record()
        N.check(L.br_roll_batches_phase(ptrs[0], 2, nb, ptrs[1], ptrs[2], ptrs[3], None, None, wsp, 1, sp), "main")
        e1[i].record()
        N.check(L.br_roll_batches_phase(ptrs[0], 2, nb, ptrs[1], ptrs[2], ptrs[3], None, None, wsp, 2, sp), "fixup")
    torch.cuda.synchronize()
    main_ms = [a.elapsed_time(b) for a, b in zip(e0, e1)]
    barrier(torch, ws)
    total_ms = max_over_ranks(torch, total_ms, ws)
    # cross-rank exchange: per-rank rejection counts (all zero unless a batch was rejected)
    extra = C.c_uint64()
    N.check(L.br_roll_check(wsp, sp, C.byref(extra)), "check")
    if ws > 1:
        import torch.distributed as dist

        mine = torch.tensor([int(extra.value)], dtype=torch.int64, device="cuda")
        gathered = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(ws)]
        dist.all_gather(gathered, mine)
        extras = torch.cat(gathered)
    rolls_total = 2 * nb * K * ws
    value = rolls_total / (total_ms / 1e3)
    t_main = statistics.mean(main_ms) / 1e3
    if args.generator == "chacha":  # ChaCha streams are rolled inside the fixup kernel: time the step
        t_main = total_ms / K / 1e3
    peak, peak_kind = load_peaks()
    achieved = BYTES_PER_BATCH_C2 * nb / t_main / 1e9
    traffic = load_traffic().get("roll_fast_kernel")
    res = {
        "value": value,
        "ms_per_step": total_ms / K,
        "main_ms": statistics.mean(main_ms),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "kernel": "roll_fast_kernel<2>" if args.generator != "chacha" else "roll_fixup_kernel<2>",
                     "algorithmic_bytes_per_launch": BYTES_PER_BATCH_C2 * nb, "peak_source": peak_kind},
        # the north star's denominator for rolls: the integer multiply pipe (HBM binds first)
        "roofline_int": int_roofline(2 * nb / t_main),
        "clocks": clk.summary(),
        "gpu_launches": 2 * K,
        "cross_rank_rejections": [int(x) for x in extras.cpu().tolist()] if ws > 1 else [int(extra.value)],
    }
    # end to end through the public API with host (pinned) buffers
    hb = bounds.cpu().pin_memory()
    hrolls = torch.empty(2 * nb, dtype=torch.int32).pin_memory()
    hwords = torch.empty(nb, dtype=torch.uint8).pin_memory()
    E = max(2, min(K, 10))
    for _ in range(2):  # warm-up (pinned pages, copy streams, allocator)
        B.roll_batches(stream, hb, 2, out=(hrolls, hwords))
    barrier(torch, ws)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(E):
        B.roll_batches(stream, hb, 2, out=(hrolls, hwords), check=False)
    t1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(torch, t0.elapsed_time(t1), ws)
    res["e2e"] = {"value": 2 * nb * E * ws / (e2e_ms / 1e3), "unit": "rolls/s",
                  "h2d_bytes_per_step": 8 * nb, "d2h_bytes_per_step": 8 * nb + nb, "steps": E,
                  "api": "paper_2408_06213_b200.roll_batches(host pinned tensors, 16-chunk pipelined copies)"}
    return res


def cpu_baseline_c2(sample_batches=1 << 24, target_s=10.0):
    """The oracle port of roll_batch on every host thread, about target_s seconds: the first
    2^24 C2 bounds, rolled repeatedly by one continuing stream.  The stream is sequential in
    the reference; the port splits it into per-thread chunks by jump-ahead and repairs chunks
    after a rejected batch in order (or_roll_batches_mt: the same results)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    O.build()
    cores = cpu_cores()
    bounds = O.gen_bounds(7, 2 * sample_batches)
    src = O.pcg64(O.array_seed(7, 1))
    O.roll_batches_mt(src, bounds, 2, nthreads=cores)  # warm-up (threads, pages)
    reps, t = 0, time.perf_counter()
    while True:
        O.roll_batches_mt(src, bounds, 2, nthreads=cores)
        reps += 1
        dt = time.perf_counter() - t
        if dt >= target_s:
            break
    return {"value": 2 * sample_batches * reps / dt, "unit": "rolls/s", "cores": cores, "kind": "port",
            "sample": f"{reps} x {sample_batches} batches of C2 bounds on one continuing stream (the reference's "
                      f"roll_batch loop in oracle/oracle.c, chunked over {cores} threads by jump-ahead: "
                      f"or_roll_batches_mt), {dt:.1f}s"}


# ------------------------------------------------------------------------------ shuffles
SHUFFLE_CFG = {
    "c3": {"n": 64, "arrays": 1 << 20, "seed": 1234, "eb": 4, "workload": "C3: 2^20 independent shuffles of u32[64], seeds hash(1234,a)"},
    "c4": {"n": 4096, "arrays": 1 << 16, "seed": 99, "eb": 4, "workload": "C4: 65,536 independent shuffles of u32[4096], seeds hash(99,a)"},
    "c5": {"n": 1 << 20, "arrays": 256, "seed": 5, "eb": 8, "workload": "C5: 256 independent shuffles of u64[2^20] (payload = words of pcg64(5)), seeds hash(5,a), HBM-resident"},
}


def bench_shuffle(cfg, args, torch, B, ws, rank, steps=None):
    n, na, eb = cfg["n"], cfg["arrays"], cfg["eb"]
    base = rank * na
    if eb == 8:  # payload: consecutive words of pcg64(seed) (this rank's section)
        data = B.pcg64_fill(cfg["seed"], n * na, offset=base * n)
    else:
        data = torch.arange(n, dtype=torch.int32, device="cuda").repeat(na)
    K = steps or args.steps
    for _ in range(args.warmup):
        B.shuffle_many(data, n, cfg["seed"], array_index_base=base, generator=args.generator)
    kernel = B.last_kernel()
    soak(torch, lambda: B.shuffle_many(data, n, cfg["seed"], array_index_base=base, generator=args.generator))
    barrier(torch, ws)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with ClockSampler(torch.cuda.current_device()) as clk:
        for a, b in evs:
            a.record()
            B.shuffle_many(data, n, cfg["seed"], array_index_base=base, generator=args.generator)
            b.record()
        torch.cuda.synchronize()
    per = [a.elapsed_time(b) for a, b in evs]
    total_ms = max_over_ranks(torch, evs[0][0].elapsed_time(evs[-1][1]), ws)
    elems = n * na * K * ws
    t = statistics.mean(per) / 1e3
    peak, kind = load_peaks()
    achieved = 2 * eb * n * na / t / 1e9
    res = {"workload": cfg["workload"], "value": elems / (total_ms / 1e3), "unit": "elements/s",
           "ms_per_step": total_ms / K, "kernel": kernel,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "traffic": load_traffic().get(kernel.split("<")[0]),
                        "algorithmic_bytes_per_launch": 2 * eb * n * na, "peak_source": kind},
           "clocks": clk.summary(), "gpu_launches": K}
    if eb == 4 and "large" not in kernel:  # payload staged in shared memory
        res["roofline_smem"] = smem_roofline(n * na / t, kernel)
    if "large" in kernel:  # payload in HBM: random accesses
        res["roofline_random"] = random_roofline((n - 1) * na / t, n * na * eb / 2**20)
    return res


def bench_c1(args, torch, B):
    import numpy as np

    z = np.arange(10000, dtype=np.uint32)
    for _ in range(3):
        B.shuffle_batched(B.Pcg64Source(42), z.copy())
    ts = []
    for _ in range(max(5, args.steps)):
        zz = z.copy()
        s = B.Pcg64Source(42)
        t = time.perf_counter()
        B.shuffle_batched(s, zz)
        ts.append(time.perf_counter() - t)
    dev = torch.arange(10000, dtype=torch.int32, device="cuda")
    from paper_2408_06213_b200 import _native as N

    ds = B.DeviceStream(42)
    regs = B.DEFAULT_SCHEDULE._regimes()
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in evs:
        a.record()
        N.check(N.lib().br_shuffle_stream(C.c_void_p(dev.data_ptr()), 4, 10000, C.c_void_p(ds.state.data_ptr()),
                                          regs, len(regs), 0, None, sp), "c1")
        b.record()
    torch.cuda.synchronize()
    kern = statistics.median([a.elapsed_time(b) for a, b in evs[5:]])
    return {"workload": "C1: one u32[10,000] stream shuffle, pcg64 seed 42 (drop-in shuffle_batched on a numpy "
                        "array: upload, kernel, download, state round trip)",
            "e2e_ms_per_shuffle": statistics.median(ts) * 1e3, "kernel_ms": kern,
            "value": 10000 / statistics.median(ts), "unit": "elements/s"}


def cpu_baseline_shuffle(cfg, sample_arrays):
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    O.build()
    n = cfg["n"]
    if cfg["eb"] == 8:
        sample_arrays = max(sample_arrays, cpu_cores())
    data = np.tile(np.arange(n, dtype=np.uint32 if cfg["eb"] == 4 else np.uint64), sample_arrays)
    t = time.perf_counter()
    O.shuffle_segmented(data, n, cfg["seed"], nthreads=0)
    dt = time.perf_counter() - t
    return {"value": n * sample_arrays / dt, "unit": "elements/s", "cores": cpu_cores(), "kind": "port",
            "sample": f"{sample_arrays} arrays of {n} (oracle shuffle_batched per array, OpenMP over arrays), {dt:.2f}s"}


# ------------------------------------------------------------------------------ reference arm
def run_reference(args, ws, rank):
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    O.build()
    cfg = args.config
    if cfg == "c2":
        sample = 1 << 21
        bounds = O.gen_bounds(7, 2 * sample)
        src = O.pcg64(O.array_seed(7, 1))
        cores = cpu_cores()
        for _ in range(args.warmup):
            O.roll_batches_mt(src, bounds, 2, nthreads=cores)
        t = time.perf_counter()
        for _ in range(args.steps):
            O.roll_batches_mt(src, bounds, 2, nthreads=cores)
        dt = time.perf_counter() - t
        value, unit = 2 * sample * args.steps / dt, "rolls/s"
        desc = (f"{sample} batches of C2 per step (one continuing stream; the reference roll_batch loop chunked over "
                f"{cores} threads by jump-ahead, or_roll_batches_mt)")
    else:
        c = SHUFFLE_CFG[cfg]
        n = c["n"]
        arrays = max(1, (1 << 22) // n)
        if c["eb"] == 8:
            arrays = max(arrays, cpu_cores())
            data = O.pcg64_fill(O.pcg64(c["seed"]), 0, n * arrays)
        else:
            data = __import__("numpy").tile(__import__("numpy").arange(n, dtype="uint32"), arrays)
        for _ in range(args.warmup):
            O.shuffle_segmented(data, n, c["seed"], nthreads=0)
        t = time.perf_counter()
        for _ in range(args.steps):
            O.shuffle_segmented(data, n, c["seed"], nthreads=0)
        dt = time.perf_counter() - t
        value, unit, cores = n * arrays * args.steps / dt, "elements/s", cpu_cores()
        desc = f"{arrays} arrays of {n} per step, OpenMP over arrays"
    metric, unit_b, config, dtype = headline(args, ws)
    assert unit == unit_b
    config = dict(config, reference_note="oracle/oracle.c port of the reference (pure Python upstream, so there is "
                                         "no compiled reference to run); each step a bounded sample: " + desc)
    line = {"impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": config,
            "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "port", "sample": desc},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


# ------------------------------------------------------------------------------ main
def headline(args, ws):
    """metric, unit, config and dtype of the line (shared by both arms)."""
    if args.config == "c2":
        config = {"workload": "C2: BASELINE configs[1], 2^25 batches x k=2 bounded rolls per GPU, bounds iid "
                              "U[2,2^16) from seed 7, words from pcg64(hash(7,1)); output 2^26 u32 rolls + 2^25 u8 "
                              "words per GPU", "batches_per_gpu": NB_C2, "k": 2,
                  "l2": "inputs+outputs 544 MiB per step > 126 MB L2 (no flush needed)",
                  "parallelism": f"dp{ws} (stream sections by jump-ahead)", "generator": args.generator}
        return "bounded rolls/sec (C2: 2^25 batches of k=2 per GPU, bounds U[2,2^16))", "rolls/s", config, "u64"
    cfg = SHUFFLE_CFG[args.config]
    config = {"workload": cfg["workload"], "l2": "payload larger than L2", "parallelism": f"dp{ws} (arrays)",
              "generator": args.generator}
    return "shuffled elements/sec", "elements/s", config, "u32" if cfg["eb"] == 4 else "u64"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--generator", default="pcg64", choices=["pcg64", "lehmer", "chacha"],
                    help="word generator of the timed path (the headline is pcg64)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    ws, rank, local = dist_info()
    if args.impl == "reference":
        line = run_reference(args, ws, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    import torch

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__

    if rank == 0:
        __graft_entry__.build()
    if ws > 1:
        torch.distributed.barrier()
    import paper_2408_06213_b200 as B

    metric, unit, config, dtype = headline(args, ws)
    if args.config == "c2":
        r = bench_c2(args, torch, B, ws, rank)
    else:
        r = bench_shuffle(SHUFFLE_CFG[args.config], args, torch, B, ws, rank)
        r["e2e"] = None
    line = {"metric": metric, "value": r["value"], "unit": unit, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic (BASELINE configs; generated on device)",
            "config": config, "roofline": r["roofline"], "clocks": r["clocks"], "gpu_launches": r["gpu_launches"],
            "e2e": r.get("e2e")}
    for extra_roof in ("roofline_int", "roofline_smem"):
        if r.get(extra_roof):
            line[extra_roof] = r[extra_roof]
    if "cross_rank_rejections" in r:
        line["cross_rank_rejections"] = r["cross_rank_rejections"]
    if not args.no_secondary:
        sec = {}
        for key in ("c3", "c4", "c5"):
            if key != args.config:
                sec[key] = bench_shuffle(SHUFFLE_CFG[key], args, torch, B, ws, rank,
                                         steps={"c3": args.steps, "c4": min(args.steps, 10)}.get(key, min(args.steps, 3)))
        if ws == 1:
            sec["c1"] = bench_c1(args, torch, B)
        line["secondary"] = sec
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        if args.config == "c2":
            line["cpu_baseline"] = cpu_baseline_c2()
        else:
            line["cpu_baseline"] = cpu_baseline_shuffle(SHUFFLE_CFG[args.config], max(1, (1 << 23) // SHUFFLE_CFG[args.config]["n"]))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
