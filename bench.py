#!/usr/bin/env python
"""Benchmark of the B200 batched-dice path (BASELINE.json metric: bounded rolls/sec and
shuffled elements/sec per GPU and box-wide vs roofline).

Headline workload = BASELINE.json configs[1] ("C2"): 2^25 batches of k=2 bounded rolls,
bounds iid U[2, 2^16) drawn from seed 7 (2 + roll_single(pcg64(7), 65534), generated on the
device by our own k=1 roll kernel), roll words from pcg64(array_seed(7, 1)).  One step = one
bulk roll_batches over the resident bounds (2^26 rolls).  Inputs (256 MiB bounds) and outputs
(256 MiB rolls + 32 MiB words) exceed the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config c2|c3|c4|c5]

Under torchrun (N > 1) the job is split (strong scaling): C2's one stream is cut
into N contiguous batch sections (rank r jumps ahead to its first word; the only exchange is
the all-gather of per-rank rejection counts, after which a shifted section is re-rolled), and
the shuffle configs' arrays into N contiguous array ranges (array_index_base; no exchange).
The shuffle configs C3/C4/C5 (and C1 at N=1) are reported under "secondary", each with its
roofline, the same-run CPU baseline and an end-to-end number through shuffle_many on pinned
host buffers.
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


def run_ahead(torch):
    """Queue ~0.5 ms of device idle-spin in front of a timed region, so that the host has the
    first steps enqueued before the device reaches the start event: the region then measures
    device time at any K, not the host's launch latency of the first call."""
    torch.cuda._sleep(1_000_000)


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
def c2_section(ws, rank):
    """This rank's contiguous (first_batch, count) of the one C2 stream."""
    from paper_2408_06213_b200 import shard

    return shard.even_split(NB_C2, ws, rank)


def setup_c2(torch, B, first, nb, generator="pcg64"):
    from paper_2408_06213_b200 import _native as N

    # bounds: 2 + roll_single(pcg64(7), 65534), drawn sequentially for the whole job (every
    # rank draws all 2^26 and keeps its section, so the sequence is exact at any N)
    st = N.Pcg64State()
    N.lib().br_pcg64_seed(7, C.byref(st))
    gen = B.DeviceStream.from_struct(st)
    spans = torch.full((2 * NB_C2,), 65534, dtype=torch.int32, device="cuda")
    r = B.roll_batches(gen, spans, 1)
    bounds = (r.rolls[2 * first: 2 * (first + nb)] + 2).contiguous()
    del spans, r
    # roll stream: make_source(generator, array_seed(7, 1)) advanced to this rank's first batch
    seed = N.lib().br_array_seed(7, 1)
    if generator == "chacha":
        st = N.ChachaState()
        N.lib().br_chacha_seed(seed, C.byref(st))
    else:
        st = N.Pcg64State()
        (N.lib().br_lehmer_seed if generator == "lehmer" else N.lib().br_pcg64_seed)(seed, C.byref(st))
    N.lib().br_pcg64_advance(C.byref(st), first)
    stream = B.DeviceStream.from_struct(st)
    rolls = torch.empty(2 * nb, dtype=torch.int32, device="cuda")
    words = torch.empty(nb, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    return bounds, stream, rolls, words


def bench_c2(args, torch, B, ws, rank):
    from paper_2408_06213_b200 import _native as N

    L = N.lib()
    first, nb = c2_section(ws, rank)
    bounds, stream, rolls, words = setup_c2(torch, B, first, nb, args.generator)
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    ptrs = [C.c_void_p(x.data_ptr()) for x in (bounds, stream.state, rolls, words)]
    wsp = C.c_void_p(stream.workspace.data_ptr())

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
        run_ahead(torch)
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
    run_ahead(torch)
    for i in range(K):
        e0[i].record()
        N.check(L.br_roll_batches_phase(ptrs[0], 2, nb, ptrs[1], ptrs[2], ptrs[3], None, None, wsp, 1, sp), "main")
        e1[i].record()
        N.check(L.br_roll_batches_phase(ptrs[0], 2, nb, ptrs[1], ptrs[2], ptrs[3], None, None, wsp, 2, sp), "fixup")
    torch.cuda.synchronize()
    main_ms = [a.elapsed_time(b) for a, b in zip(e0, e1)]
    barrier(torch, ws)
    total_ms = max_over_ranks(torch, total_ms, ws)
    # the one exchange of a split stream: per-rank rejection counts (all zero unless a batch
    # was rejected, P ~ 2^-10 per 2^25 batches); a rank after a rejecting rank is shifted and
    # re-rolls its section (shard.sharded_rolls; gloo-tested in tests/test_multi.py)
    extra = C.c_uint64()
    N.check(L.br_roll_check(wsp, sp, C.byref(extra)), "check")
    extras = [int(extra.value)]
    if ws > 1:
        from paper_2408_06213_b200 import shard

        extras = shard.all_gather_ints(int(extra.value), device="cuda")
    rolls_total = 2 * NB_C2 * K
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
        "cross_rank_rejections": extras,
    }
    # end to end through the public API with host (pinned) buffers and the production status
    # check (br_roll_check: one synchronisation and a 16-byte read per call)
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
        B.roll_batches(stream, hb, 2, out=(hrolls, hwords))
    t1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(torch, t0.elapsed_time(t1), ws)
    res["e2e"] = {"value": 2 * NB_C2 * E / (e2e_ms / 1e3), "unit": "rolls/s",
                  "h2d_bytes_per_step": 8 * nb, "d2h_bytes_per_step": 8 * nb + nb, "steps": E,
                  "api": "paper_2408_06213_b200.roll_batches(host pinned tensors, 16-chunk pipelined copies, "
                         "check=True)"}
    return res


def cpu_c2(cores, steps=None, warmup=1, target_s=None):
    """The oracle port of roll_batch (the reference's batched.py:102-123 loop, oracle/oracle.c)
    on `cores` host threads over the FULL C2 config per step: 2^25 batches of the C2 bounds on
    one continuing stream, rolls and words into preallocated arrays (what the device call
    returns).  The reference's single stream is cut into per-thread chunks by jump-ahead and
    chunks after a rejected batch are repaired in order (or_roll_batches_mt: the same
    results).  Used by both the reference arm and this arm's cpu_baseline, so the two agree."""
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    O.build()
    bounds = O.gen_bounds(7, 2 * NB_C2)
    src = O.pcg64(O.array_seed(7, 1))
    rolls = np.empty(2 * NB_C2, dtype=np.uint32)
    wds = np.empty(NB_C2, dtype=np.uint8)
    rolls.fill(0)
    wds.fill(0)  # pages touched before timing
    t_w = time.perf_counter()
    w = 0
    while w < warmup or time.perf_counter() - t_w < 0.5:  # W steps and at least 0.5 s: the host
        O.roll_batches_mt(src, bounds, 2, nthreads=cores, out=(rolls, wds))  # threads and clocks have ramped
        w += 1
    reps, t = 0, time.perf_counter()
    while True:
        O.roll_batches_mt(src, bounds, 2, nthreads=cores, out=(rolls, wds))
        reps += 1
        dt = time.perf_counter() - t
        if (steps is not None and reps >= steps) or (steps is None and dt >= target_s):
            break
    return 2 * NB_C2 * reps / dt, reps, dt


def python_reference_rate(cfg_key, budget_s=2.0):
    """The vendored reference package itself (baseline/_ref, tools/vendor_reference.sh) on one
    core: the pure-Python path a reference user runs today.  Context only (the port above is
    the conservative, much faster CPU denominator).  None when the package is not vendored."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "batchrand")):
        return None
    sys.path.insert(0, ref_dir)
    try:
        import batchrand as R
    except Exception:
        return None
    finally:
        sys.path.remove(ref_dir)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    if cfg_key == "c2":
        import numpy as np

        bounds = O.gen_bounds(7, 2 * 50000)
        src = R.make_source("pcg64", O.array_seed(7, 1))
        t, done = time.perf_counter(), 0
        while done < 50000 and time.perf_counter() - t < budget_s:
            for i in range(done, min(done + 1000, 50000)):
                R.roll_batch(src, R.BatchSpec(R.RadixBases.of((int(bounds[2 * i]), int(bounds[2 * i + 1])))))
            done = min(done + 1000, 50000)
        dt = time.perf_counter() - t
        return {"value": 2 * done / dt, "unit": "rolls/s", "cores": 1, "kind": "reference",
                "sample": f"{done} C2 batches through the reference's roll_batch(src, BatchSpec(RadixBases.of(b)))"}
    cfg = SHUFFLE_CFG[cfg_key]
    n = cfg["n"]
    t, arrays = time.perf_counter(), 0
    while True:
        z = list(range(n))
        R.shuffle_batched(R.make_source("pcg64", O.array_seed(cfg["seed"], arrays)), z)
        arrays += 1
        if time.perf_counter() - t >= budget_s:
            break
    dt = time.perf_counter() - t
    return {"value": n * arrays / dt, "unit": "elements/s", "cores": 1, "kind": "reference",
            "sample": f"{arrays} arrays of {n} through the reference's shuffle_batched(make_source('pcg64', "
                      f"hash({cfg['seed']}, a)), list(range({n})))"}


# ------------------------------------------------------------------------------ shuffles
SHUFFLE_CFG = {
    "c3": {"n": 64, "arrays": 1 << 20, "seed": 1234, "eb": 4, "workload": "C3: 2^20 independent shuffles of u32[64], seeds hash(1234,a)"},
    "c4": {"n": 4096, "arrays": 1 << 16, "seed": 99, "eb": 4, "workload": "C4: 65,536 independent shuffles of u32[4096], seeds hash(99,a)"},
    "c5": {"n": 1 << 20, "arrays": 256, "seed": 5, "eb": 8, "workload": "C5: 256 independent shuffles of u64[2^20] (payload = words of pcg64(5)), seeds hash(5,a), HBM-resident"},
}


def shuffle_payload(torch, B, cfg, first, count):
    n = cfg["n"]
    if cfg["eb"] == 8:  # payload: consecutive words of pcg64(seed) (this rank's arrays)
        return B.pcg64_fill(cfg["seed"], n * count, offset=first * n)
    return torch.arange(n, dtype=torch.int32, device="cuda").repeat(count)


def bench_shuffle(cfg, args, torch, B, ws, rank, steps=None, e2e=True):
    from paper_2408_06213_b200 import shard

    n, eb = cfg["n"], cfg["eb"]
    first, na = shard.even_split(cfg["arrays"], ws, rank)
    data = shuffle_payload(torch, B, cfg, first, na)
    K = steps or args.steps

    def call(d):
        return B.shuffle_many(d, n, cfg["seed"], array_index_base=first, generator=args.generator)

    for _ in range(args.warmup):
        call(data)
    kernel = B.last_kernel()
    soak(torch, lambda: call(data))
    barrier(torch, ws)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with ClockSampler(torch.cuda.current_device()) as clk:
        run_ahead(torch)
        for a, b in evs:
            a.record()
            call(data)
            b.record()
        torch.cuda.synchronize()
    per = [a.elapsed_time(b) for a, b in evs]
    total_ms = max_over_ranks(torch, evs[0][0].elapsed_time(evs[-1][1]), ws)
    elems = n * cfg["arrays"] * K
    t = statistics.mean(per) / 1e3
    peak, kind = load_peaks()
    achieved = 2 * eb * n * na / t / 1e9
    res = {"workload": cfg["workload"], "value": elems / (total_ms / 1e3), "unit": "elements/s",
           "ms_per_step": total_ms / K, "kernel": kernel,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "traffic": load_traffic().get(kernel.split("<")[0]),
                        "algorithmic_bytes_per_launch": 2 * eb * n * na, "peak_source": kind},
           "clocks": clk.summary(), "gpu_launches": K, "l2": "payload larger than L2 (no flush needed)"}
    if eb == 4 and "large" not in kernel and "stage" not in kernel:  # payload staged in shared memory
        res["roofline_smem"] = smem_roofline(n * na / t, kernel)
    del data
    if e2e:
        # end to end through shuffle_many on a pinned host tensor: every step copies the arrays
        # up, shuffles them and copies them back (chunked, copies overlapping the shuffles)
        host = shuffle_payload(torch, B, cfg, first, na).cpu().pin_memory()
        call(host)  # warm-up (copy streams, device chunk buffers)
        E = 3
        barrier(torch, ws)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(E):
            call(host)
        t1.record()
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(torch, t0.elapsed_time(t1), ws)
        res["e2e"] = {"value": n * cfg["arrays"] * E / (e2e_ms / 1e3), "unit": "elements/s",
                      "h2d_bytes_per_step": eb * n * na, "d2h_bytes_per_step": eb * n * na, "steps": E,
                      "api": "paper_2408_06213_b200.shuffle_many(pinned host tensor, 8-chunk pipelined copies)"}
        del host
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


def cpu_shuffle(cfg, cores, target_s=3.0, steps=None):
    """The oracle port of shuffle_batched (shuffle.py:149-225, oracle/oracle.c) over a bounded
    sample of the config's arrays, OpenMP over arrays on `cores` threads.  The sample is sized
    from a short calibration run so that it takes about target_s."""
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    O.build()
    n = cfg["n"]

    def payload(arrays):
        if cfg["eb"] == 8:
            return O.pcg64_fill(O.pcg64(cfg["seed"]), 0, n * arrays)
        return np.tile(np.arange(n, dtype=np.uint32), arrays)

    arrays = max(cores, (1 << 18) // n)
    t = time.perf_counter()
    O.shuffle_segmented(payload(arrays), n, cfg["seed"], nthreads=cores)
    per_array = (time.perf_counter() - t) / arrays
    arrays = int(min(cfg["arrays"], max(cores, target_s / max(per_array, 1e-9))))
    arrays = max(cores, arrays - arrays % cores)
    data = payload(arrays)
    # the whole config fits the budget: repeat it (the arrays keep their seeds, so every
    # repetition is the same work on the previous output)
    reps = steps or max(1, int(target_s / max(per_array * arrays, 1e-9)))
    t = time.perf_counter()
    for _ in range(reps):
        O.shuffle_segmented(data, n, cfg["seed"], nthreads=cores)
    dt = time.perf_counter() - t
    return n * arrays * reps / dt, arrays, reps, dt


def cpu_baseline_shuffle(cfg, key):
    cores = cpu_cores()
    v, arrays, reps, dt = cpu_shuffle(cfg, cores)
    out = {"value": v, "unit": "elements/s", "cores": cores, "kind": "port",
           "sample": f"{reps} x {arrays} of the {cfg['arrays']} arrays of {cfg['n']} (the reference's shuffle_batched "
                     f"per array in oracle/oracle.c, OpenMP over arrays), {dt:.2f}s"}
    py = python_reference_rate(key)
    if py is not None:
        out["python_reference_1core"] = py
    return out


# ------------------------------------------------------------------------------ reference arm
def run_reference(args, ws, rank):
    if rank != 0:
        return None
    cores = cpu_cores()
    cfg = args.config
    if cfg == "c2":
        value, reps, dt = cpu_c2(cores, steps=args.steps, warmup=args.warmup)
        unit = "rolls/s"
        desc = (f"the full C2 config per step ({NB_C2} batches on one continuing stream; the reference's roll_batch "
                f"loop in oracle/oracle.c chunked over {cores} threads by jump-ahead, or_roll_batches_mt)")
    else:
        c = SHUFFLE_CFG[cfg]
        value, arrays, reps, dt = cpu_shuffle(c, cores, target_s=1.0, steps=args.steps)
        unit = "elements/s"
        desc = f"{arrays} of the {c['arrays']} arrays of {c['n']} per step, OpenMP over arrays"
    metric, unit_b, config, dtype = headline(args, 1)
    assert unit == unit_b
    config = dict(config, reference_note="oracle/oracle.c port of the reference (pure Python upstream, so there is "
                                         "no compiled reference to run); " + desc)
    line = {"impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / reps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": config,
            "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "port", "sample": desc},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    py = python_reference_rate(cfg)
    if py is not None:
        line["cpu_baseline"]["python_reference_1core"] = py
    return line


# ------------------------------------------------------------------------------ main
def headline(args, ws):
    """metric, unit, config and dtype of the line (shared by both arms)."""
    if args.config == "c2":
        config = {"workload": "C2: BASELINE configs[1], 2^25 batches x k=2 bounded rolls on one stream, bounds iid "
                              "U[2,2^16) from seed 7, words from pcg64(hash(7,1)); output 2^26 u32 rolls + 2^25 u8 "
                              "words", "batches": NB_C2, "k": 2,
                  "l2": "inputs+outputs 544 MiB per step > 126 MB L2 (no flush needed)",
                  "parallelism": f"dp{ws} (one stream cut into {ws} sections by jump-ahead)",
                  "generator": args.generator}
        return "bounded rolls/sec (C2: 2^25 batches of k=2, bounds U[2,2^16))", "rolls/s", config, "u64"
    cfg = SHUFFLE_CFG[args.config]
    config = {"workload": cfg["workload"], "l2": "payload larger than L2", "parallelism": f"dp{ws} (arrays)",
              "generator": args.generator}
    return "shuffled elements/sec", "elements/s", config, "u32" if cfg["eb"] == 4 else "u64"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
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
    line = {"metric": metric, "value": r["value"], "unit": unit, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "strong",
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
                                         steps={"c3": args.steps, "c4": min(args.steps, 10)}.get(key, min(args.steps, 5)))
                if rank == 0 and ws == 1 and not args.no_cpu_baseline:
                    sec[key]["cpu_baseline"] = cpu_baseline_shuffle(SHUFFLE_CFG[key], key)
        if ws == 1:
            sec["c1"] = bench_c1(args, torch, B)
        line["secondary"] = sec
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cores = cpu_cores()
        if args.config == "c2":
            # the same procedure as the reference arm (--impl reference): W warm-up and K timed
            # full-config steps, so the two CPU numbers measure the same thing
            v, reps, dt = cpu_c2(cores, steps=args.steps, warmup=args.warmup)
            line["cpu_baseline"] = {
                "value": v, "unit": "rolls/s", "cores": cores, "kind": "port",
                "sample": f"{reps} x the full C2 config ({NB_C2} batches on one continuing stream; the reference's "
                          f"roll_batch loop in oracle/oracle.c chunked over {cores} threads by jump-ahead: "
                          f"or_roll_batches_mt, the same call the reference arm times), {dt:.1f}s"}
            py = python_reference_rate("c2")
            if py is not None:
                line["cpu_baseline"]["python_reference_1core"] = py
        else:
            line["cpu_baseline"] = cpu_baseline_shuffle(SHUFFLE_CFG[args.config], args.config)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
