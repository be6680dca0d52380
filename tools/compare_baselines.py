"""Device timing of the batched path against the division-based baselines and across
generators.  One JSON line per measurement on stdout.

    python tools/compare_baselines.py [--steps 10]

Rolls: C2 (2^25 batches of k=2) through br_roll_batches vs br_roll_batches_naive.
Shuffles: C3 / C4 / C5 through shuffle_many with the default schedule, the pair schedule
and shuffle_naive_batched (division pairs), for pcg64 / lehmer / chacha.
CUDA events around each call on the launching stream, after warm-up.
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_06213_b200 as B  # noqa: E402
from paper_2408_06213_b200 import _native as N  # noqa: E402
from paper_2408_06213_b200 import cost_model  # noqa: E402


def timed(fn, steps, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    L = N.lib()
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if args.only in ("", "c2"):
        for gen in ("pcg64", "lehmer", "chacha"):
            nb = bench.NB_C2
            bounds, stream, rolls, words = bench.setup_c2(torch, B, 0, nb, gen)
            p = [C.c_void_p(x.data_ptr()) for x in (bounds, stream.state, rolls, words)]
            ws = C.c_void_p(stream.workspace.data_ptr())
            for naive in (False, True):
                f = L.br_roll_batches_naive if naive else L.br_roll_batches
                ms = timed(lambda: f(p[0], 2, nb, p[1], p[2], p[3], None, None, ws, sp), args.steps)
                print(json.dumps({"workload": "C2 rolls k=2", "generator": gen,
                                  "algorithm": "roll_batch_naive" if naive else "roll_batch",
                                  "ms": ms, "rolls_per_s": 2 * nb / (ms / 1e3)}), flush=True)
            del bounds, rolls, words, stream
            torch.cuda.empty_cache()
    for key in ("c3", "c4", "c5"):
        if args.only and args.only != key:
            continue
        cfg = bench.SHUFFLE_CFG[key]
        n, na, eb = cfg["n"], cfg["arrays"], cfg["eb"]
        data = (B.pcg64_fill(cfg["seed"], n * na) if eb == 8
                else torch.arange(n, dtype=torch.int32, device="cuda").repeat(na))
        steps = max(2, args.steps // (4 if key == "c5" else 1))
        for gen in ("pcg64", "lehmer", "chacha"):
            for alg, kw in (("shuffle_6", {}), ("shuffle_2", {"schedule": B.PAIR_SCHEDULE}),
                            ("naive_shuffle_2", {"naive": True}),
                            ("shuffle_6_gpu_cost_model", {"schedule": cost_model.gpu_schedule(gen)})):
                ms = timed(lambda: B.shuffle_many(data, n, cfg["seed"], generator=gen, **kw), steps, warmup=2)
                print(json.dumps({"workload": cfg["workload"], "generator": gen, "algorithm": alg, "ms": ms,
                                  "elements_per_s": n * na / (ms / 1e3), "kernel": B.last_kernel()}), flush=True)
        del data
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
