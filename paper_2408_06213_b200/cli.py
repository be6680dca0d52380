"""Command line for the device path, mirroring the reference CLI (cli.py:256-293).

    python -m paper_2408_06213_b200.cli bench [--generator pcg64|lehmer] [--sizes 64,...]
                                              [--algorithms shuffle_6_b200,...] [--output x.csv]
    python -m paper_2408_06213_b200.cli shuffle [input] [--seed S] [--generator G] [--max-batch K]

`bench` writes the reference's CSV schema (cli.py:27, 124-127):
algorithm,generator,n,avg_ns_per_element,min_ns_per_element.  Rows produced here can be
concatenated with the reference's own CSV and fed to its benchplots ratio curves
(plots.py:90-156).  The device algorithms are registered like the reference's ALGORITHMS
(cli.py:44-49):

  * ``shuffle_b200`` / ``naive_shuffle_2_b200`` / ``shuffle_2_b200`` / ``shuffle_6_b200``: one
    array per call through the drop-in API on a device-resident tensor (includes the
    generator-state round trip that a single call implies) -- the reference's four
    algorithms (cli.py:44-49) on the device;
  * ``many_naive_2_b200`` / ``many_6_b200``: the bulk segmented shuffle of 4096 independent
    arrays of length n per call (ns per element amortised over all arrays) -- the workload a
    GPU is built for -- with division-split pairs and with the default 6-dice schedule.

Each cell repeats the call until the time budget is spent (cli.py:75-121), timed with CUDA
events; the "min" column is the fastest single call.
"""

from __future__ import annotations

import argparse
import os
import sys
import warnings

from . import batchrand as B

CSV_HEADER = "algorithm,generator,n,avg_ns_per_element,min_ns_per_element"
DEFAULT_SIZES = tuple(1 << p for p in range(6, 17))
DEFAULT_BUDGET_NS = 2_000_000  # device calls are ~10-100 us; 2 ms per cell keeps the spread low
MANY_ARRAYS = 4096


def _one_array(schedule):
    def run(source, data):
        return B.shuffle_batched(source, data, schedule)

    return run


def _unbatched(source, data):
    return B.shuffle_unbatched(source, data)


def _naive(source, data):
    return B.shuffle_naive_batched(source, data)


ALGORITHMS = {
    "shuffle_b200": _unbatched,
    "naive_shuffle_2_b200": _naive,
    "shuffle_2_b200": _one_array(B.default_schedule(2)),
    "shuffle_6_b200": _one_array(B.default_schedule(6)),
    "many_naive_2_b200": None,  # bulk segmented shuffles, see bench()
    "many_6_b200": None,
}


def bench(generator="pcg64", sizes=DEFAULT_SIZES, algorithms=tuple(ALGORITHMS), seed=1,
          budget_ns=DEFAULT_BUDGET_NS):
    """One (algorithm, n) record per cell: avg and min ns per element (cli.py:75-121)."""
    import torch

    for name in algorithms:
        if name not in ALGORITHMS:
            raise B.BatchRandError(f"unknown algorithm {name!r}; expected one of {sorted(ALGORITHMS)}")
    records = []
    for name in algorithms:
        for n in sizes:
            if name.startswith("many_"):
                data = torch.arange(n, dtype=torch.int32, device="cuda").repeat(MANY_ARRAYS)
                elems = n * MANY_ARRAYS

                def call(data=data, n=n, naive=name == "many_naive_2_b200"):
                    B.shuffle_many(data, n, seed, generator=generator, naive=naive)
            else:
                source = B.make_source(generator, seed)
                data = torch.arange(n, dtype=torch.int32, device="cuda")
                elems = n
                fn = ALGORITHMS[name]

                def call(fn=fn, source=source, data=data):
                    fn(source, data)
            call()
            torch.cuda.synchronize()
            total, best, reps = 0.0, None, 0
            while total < budget_ns:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                call()
                b.record()
                b.synchronize()
                dt = a.elapsed_time(b) * 1e6
                total += dt
                reps += 1
                best = dt if best is None or dt < best else best
            avg, low = total / reps / elems, best / elems
            if low < 0.9 * avg:
                warnings.warn(f"unstable timing for {name} at n={n}: min {low:.3f} < 90% of avg {avg:.3f} ns/element",
                              stacklevel=2)
            records.append((name, generator, n, avg, low))
    return records


def write_csv(records, stream) -> None:
    stream.write(CSV_HEADER + "\n")
    for name, gen, n, avg, low in records:
        stream.write(f"{name},{gen},{n},{avg:.3f},{low:.3f}\n")


def _cmd_bench(args) -> int:
    records = bench(args.generator, args.sizes, args.algorithms, args.seed)
    if args.output:
        with open(args.output, "w", encoding="utf-8", newline="\n") as fh:
            write_csv(records, fh)
    else:
        write_csv(records, sys.stdout)
    return 0


def _cmd_shuffle(args) -> int:
    """cli.py:219-239 on the device: the lines are permuted through an index shuffle."""
    if args.input and args.input != "-":
        with open(args.input, "r", encoding="utf-8") as fh:
            lines = fh.read().splitlines()
    else:
        lines = sys.stdin.read().splitlines()
    seed = args.seed if args.seed is not None else int.from_bytes(os.urandom(8), "little")
    if not 2 <= args.max_batch <= 6:
        raise SystemExit("--max-batch must be in [2, 6] on the device path")
    B.shuffle_batched(B.make_source(args.generator, seed), lines, B.default_schedule(args.max_batch))
    out = open(args.output, "w", encoding="utf-8", newline="\n") if args.output else sys.stdout
    try:
        for line in lines:
            out.write(line + "\n")
    finally:
        if args.output:
            out.close()
    return 0


def _sizes_arg(text: str):
    try:
        sizes = tuple(int(part) for part in text.split(",") if part)
    except ValueError:
        raise argparse.ArgumentTypeError(f"bad size list {text!r}") from None
    if not sizes or any(n < 2 for n in sizes):
        raise argparse.ArgumentTypeError("sizes must be integers >= 2")
    return sizes


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="batchrand-b200", description="Device batched dice rolls and shuffles.")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("bench", help="time the device shuffles, emit the reference CSV schema")
    p.add_argument("--generator", choices=("pcg64", "lehmer", "chacha"), default="pcg64")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--sizes", type=_sizes_arg, default=DEFAULT_SIZES)
    p.add_argument("--algorithms", type=lambda t: tuple(x for x in t.split(",") if x), default=tuple(ALGORITHMS))
    p.add_argument("--output")
    p.set_defaults(func=_cmd_bench)
    p = sub.add_parser("shuffle", help="shuffle input lines on the device")
    p.add_argument("input", nargs="?")
    p.add_argument("--generator", choices=("pcg64", "lehmer", "chacha"), default="pcg64")
    p.add_argument("--seed", type=int, default=None)
    p.add_argument("--output")
    p.add_argument("--max-batch", type=int, default=6)
    p.set_defaults(func=_cmd_shuffle)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
