"""The reference package itself, driven through the B200 path (paper_2408_06213_b200.refbind).

The reference (pkg/src/batchrand, vendored UNMODIFIED into baseline/_ref by
tools/vendor_reference.sh) provides the sources, schedules, specs and the expected results: each
test runs the reference's own pure-Python function on one source object and the device-bound
function (refbind.bind) on an identical one, then compares the outputs, the returned values and
the next words the two sources give afterwards (so the advanced state matches exactly).
"""

import copy
import importlib
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _import_ref():
    if not os.path.isdir(os.path.join(REF_DIR, "batchrand")):
        pytest.skip("reference not vendored (tools/vendor_reference.sh)")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    return importlib.import_module("batchrand")


@pytest.fixture(scope="module")
def ref():
    return _import_ref()


# ------------------------------------------------------------------ host logic (no GPU)
def test_bind_install_uninstall(ref):
    """bind/install/register_algorithms wire the reference's names without a device call."""
    from paper_2408_06213_b200 import refbind

    dev = refbind.bind(ref)
    for name in ("shuffle_batched", "shuffle_unbatched", "shuffle_naive_batched", "partial_shuffle_batch",
                 "roll_batch", "roll_batch_known_threshold", "roll_batch_naive", "digit_pass"):
        assert callable(getattr(dev, name))
    cli = importlib.import_module("batchrand.cli")
    orig = {n: getattr(ref, n) for n in ("shuffle_batched", "roll_batch")}
    orig_shuffle_mod = importlib.import_module("batchrand.shuffle").shuffle_batched
    cpu_rows = dict(cli.ALGORITHMS)
    undo = refbind.install(ref)
    try:
        assert ref.shuffle_batched is not orig["shuffle_batched"]
        assert importlib.import_module("batchrand.shuffle").shuffle_batched is ref.shuffle_batched
        assert ref.roll_batch is not orig["roll_batch"]
        assert set(cli.ALGORITHMS) == set(cpu_rows) | {n + "_b200" for n in cpu_rows}
        assert all(cli.ALGORITHMS[n] is cpu_rows[n] for n in cpu_rows)  # CPU rows untouched
    finally:
        undo()
    assert ref.shuffle_batched is orig["shuffle_batched"] and ref.roll_batch is orig["roll_batch"]
    assert importlib.import_module("batchrand.shuffle").shuffle_batched is orig_shuffle_mod
    assert dict(cli.ALGORITHMS) == cpu_rows


# ------------------------------------------------------------------ device parity
gpu = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(ref):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    from paper_2408_06213_b200 import refbind

    return refbind.bind(ref)


def _same_stream(a, b, count=24):
    """The two sources are at the same position: their next words agree."""
    return [a.next_word() for _ in range(count)] == [b.next_word() for _ in range(count)]


GENS = ("pcg64", "lehmer", "chacha")


@gpu
def test_c1_through_reference_objects(ref, dev):
    """BASELINE configs[0]: the reference's own Pcg64Source(42) and list(range(10000))."""
    for fn in ("shuffle_batched", "shuffle_unbatched"):
        s_ref, s_dev = ref.make_source("pcg64", 42), ref.make_source("pcg64", 42)
        z_ref, z_dev = list(range(10000)), list(range(10000))
        out_ref = getattr(ref, fn)(s_ref, z_ref)
        out_dev = getattr(dev, fn)(s_dev, z_dev)
        assert out_dev is z_dev and out_ref == z_dev, fn
        assert s_dev.state == s_ref.state, fn


@gpu
@pytest.mark.parametrize("gen", GENS)
def test_shuffles_every_generator_and_schedule(ref, dev, gen):
    schedules = [ref.DEFAULT_SCHEDULE, ref.PAIR_SCHEDULE] + [ref.default_schedule(m) for m in range(2, 7)]
    rng = np.random.default_rng(hash(gen) & 0xFFFF)
    lengths = [0, 1, 2, 3, 5, 7, 64, 300, 1000, 4096, 5000]
    for si, sched in enumerate(schedules):
        for n in lengths:
            seed = int(rng.integers(0, 2**63))
            s_ref, s_dev = ref.make_source(gen, seed), ref.make_source(gen, seed)
            for _ in range(int(rng.integers(0, 20))):  # start mid-block / mid-stream
                s_ref.next_word()
                s_dev.next_word()
            z = [int(x) for x in rng.integers(0, 2**31, n)]
            a, b = list(z), list(z)
            ref.shuffle_batched(s_ref, a, sched)
            dev.shuffle_batched(s_dev, b, sched)
            assert a == b, (gen, si, n)
            assert _same_stream(s_ref, s_dev), (gen, si, n)


@gpu
@pytest.mark.parametrize("gen", GENS)
def test_unbatched_naive_partial(ref, dev, gen):
    for n in (2, 3, 10, 257, 2048):
        for fn in ("shuffle_unbatched", "shuffle_naive_batched"):
            s_ref, s_dev = ref.make_source(gen, n), ref.make_source(gen, n)
            a, b = list(range(n)), list(range(n))
            getattr(ref, fn)(s_ref, a)
            getattr(dev, fn)(s_dev, b)
            assert a == b and _same_stream(s_ref, s_dev), (gen, fn, n)
    for n, k in ((52, 2), (52, 6), (5, 5), (1000, 3)):
        ff = ref.falling_factorial(n, k)
        for u in (ff, 1 << 64, ff + 12345):
            s_ref, s_dev = ref.make_source(gen, 9 + k), ref.make_source(gen, 9 + k)
            a, b = list(range(n)), list(range(n))
            u_ref = ref.partial_shuffle_batch(s_ref, a, n, k, u)
            u_dev = dev.partial_shuffle_batch(s_dev, b, n, k, u)
            assert (a, u_ref) == (b, u_dev) and _same_stream(s_ref, s_dev), (gen, n, k, u)


@gpu
@pytest.mark.parametrize("gen", GENS)
def test_roll_batch_streams(ref, dev, gen):
    """Sequences of roll_batch / roll_batch_known_threshold / roll_batch_naive on one source,
    including products close to 2^64 (rejections) and 64-bit bases."""
    cases = [(52, 51), (6,), (6, 6, 6, 6, 6, 6), (0xFFFFFFFF, 3006477107), (1 << 31, 1 << 31, 4), (3,) * 40,
             ((1 << 40) + 7,), ((1 << 63) + 5,), (2,) * 64, (1000, 999, 998, 997, 996)]
    s_ref, s_dev = ref.make_source(gen, 123), ref.make_source(gen, 123)
    for rep in range(3):
        for bases in cases:
            rb = ref.RadixBases.of(bases)
            for spec in (ref.BatchSpec(rb), ref.BatchSpec(rb, upper_bound=rb.product.value)):
                assert dev.roll_batch(s_dev, spec) == ref.roll_batch(s_ref, spec), (gen, bases)
            spec = ref.BatchSpec.with_threshold(rb)
            assert dev.roll_batch_known_threshold(s_dev, spec) == ref.roll_batch_known_threshold(s_ref, spec)
            if len(bases) <= 8 and all(b < 1 << 32 for b in bases):
                assert dev.roll_batch_naive(s_dev, rb) == ref.roll_batch_naive(s_ref, rb), (gen, bases)
    assert _same_stream(s_ref, s_dev)
    for r0 in (0, 1, 2**63, 2**64 - 1, 0x9E3779B97F4A7C15):
        for bases in cases:
            rb = ref.RadixBases.of(bases)
            assert dev.digit_pass(r0, rb) == ref.digit_pass(r0, rb), (r0, bases)


@gpu
def test_fixed_sequence_source(ref, dev):
    words = [int(x) for x in np.random.default_rng(3).integers(0, 2**64 - 1, 4000, dtype=np.uint64)]
    words[5] = 0  # a forced rejection early in the stream
    a_src, b_src = ref.FixedSequenceSource(words), ref.FixedSequenceSource(words)
    a, b = list(range(3000)), list(range(3000))
    ref.shuffle_batched(a_src, a)
    dev.shuffle_batched(b_src, b)
    assert a == b and a_src.cursor == b_src.cursor
    # over-read: the reference's own exception class
    short = ref.FixedSequenceSource(words[:10])
    with pytest.raises(ref.SourceExhausted):
        dev.shuffle_batched(short, list(range(1000)))


@gpu
def test_reference_exceptions(ref, dev):
    with pytest.raises(ref.BoundOverflow):
        dev.partial_shuffle_batch(ref.make_source("pcg64", 1), list(range(52)), 52, 2, 100)
    with pytest.raises(ValueError):
        dev.shuffle_batched(ref.make_source("pcg64", 1), list(range(10)),
                            ref.ShuffleSchedule(entries=((1 << 16, 2),), max_batch=2, word_bits=32))


@gpu
def test_cli_algorithms_through_the_library(ref, dev):
    """cli.ALGORITHMS (cli.py:44-49): each CPU row and its *_b200 row give the same permutation
    and leave the source at the same position; the reference's bench() times the GPU rows."""
    from paper_2408_06213_b200 import refbind

    cli = importlib.import_module("batchrand.cli")
    undo = refbind.install(ref)
    try:
        for name in ("shuffle", "naive_shuffle_2", "shuffle_2", "shuffle_6"):
            for gen in GENS:
                for n in (64, 1000, 4096):
                    s_cpu, s_gpu = ref.make_source(gen, n + 1), ref.make_source(gen, n + 1)
                    a, b = list(range(n)), list(range(n))
                    cli.ALGORITHMS[name](s_cpu, a)
                    cli.ALGORITHMS[name + "_b200"](s_gpu, b)
                    assert a == b and _same_stream(s_cpu, s_gpu), (name, gen, n)
        recs = cli.bench("pcg64", sizes=(64, 1024), algorithms=("shuffle_6", "shuffle_6_b200"), budget_ns=2_000_000)
        assert [(r.algorithm, r.n) for r in recs] == [("shuffle_6", 64), ("shuffle_6", 1024), ("shuffle_6_b200", 64),
                                                      ("shuffle_6_b200", 1024)]
    finally:
        undo()
