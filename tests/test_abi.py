"""CPU-side checks of the C-ABI library: it loads, exports every symbol the header declares,
and its host helpers (generator seeding/jump-ahead, schedule validation, plan compiler)
agree with the oracle.  No device compute is called here."""

import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def N():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2408_06213_b200 import _native

    return _native


def header_symbols():
    with open(os.path.join(ROOT, "include", "batchrand_b200.h")) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(br_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound(N):
    L = N.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
        assert s in N.PROTOTYPES, f"{s} declared in the header but not bound in _native.py"


def test_struct_layouts(N):
    assert C.sizeof(N.Pcg64State) == 32
    assert C.sizeof(N.Regime) == 16
    assert C.sizeof(N.Segment) == 24
    assert N.lib().br_abi_version() == 3


def test_host_generator_helpers_match_oracle(N, O, golden):
    L = N.lib()
    for rec in golden["pcg64"]:
        st = N.Pcg64State()
        L.br_pcg64_seed(rec["seed"], C.byref(st))
        assert (st.state_hi << 64 | st.state_lo) == rec["state"]
        assert (st.inc_hi << 64 | st.inc_lo) == rec["inc"]
        assert [L.br_pcg64_next(C.byref(st)) for _ in range(16)] == rec["words"]
    for rec in golden["array_seed"]:
        assert L.br_array_seed(rec["run_seed"], rec["a"]) == rec["seed"]
    for d in (0, 1, 31, 32, 12345, 99999, (1 << 40) + 3):
        st = N.Pcg64State()
        L.br_pcg64_seed(5, C.byref(st))
        L.br_pcg64_advance(C.byref(st), d)
        o = O.pcg64(5)
        O.advance(o, d)
        assert (st.state_hi << 64 | st.state_lo) == o.state


def _regimes(N, entries):
    arr = (N.Regime * len(entries))()
    for i, (n, k) in enumerate(entries):
        arr[i].max_length, arr[i].batch_size = n, k
    return arr


def test_plan_compiler_matches_oracle_walk(N, O, golden):
    L = N.lib()
    for name, sched in golden["schedules"].items():
        entries = [tuple(e) for e in sched["entries"]]
        regs = _regimes(N, entries)
        for n in list(range(0, 80)) + [100, 511, 512, 513, 1000, 2047, 2048, 2049, 4096, 10000, 65536, 1 << 20,
                                       (1 << 20) + 7]:
            segs = (N.Segment * 64)()
            nb = C.c_uint64()
            ns = L.br_plan_build(n, regs, len(entries), segs, 64, C.byref(nb))
            assert ns >= 0
            bn, bk = O.shuffle_trace(n, entries)
            got_n, got_k = [], []
            for i in range(ns):
                for c in range(segs[i].count):
                    got_n.append(segs[i].start_n - c * segs[i].k)
                    got_k.append(segs[i].k)
            assert got_n == bn.tolist() and got_k == bk.tolist(), (name, n)
            assert nb.value == len(bn)


def test_schedule_validation_codes(N):
    L = N.lib()
    ok = _regimes(N, [(1 << 30, 2), (1 << 19, 3), (1 << 14, 4), (1 << 11, 5), (1 << 9, 6)])
    assert L.br_schedule_validate(ok, 5, 6, 64) == N.BR_OK
    assert L.br_schedule_validate(_regimes(N, [(8, 2), (16, 3)]), 2, 3, 64) == N.BR_E_INVALID
    assert L.br_schedule_validate(_regimes(N, [(16, 3), (8, 2)]), 2, 2, 64) == N.BR_E_INVALID
    assert L.br_schedule_validate(_regimes(N, [(16, 2)]), 1, 3, 64) == N.BR_E_INVALID
    assert L.br_schedule_validate(_regimes(N, [(1 << 33, 2)]), 1, 2, 64) == N.BR_E_BOUND_OVERFLOW
    assert L.br_schedule_validate(ok, 5, 6, 16) == N.BR_E_UNSUPPORTED


def test_falling_factorial_abi(N):
    L = N.lib()
    lo, hi = C.c_uint64(), C.c_uint64()
    assert L.br_falling_factorial(1 << 19, 3, C.byref(lo), C.byref(hi)) == 0
    assert (hi.value << 64 | lo.value) == (1 << 19) * ((1 << 19) - 1) * ((1 << 19) - 2)
    assert L.br_falling_factorial((1 << 32) + 1, 2, C.byref(lo), C.byref(hi)) == N.BR_E_BOUND_OVERFLOW
    assert L.br_falling_factorial(3, 4, C.byref(lo), C.byref(hi)) == N.BR_E_INVALID


def test_python_api_validation_without_gpu():
    """Argument validation mirrors the reference before any device work is attempted."""
    import paper_2408_06213_b200 as B

    with pytest.raises(ValueError):
        B.ShuffleSchedule((), max_batch=2)
    with pytest.raises(ValueError):
        B.ShuffleSchedule(((8, 2), (16, 3)), max_batch=3)
    with pytest.raises(B.BoundOverflow):
        B.ShuffleSchedule(((1 << 33, 2),), max_batch=2)
    with pytest.raises(ValueError):
        B.default_schedule(7)
    assert B.default_schedule(2).entries == ((1 << 30, 2),)
    with pytest.raises(ValueError):
        B.RadixBases.of((0, 2))
    with pytest.raises(B.BoundOverflow):
        B.RadixBases.of((2**33, 2**32))
    spec = B.BatchSpec.with_threshold(B.RadixBases.of((2, 6), bits=4))
    assert spec.precomputed_threshold == 4
    with pytest.raises(B.UnknownGenerator):
        B.make_source("mersenne", 1)

    class Narrow:
        word_bits = 16

    with pytest.raises(ValueError):
        B.shuffle_batched(Narrow(), [1, 2, 3])  # width mismatch (shuffle.py:163-167)
    # trivial lengths consume nothing and need no device (test_shuffle.py:61-67)
    s = B.Pcg64Source(1)
    st0 = s.state
    assert B.shuffle_batched(s, []) == [] and B.shuffle_batched(s, [42]) == [42]
    assert s.state == st0


def test_host_source_matches_oracle(O):
    import paper_2408_06213_b200 as B

    s = B.Pcg64Source(42)
    o = O.pcg64(42)
    assert (s.state, s.increment) == (o.state, o.increment)
    assert [s.next_word() for _ in range(10)] == O.words(o, 10)
    assert [next(g) for g in [B.splitmix64_stream(7)] for _ in range(3)] == O.splitmix64(7, 3)


def test_host_lehmer_matches_golden(N, golden):
    import paper_2408_06213_b200 as B

    L = N.lib()
    for rec in golden["lehmer"]:
        st = N.Pcg64State()
        L.br_lehmer_seed(rec["seed"], C.byref(st))
        assert (st.state_hi << 64 | st.state_lo) == rec["state"] and st.inc_hi == st.inc_lo == 0
        assert [L.br_pcg64_next(C.byref(st)) for _ in range(8)] == rec["words"]
        s = B.make_source("lehmer", rec["seed"])
        assert [s.next_word() for _ in range(8)] == rec["words"]


def test_cli_parser_and_csv_schema():
    """The device CLI keeps the reference's CSV schema (cli.py:27) and argument surface."""
    import io

    from paper_2408_06213_b200 import cli

    assert cli.CSV_HEADER == "algorithm,generator,n,avg_ns_per_element,min_ns_per_element"
    args = cli.build_parser().parse_args(["bench", "--sizes", "64,128", "--algorithms", "shuffle_6_b200"])
    assert args.sizes == (64, 128) and args.algorithms == ("shuffle_6_b200",)
    buf = io.StringIO()
    cli.write_csv([("shuffle_6_b200", "pcg64", 64, 12.5, 11.25)], buf)
    assert buf.getvalue().splitlines() == [cli.CSV_HEADER, "shuffle_6_b200,pcg64,64,12.500,11.250"]
    with pytest.raises(SystemExit):
        cli.build_parser().parse_args(["bench", "--sizes", "1"])


def test_host_chacha_matches_golden(N, O, golden):
    import paper_2408_06213_b200 as B

    L = N.lib()
    assert C.sizeof(N.ChachaState) == 64
    for rec in golden["chacha"]:
        st = N.ChachaState()
        L.br_chacha_seed(rec["seed"], C.byref(st))
        assert list(st.key) == rec["key"] and st.inc_hi == rec["nonce"] and st.inc_lo == N.BR_CHACHA_TAG
        assert [L.br_pcg64_next(C.byref(st)) for _ in range(20)] == rec["words"]
        s = B.make_source("chacha", rec["seed"])
        assert s.key_words == tuple(rec["key"]) and s.nonce == rec["nonce"]
        assert [s.next_word() for _ in range(20)] == rec["words"]
    st = N.ChachaState()
    L.br_chacha_seed(11, C.byref(st))
    L.br_pcg64_advance(C.byref(st), 1000)
    assert L.br_pcg64_next(C.byref(st)) == O.words(O.chacha(11), 1001)[-1]
    rec = golden["chacha_block_rfc8439"]
    from paper_2408_06213_b200 import batchrand as BR

    assert BR._chacha_block_words(rec["key"], rec["nonce"], rec["counter"]) == rec["block"]


def test_chacha_position_mapping():
    from paper_2408_06213_b200 import batchrand as B

    s = B.ChaChaSource(3)
    for drawn in range(0, 20):
        assert B._chacha_position(s) == drawn
        s.next_word()
    t = B.ChaChaSource(3)
    B._chacha_set_position(t, 13)
    assert (t.counter, t._pos) == (2, 10)
    u = B.ChaChaSource(3)
    w = [u.next_word() for _ in range(20)]
    v = B.ChaChaSource(3)
    B._chacha_set_position(v, 13)
    assert [v.next_word() for _ in range(7)] == w[13:20]


def test_public_api_covers_the_reference():
    """Every public name of the reference package (batchrand/__init__.py) exists here."""
    import paper_2408_06213_b200 as B

    names = ["BatchRandError", "BatchResult", "BatchSpec", "BoundEncoding", "BoundOverflow", "ChaChaSource",
             "CostParams", "DEFAULT_SCHEDULE", "DigitOutOfRange", "FullProduct", "InsufficientTrials", "LehmerSource",
             "NoCrossover", "PAIR_SCHEDULE", "Pcg64Source", "RadixBases", "RollOutcome", "ShuffleSchedule",
             "SourceExhausted", "UnknownAlgorithm", "UnknownGenerator", "ValueOutOfRange", "WordSource",
             "build_schedule", "chacha_block", "cost_per_roll", "decode", "default_schedule", "digit_pass", "encode",
             "falling_factorial", "find_nk", "make_source", "mul_full", "partial_shuffle_batch", "roll_batch",
             "roll_batch_known_threshold", "roll_batch_naive", "roll_single", "roll_single_traced",
             "shuffle_batched", "shuffle_naive_batched", "shuffle_unbatched", "threshold", "FixedSequenceSource",
             "ExhaustiveSource"]
    assert [n for n in names if not hasattr(B, n)] == []
    rb = B.RadixBases.of((4, 3, 5))
    assert B.decode(37, rb) == (2, 1, 2) and B.encode((2, 1, 2), rb) == 37  # mixed_radix.py:40-67
    with pytest.raises(B.DigitOutOfRange):
        B.encode((4, 0, 0), rb)
    with pytest.raises(B.ValueOutOfRange):
        B.decode(60, rb)
