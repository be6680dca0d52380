"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

The oracle is a plain-C restatement of the reference's hot path
(/root/reference/pkg/src/batchrand; see oracle.c for the file:line each function
follows).  It is the checker for the CUDA product and the CPU baseline in bench.py; the
product package never imports it.  Build: ``make -C oracle`` (also done by
``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")

MASK64 = (1 << 64) - 1

# shuffle.py:56-66 DEFAULT_SCHEDULE
DEFAULT_ENTRIES = ((1 << 30, 2), (1 << 19, 3), (1 << 14, 4), (1 << 11, 5), (1 << 9, 6))

OK, E_INVALID, E_BOUND_OVERFLOW, E_EXHAUSTED = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


class Source(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("word_bits", C.c_int32),
        ("state_hi", C.c_uint64),
        ("state_lo", C.c_uint64),
        ("inc_hi", C.c_uint64),
        ("inc_lo", C.c_uint64),
        ("words", C.c_void_p),
        ("nwords", C.c_int64),
        ("cursor", C.c_int64),
        ("drawn", C.c_int64),
        ("key", C.c_uint32 * 8),
        ("nonce", C.c_uint64),
        ("counter", C.c_uint64),
        ("pos", C.c_int32),
        ("buf", C.c_uint32 * 16),
    ]

    @property
    def state(self) -> int:
        return (self.state_hi << 64) | self.state_lo

    @state.setter
    def state(self, v: int) -> None:
        self.state_hi, self.state_lo = (v >> 64) & MASK64, v & MASK64

    @property
    def increment(self) -> int:
        return (self.inc_hi << 64) | self.inc_lo

    @increment.setter
    def increment(self, v: int) -> None:
        self.inc_hi, self.inc_lo = (v >> 64) & MASK64, v & MASK64


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        u64, u32, i32, i64 = C.c_uint64, C.c_uint32, C.c_int32, C.c_int64
        vp = C.c_void_p
        sig = {
            "or_splitmix64_next": (u64, [P(u64)]),
            "or_source_pcg64": (None, [P(Source), u64]),
            "or_source_lehmer": (None, [P(Source), u64]),
            "or_source_fixed": (None, [P(Source), vp, i64, i32]),
            "or_next_word": (C.c_int, [P(Source), P(u64)]),
            "or_pcg64_advance": (None, [P(Source), u64]),
            "or_array_seed": (u64, [u64, u64]),
            "or_falling_factorial": (C.c_int, [u64, u64, i32, P(u64), P(u64)]),
            "or_threshold": (u64, [u64, u64, i32]),
            "or_roll_single": (C.c_int, [P(Source), u64, u64, P(u64), P(u64), P(i32)]),
            "or_digit_pass": (None, [u64, vp, i32, i32, vp, P(u64)]),
            "or_roll_batch": (C.c_int, [P(Source), vp, i32, i32, i32, u64, u64, vp, P(u64), P(i32), P(u64)]),
            "or_roll_batch_known_threshold": (C.c_int, [P(Source), vp, i32, i32, u64, vp, P(u64), P(u64)]),
            "or_schedule_validate": (C.c_int, [vp, vp, i32, i32, i32]),
            "or_shuffle_unbatched": (C.c_int, [P(Source), vp, i32, u64]),
            "or_shuffle_batched": (C.c_int, [P(Source), vp, i32, u64, vp, vp, i32, i32, i32]),
            "or_partial_shuffle_batch": (C.c_int, [P(Source), vp, i32, u64, u32, u64, u64, P(u64), P(u64)]),
            "or_shuffle_trace": (i64, [u64, vp, vp, i32, i32, vp, vp, i64]),
            "or_roll_batches": (C.c_int, [P(Source), vp, i32, i64, vp, vp, vp, vp]),
            "or_roll_batches_mt": (C.c_int, [P(Source), vp, i32, i64, vp, vp, vp, vp, i32]),
            "or_gen_bounds": (C.c_int, [P(Source), vp, i64, u64, u64]),
            "or_shuffle_segmented": (C.c_int, [vp, i32, i64, u64, u64, i64, vp, vp, i32, vp, i32, i32]),
            "or_shuffle_segmented_gen": (C.c_int, [vp, i32, i64, u64, u64, i64, vp, vp, i32, vp, i32, i32, i32]),
            "or_pcg64_fill": (None, [P(Source), u64, vp, i64]),
            "or_chacha_block": (None, [vp, u64, u64, vp]),
            "or_shuffle_naive_batched": (C.c_int, [P(Source), vp, i32, u64]),
            "or_roll_batch_naive": (C.c_int, [P(Source), vp, i32, vp]),
            "or_shuffle_naive_segmented": (C.c_int, [vp, i32, i64, u64, u64, i64, vp, i32, i32]),
            "or_source_chacha": (None, [P(Source), u64]),
            "or_chacha_advance": (None, [P(Source), u64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _check(code, what):
    if code:
        raise OracleError(code, what)


# ---------------------------------------------------------------- word sources
def splitmix64(seed: int, count: int) -> list[int]:
    x = C.c_uint64(seed & MASK64)
    return [lib().or_splitmix64_next(C.byref(x)) for _ in range(count)]


def pcg64(seed: int) -> Source:
    s = Source()
    lib().or_source_pcg64(C.byref(s), seed & MASK64)
    return s


def pcg64_from_state(state: int, inc: int) -> Source:
    s = pcg64(0)
    s.state, s.increment = state, inc
    return s


def lehmer(seed: int) -> Source:
    s = Source()
    lib().or_source_lehmer(C.byref(s), seed & MASK64)
    return s


def chacha(seed: int) -> Source:
    s = Source()
    lib().or_source_chacha(C.byref(s), seed & MASK64)
    return s


def chacha_block(key_words, counter: int, nonce: int) -> list[int]:
    key = np.asarray(key_words, dtype=np.uint32)
    out = np.zeros(16, dtype=np.uint32)
    lib().or_chacha_block(_ptr(key), counter & MASK64, nonce & MASK64, _ptr(out))
    return out.tolist()


def chacha_position(s: Source) -> int:
    """Absolute word position of a ChaCha source's next word (block*8 + word)."""
    return s.counter * 8 if s.pos == 16 else (s.counter - 1) * 8 + s.pos // 2





def fixed(words, bits: int = 64) -> Source:
    arr = np.ascontiguousarray(np.asarray(words, dtype=np.uint64))
    s = Source()
    lib().or_source_fixed(C.byref(s), _ptr(arr), len(arr), bits)
    s._keep = arr  # keep the buffer alive
    return s


def next_word(s: Source) -> int:
    w = C.c_uint64()
    _check(lib().or_next_word(C.byref(s), C.byref(w)), "next_word")
    return w.value


def words(s: Source, count: int) -> list[int]:
    return [next_word(s) for _ in range(count)]


def advance(s: Source, delta: int) -> None:
    if s.kind == 3:
        lib().or_chacha_advance(C.byref(s), delta & MASK64)
    else:
        lib().or_pcg64_advance(C.byref(s), delta & MASK64)


def array_seed(run_seed: int, a: int) -> int:
    return lib().or_array_seed(run_seed & MASK64, a & MASK64)


def pcg64_fill(s: Source, offset: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().or_pcg64_fill(C.byref(s), offset, _ptr(out), count)
    return out


# ---------------------------------------------------------------- bounded / batched
def falling_factorial(n: int, k: int, bits: int = 64) -> int:
    lo, hi = C.c_uint64(), C.c_uint64()
    _check(lib().or_falling_factorial(n, k, bits, C.byref(lo), C.byref(hi)), "falling_factorial")
    return (hi.value << 64) | lo.value


def threshold(b: int, bits: int = 64) -> int:
    return lib().or_threshold(b & MASK64, b >> 64, bits)


def roll_single(s: Source, b: int):
    v, w, ro = C.c_uint64(), C.c_uint64(), C.c_int32()
    _check(lib().or_roll_single(C.byref(s), b & MASK64, b >> 64, C.byref(v), C.byref(w), C.byref(ro)), "roll_single")
    return v.value, w.value, ro.value


def digit_pass(r0: int, bases, bits: int = 64):
    b = np.asarray(bases, dtype=np.uint64)
    d = np.zeros(len(b), dtype=np.uint64)
    rk = C.c_uint64()
    lib().or_digit_pass(r0, _ptr(b), len(b), bits, _ptr(d), C.byref(rk))
    return tuple(int(x) for x in d), rk.value


def roll_batch(s: Source, bases, bits: int = 64, upper_bound=None):
    b = np.asarray(bases, dtype=np.uint64)
    d = np.zeros(len(b), dtype=np.uint64)
    w, tc, rk = C.c_uint64(), C.c_int32(), C.c_uint64()
    u = upper_bound or 0
    _check(
        lib().or_roll_batch(C.byref(s), _ptr(b), len(b), bits, int(upper_bound is not None), u & MASK64, u >> 64,
                            _ptr(d), C.byref(w), C.byref(tc), C.byref(rk)),
        "roll_batch",
    )
    return tuple(int(x) for x in d), w.value, bool(tc.value), rk.value


def roll_batch_known_threshold(s: Source, bases, bits: int = 64):
    """batched.py:85-99: re-draw whole passes until r_k >= 2^bits mod product."""
    b = np.asarray(bases, dtype=np.uint64)
    prod = 1
    for x in bases:
        prod *= int(x)
    t = threshold(prod, bits) if prod < 1 << bits else 0
    d = np.zeros(len(b), dtype=np.uint64)
    w, rk = C.c_uint64(), C.c_uint64()
    _check(lib().or_roll_batch_known_threshold(C.byref(s), _ptr(b), len(b), bits, t, _ptr(d), C.byref(w),
                                               C.byref(rk)), "roll_batch_known_threshold")
    return tuple(int(x) for x in d), w.value, False, rk.value


def roll_batches_mt(s: Source, bounds: np.ndarray, k: int, nthreads: int = 0, out=None):
    """roll_batches on all host threads (chunked jump-ahead with in-order repair; same results).
    ``out=(rolls, words)`` writes into preallocated arrays and skips flags/final remainders
    (what the bulk device call returns by default)."""
    bounds = np.ascontiguousarray(bounds, dtype=np.uint32)
    nb = len(bounds) // k
    if out is not None:
        rolls, wds = out
        _check(lib().or_roll_batches_mt(C.byref(s), _ptr(bounds), k, nb, _ptr(rolls), _ptr(wds), None, None,
                                        nthreads), "roll_batches_mt")
        return rolls, wds, None, None
    rolls = np.empty(nb * k, dtype=np.uint32)
    wds = np.empty(nb, dtype=np.uint8)
    flags = np.empty(nb, dtype=np.uint8)
    rk = np.empty(nb, dtype=np.uint64)
    _check(lib().or_roll_batches_mt(C.byref(s), _ptr(bounds), k, nb, _ptr(rolls), _ptr(wds), _ptr(flags), _ptr(rk),
                                    nthreads), "roll_batches_mt")
    return rolls, wds, flags, rk


def roll_batches(s: Source, bounds: np.ndarray, k: int):
    bounds = np.ascontiguousarray(bounds, dtype=np.uint32)
    nb = len(bounds) // k
    rolls = np.empty(nb * k, dtype=np.uint32)
    wds = np.empty(nb, dtype=np.uint8)
    flags = np.empty(nb, dtype=np.uint8)
    rk = np.empty(nb, dtype=np.uint64)
    _check(lib().or_roll_batches(C.byref(s), _ptr(bounds), k, nb, _ptr(rolls), _ptr(wds), _ptr(flags), _ptr(rk)),
           "roll_batches")
    return rolls, wds, flags, rk


def gen_bounds(seed: int, count: int, lo: int = 2, span: int = (1 << 16) - 2) -> np.ndarray:
    s = pcg64(seed)
    out = np.empty(count, dtype=np.uint32)
    _check(lib().or_gen_bounds(C.byref(s), _ptr(out), count, lo, span), "gen_bounds")
    return out


# ---------------------------------------------------------------- shuffles
def _sched(entries):
    lengths = np.asarray([e[0] for e in entries], dtype=np.uint64)
    sizes = np.asarray([e[1] for e in entries], dtype=np.uint32)
    return lengths, sizes


def schedule_validate(entries, max_batch, bits=64) -> int:
    lengths, sizes = _sched(entries)
    return lib().or_schedule_validate(_ptr(lengths), _ptr(sizes), len(entries), max_batch, bits)


def _as_array(z):
    arr = np.ascontiguousarray(z)
    if arr.dtype.itemsize not in (1, 2, 4, 8, 16, 32, 64):
        raise TypeError(f"unsupported itemsize {arr.dtype.itemsize}")
    return arr


def shuffle_batched(s: Source, z, entries=DEFAULT_ENTRIES, bits=64, check_bounds=False) -> np.ndarray:
    arr = _as_array(z).copy()
    lengths, sizes = _sched(entries)
    _check(lib().or_shuffle_batched(C.byref(s), _ptr(arr), arr.dtype.itemsize, arr.size, _ptr(lengths), _ptr(sizes),
                                    len(entries), bits, int(check_bounds)), "shuffle_batched")
    return arr


def shuffle_unbatched(s: Source, z) -> np.ndarray:
    arr = _as_array(z).copy()
    _check(lib().or_shuffle_unbatched(C.byref(s), _ptr(arr), arr.dtype.itemsize, arr.size), "shuffle_unbatched")
    return arr


def partial_shuffle_batch(s: Source, z, n: int, k: int, u: int):
    arr = _as_array(z).copy()
    lo, hi = C.c_uint64(), C.c_uint64()
    _check(lib().or_partial_shuffle_batch(C.byref(s), _ptr(arr), arr.dtype.itemsize, n, k, u & MASK64, u >> 64,
                                          C.byref(lo), C.byref(hi)), "partial_shuffle_batch")
    return arr, (hi.value << 64) | lo.value


def shuffle_trace(n: int, entries=DEFAULT_ENTRIES, bits=64):
    lengths, sizes = _sched(entries)
    cnt = lib().or_shuffle_trace(n, _ptr(lengths), _ptr(sizes), len(entries), bits, None, None, 0)
    bn = np.empty(max(cnt, 1), dtype=np.uint64)
    bk = np.empty(max(cnt, 1), dtype=np.uint32)
    lib().or_shuffle_trace(n, _ptr(lengths), _ptr(sizes), len(entries), bits, _ptr(bn), _ptr(bk), cnt)
    return bn[:cnt], bk[:cnt]


def shuffle_segmented(data: np.ndarray, n: int, run_seed: int, array_index_base: int = 0,
                      entries=DEFAULT_ENTRIES, nthreads: int = 0, unbatched: bool = False, generator: str = "pcg64"):
    """Shuffle data (num_arrays*n elements, in place) like the device segmented shuffle."""
    assert data.flags.c_contiguous
    num_arrays = data.size // n
    lengths, sizes = _sched(entries)
    wds = np.empty(num_arrays, dtype=np.uint32)
    _check(lib().or_shuffle_segmented_gen(_ptr(data), data.dtype.itemsize, num_arrays, n, run_seed & MASK64,
                                          array_index_base, _ptr(lengths), _ptr(sizes), len(entries), _ptr(wds),
                                          nthreads, int(unbatched), {"pcg64": 0, "lehmer": 1, "chacha": 2}[generator]),
           "shuffle_segmented")
    return wds


# ---------------------------------------------------------------- division-based baselines
def shuffle_naive_batched(s: Source, z) -> np.ndarray:
    """shuffle.py:228-266 (in place on a copy; returns it)."""
    a = _as_array(z)
    _check(lib().or_shuffle_naive_batched(C.byref(s), _ptr(a), a.dtype.itemsize, a.size), "shuffle_naive_batched")
    return a


def roll_batch_naive(s: Source, bases) -> tuple:
    """batched.py:126-128."""
    b = np.asarray(bases, dtype=np.uint64)
    d = np.zeros(len(b), dtype=np.uint64)
    _check(lib().or_roll_batch_naive(C.byref(s), _ptr(b), len(b), _ptr(d)), "roll_batch_naive")
    return tuple(int(x) for x in d)


def shuffle_naive_segmented(data: np.ndarray, n: int, run_seed: int, array_index_base: int = 0,
                            nthreads: int = 0, generator: str = "pcg64"):
    assert data.flags.c_contiguous
    num_arrays = data.size // n
    wds = np.empty(num_arrays, dtype=np.uint32)
    _check(lib().or_shuffle_naive_segmented(_ptr(data), data.dtype.itemsize, num_arrays, n, run_seed & MASK64,
                                            array_index_base, _ptr(wds), nthreads,
                                            {"pcg64": 0, "lehmer": 1, "chacha": 2}[generator]),
           "shuffle_naive_segmented")
    return wds


GENERATOR_MAKERS = {"pcg64": pcg64, "lehmer": lehmer, "chacha": chacha}
