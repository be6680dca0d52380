"""ctypes binding of the C ABI (include/batchrand_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2408_06213_b200/csrc``).  There is no fallback: importing the drop-in API works
without a GPU, but every device call raises when the library or the device is missing.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import BoundOverflow, SourceExhausted

HERE = os.path.dirname(os.path.abspath(__file__))
# BR_LIB overrides the library path (A/B timing of two builds; tools/ only)
LIB_PATH = os.environ.get("BR_LIB") or os.path.join(HERE, "lib", "libbatchrand_b200.so")

BR_OK, BR_E_INVALID, BR_E_BOUND_OVERFLOW, BR_E_EXHAUSTED, BR_E_CUDA, BR_E_UNSUPPORTED = range(6)

u64, u32, i32, i64, vp, sz = C.c_uint64, C.c_uint32, C.c_int32, C.c_int64, C.c_void_p, C.c_size_t


class Pcg64State(C.Structure):
    _fields_ = [("state_hi", u64), ("state_lo", u64), ("inc_hi", u64), ("inc_lo", u64)]


class ChachaState(Pcg64State):
    """br_chacha: the br_pcg64 head (position, nonce, tag) followed by the 8 key words."""

    _fields_ = [("key", u32 * 8)]


BR_CHACHA_TAG = 2
BR_WORDS_TAG = 4


class Regime(C.Structure):
    _fields_ = [("max_length", u64), ("batch_size", u32), ("reserved", u32)]


class Segment(C.Structure):
    _fields_ = [("start_n", u64), ("k", u32), ("reserved", u32), ("count", u64)]


P = C.POINTER
PROTOTYPES = {
    "br_abi_version": (C.c_int, []),
    "br_last_error": (C.c_char_p, []),
    "br_last_kernel": (C.c_char_p, []),
    "br_device_count": (C.c_int, []),
    "br_splitmix64_next": (u64, [P(u64)]),
    "br_pcg64_seed": (None, [u64, P(Pcg64State)]),
    "br_lehmer_seed": (None, [u64, P(Pcg64State)]),
    "br_chacha_seed": (None, [u64, P(ChachaState)]),
    "br_words_state": (C.c_int, [vp, u64, P(ChachaState)]),
    "br_pcg64_next": (u64, [P(Pcg64State)]),
    "br_pcg64_advance": (None, [P(Pcg64State), u64]),
    "br_array_seed": (u64, [u64, u64]),
    "br_schedule_validate": (C.c_int, [P(Regime), C.c_int, u32, C.c_int]),
    "br_falling_factorial": (C.c_int, [u64, u32, P(u64), P(u64)]),
    "br_plan_build": (i64, [u64, P(Regime), C.c_int, P(Segment), i64, P(u64)]),
    "br_pcg64_fill": (C.c_int, [vp, i64, P(Pcg64State), u64, vp]),
    "br_state_upload": (C.c_int, [vp, P(Pcg64State), vp]),
    "br_state_download": (C.c_int, [P(Pcg64State), vp, vp]),
    "br_roll_workspace_bytes": (sz, []),
    "br_roll_batches": (C.c_int, [vp, C.c_int, i64, vp, vp, vp, vp, vp, vp, vp]),
    "br_roll_batches_phase": (C.c_int, [vp, C.c_int, i64, vp, vp, vp, vp, vp, vp, C.c_int, vp]),
    "br_roll_batches_naive": (C.c_int, [vp, C.c_int, i64, vp, vp, vp, vp, vp, vp, vp]),
    "br_roll_check": (C.c_int, [vp, vp, P(u64)]),
    "br_digit_pass": (C.c_int, [vp, vp, C.c_int, i64, vp, vp, vp]),
    "br_roll_batch64": (C.c_int, [vp, C.c_int, vp, vp, vp, vp]),
    "br_shuffle_stream": (C.c_int, [vp, C.c_int, u64, vp, P(Regime), C.c_int, C.c_int, vp, vp]),
    "br_shuffle_stream_segments": (C.c_int, [vp, C.c_int, u64, vp, P(Segment), C.c_int, vp, vp, vp]),
    "br_shuffle_segmented": (C.c_int, [vp, C.c_int, i64, u64, u64, i64, P(Regime), C.c_int, C.c_int, vp, vp]),
    "br_shuffle_naive_stream": (C.c_int, [vp, C.c_int, u64, vp, vp, vp]),
    "br_shuffle_naive_segmented": (C.c_int, [vp, C.c_int, i64, u64, u64, i64, C.c_int, vp, vp]),
    "br_release": (None, []),
}

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def lib():
    """Load the C-ABI library (raises NativeLibraryMissing if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            if os.environ.get("BR_LIB") and not hasattr(L, name):
                continue  # an older build under A/B test
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return (lib().br_last_error() or b"").decode()


def last_kernel() -> str:
    return (lib().br_last_kernel() or b"").decode()


def check(status: int, what: str = "") -> None:
    """Map a C-ABI status to the reference's exception types (errors.py)."""
    if status == BR_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == BR_E_INVALID:
        raise ValueError(msg)
    if status == BR_E_BOUND_OVERFLOW:
        raise BoundOverflow(msg)
    if status == BR_E_EXHAUSTED:
        raise SourceExhausted(msg)
    if status == BR_E_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"CUDA failure in {what}: {last_error()}")
