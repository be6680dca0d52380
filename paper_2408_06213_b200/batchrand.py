"""Drop-in, GPU-backed replacement for the reference ``batchrand`` hot path.

Same names, argument meaning and error behaviour as
/root/reference/pkg/src/batchrand (arXiv 2408.06213):

  * ``shuffle_batched`` / ``shuffle_unbatched`` / ``partial_shuffle_batch``  (shuffle.py:80-225)
  * ``roll_batch`` / ``roll_batch_known_threshold`` / ``digit_pass``          (batched.py:69-123)
  * ``Pcg64Source`` / ``make_source`` / ``splitmix64_stream``                 (wordsource.py)
  * ``ShuffleSchedule`` / ``DEFAULT_SCHEDULE`` / ``PAIR_SCHEDULE`` / ``default_schedule``
  * ``RadixBases`` / ``BoundEncoding`` / ``BatchSpec`` / ``BatchResult`` and the errors.

Every roll and every swap runs in the CUDA library (paper_2408_06213_b200/lib, sm_100a)
through its C ABI; the Python layer only validates arguments (exactly like the reference)
and moves state.  Sources: any PCG64 source with ``state``/``increment`` attributes (ours
or the reference's own ``Pcg64Source``) is accepted and advanced by exactly the words the
device consumed.  Other generators raise ``TypeError`` (device versions are a later row).

Bulk entry points that have no reference counterpart (the reason for a GPU):
``roll_batches`` (many batches on one stream), ``shuffle_many`` (many independent arrays,
one seed each), ``pcg64_fill`` and ``digit_pass_many``.
"""

from __future__ import annotations

import ctypes as C
import threading
import math
from dataclasses import dataclass
from typing import NamedTuple, Optional

from . import _native as N
from .errors import (
    BatchRandError,
    BoundOverflow,
    DigitOutOfRange,
    SourceExhausted,
    UnknownGenerator,
    ValueOutOfRange,
)

MASK64 = (1 << 64) - 1
PCG_MULTIPLIER = 0x2360ED051FC65DA44385DF649FCCF645


# ---------------------------------------------------------------------------- word sources
def splitmix64_stream(seed: int):
    """wordsource.py:22-35 (computed by the native library)."""
    x = C.c_uint64(seed & MASK64)
    L = N.lib()
    while True:
        yield L.br_splitmix64_next(C.byref(x))


class WordSource:
    """wordsource.py:38-48 protocol."""

    word_bits: int = 64

    def next_word(self) -> int:
        raise NotImplementedError


class Pcg64Source(WordSource):
    """PCG64 XSL-RR 128/64 (wordsource.py:71-89); state lives on the host between calls."""

    word_bits = 64

    def __init__(self, seed: int = 0):
        st = N.Pcg64State()
        N.lib().br_pcg64_seed(seed & MASK64, C.byref(st))
        self.state = (st.state_hi << 64) | st.state_lo
        self.increment = (st.inc_hi << 64) | st.inc_lo

    def next_word(self) -> int:
        st = _state_struct(self)
        w = N.lib().br_pcg64_next(C.byref(st))
        self.state = (st.state_hi << 64) | st.state_lo
        return w

    def advance(self, delta: int) -> None:
        st = _state_struct(self)
        N.lib().br_pcg64_advance(C.byref(st), delta & MASK64)
        self.state = (st.state_hi << 64) | st.state_lo


class LehmerSource(WordSource):
    """128-bit multiplicative generator, output = top 64 bits (wordsource.py:51-67).  On the
    device a Lehmer stream is a generator state with increment 0."""

    word_bits = 64

    def __init__(self, seed: int = 0):
        st = N.Pcg64State()
        N.lib().br_lehmer_seed(seed & MASK64, C.byref(st))
        self.state = (st.state_hi << 64) | st.state_lo

    def next_word(self) -> int:
        st = _state_struct(self)
        w = N.lib().br_pcg64_next(C.byref(st))
        self.state = (st.state_hi << 64) | st.state_lo
        return w


class ChaChaSource(WordSource):
    """ChaCha20 keystream consumed as 64-bit words (wordsource.py:136-164), with the
    reference's fields (key_words, nonce, counter, _buffer, _pos).  On the device a ChaCha
    stream is a position plus key and nonce (br_chacha); blocks are computed by the native
    library."""

    word_bits = 64

    def __init__(self, seed: int = 0):
        st = N.ChachaState()
        N.lib().br_chacha_seed(seed & MASK64, C.byref(st))
        self.key_words = tuple(int(k) for k in st.key)
        self.nonce = st.inc_hi
        self.counter = 0
        self._buffer = [0] * 16
        self._pos = 16  # empty; filled on first use

    def next_word(self) -> int:
        pos = self._pos
        if pos == 16:
            self._buffer = _chacha_block_words(self.key_words, self.nonce, self.counter)
            self.counter = (self.counter + 1) & MASK64
            pos = 0
        self._pos = pos + 2
        return self._buffer[pos] | (self._buffer[pos + 1] << 32)


def _chacha_block_words(key_words, nonce: int, block: int) -> list:
    """The 16 keystream u32 of one block (wordsource.py:102-133), from the native library."""
    st = N.ChachaState()
    st.state_hi, st.state_lo = block >> 61, (block << 3) & MASK64
    st.inc_hi, st.inc_lo = nonce & MASK64, N.BR_CHACHA_TAG
    for i, k in enumerate(key_words):
        st.key[i] = k
    out = []
    for _ in range(8):
        w = N.lib().br_pcg64_next(C.byref(st))
        out += [w & 0xFFFFFFFF, w >> 32]
    return out


def _is_chacha(source) -> bool:
    return all(hasattr(source, a) for a in ("key_words", "nonce", "counter", "_pos"))


def _chacha_position(source) -> int:
    """Absolute position of the next word: counter*8 with an empty buffer, else the
    buffered block (counter-1) and word _pos/2 (wordsource.py:155-164)."""
    if source._pos == 16:
        return int(source.counter) * 8
    return ((int(source.counter) - 1) & MASK64) * 8 + source._pos // 2


def _chacha_set_position(source, p: int) -> None:
    p &= (1 << 67) - 1
    blk, q = p >> 3, p & 7
    if q == 0:
        source.counter, source._pos = blk, 16
    else:
        source._buffer = _chacha_block_words(source.key_words, source.nonce, blk)
        source.counter, source._pos = (blk + 1) & MASK64, 2 * q


class FixedSequenceSource(WordSource):
    """Replays a given word sequence (wordsource.py:191-207); raises SourceExhausted on an
    over-read.  With 64-bit words the device draws from it too: the remaining words are
    copied to the device for the call and `cursor` advances by the words consumed.  A call
    that would read past the end raises SourceExhausted and leaves the payload unchanged
    (the reference would have left it partly shuffled)."""

    def __init__(self, words, bit_width: int = 64):
        self.word_bits = bit_width
        self.words = list(words)
        for w in self.words:
            if not 0 <= w < 1 << bit_width:
                raise ValueError(f"word {w} does not fit in {bit_width} bits")
        self.cursor = 0

    def next_word(self) -> int:
        if self.cursor >= len(self.words):
            raise SourceExhausted(f"sequence of {len(self.words)} words over-read")
        w = self.words[self.cursor]
        self.cursor += 1
        return w


class ExhaustiveSource(WordSource):
    """Every word of a small width once, in order (wordsource.py:167-188).  Host only: the
    device path needs 64-bit words, so device calls with it raise TypeError."""

    def __init__(self, bit_width: int):
        if not 1 <= bit_width <= 16:
            raise ValueError(f"bit_width must be in [1, 16], got {bit_width}")
        self.word_bits = bit_width
        self.cursor = 0

    @property
    def exhausted(self) -> bool:
        return self.cursor == 1 << self.word_bits

    def next_word(self) -> int:
        if self.exhausted:
            raise SourceExhausted(f"all {1 << self.word_bits} words emitted")
        self.cursor += 1
        return self.cursor - 1


def _is_fixed(source) -> bool:
    return hasattr(source, "words") and hasattr(source, "cursor") and not hasattr(source, "state")


GENERATORS = {"pcg64": Pcg64Source, "lehmer": LehmerSource, "chacha": ChaChaSource}
_GENERATOR_IDS = {"pcg64": 0, "lehmer": 1, "chacha": 2}


def make_source(name: str, seed: int = 0) -> WordSource:
    """wordsource.py:217-225.  Every named generator has a device implementation."""
    try:
        cls = GENERATORS[name]
    except KeyError:
        raise UnknownGenerator(f"unknown generator {name!r}; expected one of {sorted(GENERATORS)}") from None
    return cls(seed)


def array_seed(run_seed: int, array_index: int) -> int:
    """Per-array seed of the segmented shuffle: next(splitmix64_stream(((s<<32)|a) & MASK64))."""
    return N.lib().br_array_seed(run_seed & MASK64, array_index & MASK64)


def _is_lehmer(source) -> bool:
    return not hasattr(source, "increment") and hasattr(source, "state") and "lehmer" in type(source).__name__.lower()


def _state_struct(source) -> N.Pcg64State:
    if getattr(source, "word_bits", 64) != 64:
        raise TypeError("the device path needs 64-bit words")
    if _is_fixed(source):  # the remaining words go to the device for this call
        torch = _torch()
        rest = [w - (1 << 64) if w >= 1 << 63 else w for w in source.words[source.cursor:]]
        dev = torch.tensor(rest if rest else [0], dtype=torch.int64, device="cuda")
        st = N.ChachaState()
        N.check(N.lib().br_words_state(_ptr(dev), len(rest), C.byref(st)), "words state")
        st._keep = dev  # the device words live as long as the state that points at them
        return st
    if _is_chacha(source):
        st = N.ChachaState()
        p = _chacha_position(source)
        st.state_hi, st.state_lo = p >> 64, p & MASK64
        st.inc_hi, st.inc_lo = int(source.nonce) & MASK64, N.BR_CHACHA_TAG
        for i, k in enumerate(source.key_words):
            st.key[i] = int(k)
        return st
    try:
        if _is_lehmer(source):  # reference LehmerSource or ours: state only, increment 0
            state, inc = int(source.state), 0
        else:
            state, inc = int(source.state), int(source.increment)
    except AttributeError:
        raise TypeError(
            f"{type(source).__name__} is not a PCG64, Lehmer or ChaCha source; the device path draws those words only"
        ) from None
    st = N.Pcg64State()
    st.state_hi, st.state_lo = (state >> 64) & MASK64, state & MASK64
    st.inc_hi, st.inc_lo = (inc >> 64) & MASK64, inc & MASK64
    return st


# ---------------------------------------------------------------------------- bounded.py
class FullProduct(NamedTuple):
    hi: int
    lo: int


def mul_full(a: int, b: int, bits: int = 64) -> FullProduct:
    """bounded.py:29-32 (host helper)."""
    p = a * b
    return FullProduct(p >> bits, p & ((1 << bits) - 1))


@dataclass(frozen=True)
class BoundEncoding:
    """bounded.py:35-56."""

    raw: int
    is_full_range: bool
    bits: int

    @classmethod
    def of(cls, bound: int, bits: int = 64) -> "BoundEncoding":
        if not 1 <= bound <= 1 << bits:
            raise BoundOverflow(f"bound {bound} not in [1, 2**{bits}]")
        full = bound == 1 << bits
        return cls(0 if full else bound, full, bits)

    @property
    def value(self) -> int:
        return (1 << self.bits) if self.is_full_range else self.raw


def threshold(bound: BoundEncoding) -> int:
    """bounded.py:59-62: 2**bits mod b."""
    neg = (-bound.raw) & ((1 << bound.bits) - 1)
    return neg % bound.value


class RollOutcome(NamedTuple):
    """bounded.py:65-70."""

    value: int
    words_consumed: int
    remainder_ops: int


def roll_single_traced(source, bound) -> RollOutcome:
    """bounded.py:73-99 on the device: a single Lemire roll is a k=1 batch (same acceptance
    rule, lo >= 2^64 mod b); remainder_ops = 1 iff the first low word fell below b."""
    if isinstance(bound, BoundEncoding):
        bits, b = bound.bits, bound.value
    else:
        bits, b = getattr(source, "word_bits", 64), bound
        if not 1 <= b <= 1 << bits:
            raise BoundOverflow(f"bound {b} not in [1, 2**{bits}]")
    if bits != 64:
        raise TypeError("the device path needs 64-bit words")
    r = _roll_one(source, BatchSpec(RadixBases.of((b,), 64)))
    return RollOutcome(r.digits[0], r.words_consumed, int(r.threshold_computed))


def roll_single(source, bound) -> int:
    """bounded.py:102-104."""
    return roll_single_traced(source, bound).value


def falling_factorial(n: int, k: int, bits: int = 64) -> int:
    """bounded.py:107-119."""
    if k < 0 or k > n:
        raise ValueError(f"need 0 <= k <= n, got n={n} k={k}")
    limit = 1 << bits
    out = 1
    for factor in range(n, n - k, -1):
        out *= factor
        if out > limit:
            raise BoundOverflow(f"falling factorial of {n} over {k} terms exceeds 2**{bits}")
    return out


# ---------------------------------------------------------------------------- mixed_radix.py
@dataclass(frozen=True)
class RadixBases:
    """mixed_radix.py:18-37."""

    bases: tuple
    bits: int
    product: BoundEncoding

    @classmethod
    def of(cls, bases, bits: int = 64) -> "RadixBases":
        bases = tuple(bases)
        if not bases:
            raise ValueError("at least one base is required")
        if any(b < 1 for b in bases):
            raise ValueError(f"bases must be positive, got {bases}")
        return cls(bases, bits, BoundEncoding.of(math.prod(bases), bits))

    def __len__(self) -> int:
        return len(self.bases)


def encode(digits, bases: RadixBases) -> int:
    """mixed_radix.py:40-51: the value of a digit tuple, most significant digit first
    (host arithmetic; the device produces digits, this is the inverse view)."""
    if len(digits) != len(bases.bases):
        raise DigitOutOfRange(f"expected {len(bases.bases)} digits, got {len(digits)}")
    acc = 0
    for base, digit in zip(bases.bases, digits):
        if digit < 0 or digit >= base:
            raise DigitOutOfRange(f"digit {digit} not in [0, {base})")
        acc = acc * base + digit
    return acc


def decode(value: int, bases: RadixBases) -> tuple:
    """mixed_radix.py:54-67: the digit tuple of value < prod(bases) (host arithmetic)."""
    if value < 0 or value >= bases.product.value:
        raise ValueOutOfRange(f"value {value} not in [0, {bases.product.value})")
    out = [0] * len(bases.bases)
    for pos in range(len(bases.bases) - 1, -1, -1):
        value, out[pos] = divmod(value, bases.bases[pos])
    return tuple(out)


def chacha_block(key_words, counter: int, nonce: int) -> list:
    """wordsource.py:102-133: one 16-word ChaCha20 block (64-bit counter and nonce), computed
    by the native library's block function."""
    return _chacha_block_words(tuple(key_words), nonce, counter & MASK64)


# ---------------------------------------------------------------------------- batched.py
@dataclass(frozen=True)
class BatchSpec:
    """batched.py:26-51."""

    bases: RadixBases
    precomputed_threshold: Optional[int] = None
    upper_bound: Optional[int] = None

    def __post_init__(self):
        if self.precomputed_threshold is not None:
            expected = threshold(self.bases.product)
            if self.precomputed_threshold != expected:
                raise ValueError(
                    f"threshold {self.precomputed_threshold} does not match {expected} for bases {self.bases.bases}"
                )
        if self.upper_bound is not None and self.upper_bound < self.bases.product.value:
            raise BoundOverflow(f"upper bound {self.upper_bound} below product {self.bases.product.value}")

    @classmethod
    def with_threshold(cls, bases: RadixBases) -> "BatchSpec":
        return cls(bases, precomputed_threshold=threshold(bases.product))


@dataclass(frozen=True)
class BatchResult:
    """batched.py:54-66."""

    digits: tuple
    words_consumed: int
    threshold_computed: bool
    final_remainder: int


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the batchrand B200 path has no CPU fallback")
    return torch


def _stream_ptr(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(None)


def _device_bases(bases, torch):
    import numpy as np

    if any(b >= 1 << 32 for b in bases):
        raise NotImplementedError("device batches take bounds below 2**32")
    host = np.asarray([int(b) for b in bases], dtype=np.uint32).view(np.int32)
    return torch.from_numpy(host).cuda()


def _wide64(torch, values):
    """u64 values (2^64 encoded as 0) as an int64 CUDA tensor."""
    vals = [v & MASK64 for v in values]
    return torch.tensor([v - (1 << 64) if v >= 1 << 63 else v for v in vals], dtype=torch.int64, device="cuda")


def _roll_one64(source, bases) -> BatchResult:
    """One batch with a base of 2^32 or more: br_roll_batch64 (one device thread, 64-bit
    bases; a base of 2^64 travels as 0, the full range)."""
    torch = _torch()
    st = _state_struct(source)
    dstream = DeviceStream.from_struct(st)
    b = _wide64(torch, bases)
    out = torch.empty(len(bases) + 3, dtype=torch.int64, device="cuda")
    N.check(N.lib().br_roll_batch64(_ptr(b), len(bases), _ptr(dstream.state), None, _ptr(out), _stream_ptr(torch)),
            "roll_batch")
    dstream.write_back(source)
    v = [int(x) & MASK64 for x in out.cpu().tolist()]
    k = len(bases)
    return BatchResult(tuple(v[:k]), v[k], bool(v[k + 1]), v[k + 2])


def _roll_one(source, spec: BatchSpec) -> BatchResult:
    torch = _torch()
    bases = spec.bases.bases
    if spec.bases.bits != 64:
        raise TypeError("the device path needs 64-bit words")
    # bases of 2^32 or more, or more than the bulk kernels' 8 dice: the 64-bit single-batch kernel
    if len(bases) > 8 or any(b >= 1 << 32 for b in bases):
        return _roll_one64(source, bases)
    st = _state_struct(source)
    dstream = DeviceStream.from_struct(st)
    b = _device_bases(bases, torch)
    r = roll_batches(dstream, b, len(bases), flags=True, final_remainder=True, check=False)
    # exact words consumed: 1 + the rejections the fixup counted (the per-batch u8 saturates)
    extra = C.c_uint64()
    N.check(N.lib().br_roll_check(_ptr(dstream.workspace), _stream_ptr(torch), C.byref(extra)), "roll_batch")
    dstream.write_back(source)
    digits = tuple(int(x) & 0xFFFFFFFF for x in r.rolls.cpu().tolist())
    return BatchResult(digits, 1 + int(extra.value), bool(int(r.flags[0])), int(r.final_remainder[0]) & MASK64)


def digit_pass(r0: int, bases: RadixBases):
    """batched.py:69-82 on the device (one word)."""
    torch = _torch()
    if bases.bits != 64:
        raise TypeError("the device path needs 64-bit words")
    if any(b >= 1 << 32 for b in bases.bases):
        k = len(bases.bases)
        out = torch.empty(k + 3, dtype=torch.int64, device="cuda")
        b, w = _wide64(torch, bases.bases), _wide64(torch, [r0])  # alive until the result is read
        N.check(N.lib().br_roll_batch64(_ptr(b), k, None, _ptr(w), _ptr(out), _stream_ptr(torch)), "digit_pass")
        v = [int(x) & MASK64 for x in out.cpu().tolist()]
        return tuple(v[:k]), v[k + 2]
    w = torch.tensor([r0 - (1 << 64) if r0 >= 1 << 63 else r0], dtype=torch.int64).cuda()
    d, rk = digit_pass_many(w, _device_bases(bases.bases, torch), len(bases.bases))
    return tuple(int(x) & 0xFFFFFFFF for x in d.cpu().tolist()), int(rk[0]) & MASK64


def roll_batch_naive(source, bases: RadixBases) -> tuple:
    """batched.py:126-128: one uniform draw on the product, decoded by division (device)."""
    torch = _torch()
    if bases.bits != 64:
        raise TypeError("the device path needs 64-bit words")
    st = _state_struct(source)
    dstream = DeviceStream.from_struct(st)
    r = roll_batches(dstream, _device_bases(bases.bases, torch), len(bases.bases), naive=True)
    dstream.write_back(source)
    return tuple(int(x) & 0xFFFFFFFF for x in r.rolls.cpu().tolist())


def roll_batch_known_threshold(source, spec: BatchSpec) -> BatchResult:
    """batched.py:85-99."""
    if spec.precomputed_threshold is None:
        raise ValueError("spec has no precomputed threshold")
    r = _roll_one(source, spec)
    return BatchResult(r.digits, r.words_consumed, False, r.final_remainder)


def roll_batch(source, spec: BatchSpec) -> BatchResult:
    """batched.py:102-123 (threshold_computed == final remainder of the first word < product)."""
    return _roll_one(source, spec)


# ---------------------------------------------------------------------------- shuffle.py
@dataclass(frozen=True)
class ShuffleSchedule:
    """shuffle.py:22-49."""

    entries: tuple
    max_batch: int
    word_bits: int = 64

    def __post_init__(self):
        if not self.entries:
            raise ValueError("schedule needs at least one regime")
        lengths = [n for n, _ in self.entries]
        sizes = [k for _, k in self.entries]
        if any(a <= b for a, b in zip(lengths, lengths[1:])):
            raise ValueError(f"regime lengths must strictly decrease: {lengths}")
        if any(a >= b for a, b in zip(sizes, sizes[1:])):
            raise ValueError(f"batch sizes must strictly increase: {sizes}")
        if sizes[-1] != self.max_batch:
            raise ValueError(f"last batch size {sizes[-1]} != max_batch {self.max_batch}")
        for n, k in self.entries:
            if k > n:
                raise ValueError(f"batch size {k} exceeds regime length {n}")
            falling_factorial(n, k, self.word_bits)

    def _regimes(self):
        arr = (N.Regime * len(self.entries))()
        for i, (n, k) in enumerate(self.entries):
            arr[i].max_length = min(n, MASK64)
            arr[i].batch_size = k
        return arr


DEFAULT_SCHEDULE = ShuffleSchedule(
    entries=((1 << 30, 2), (1 << 19, 3), (1 << 14, 4), (1 << 11, 5), (1 << 9, 6)), max_batch=6, word_bits=64
)
PAIR_SCHEDULE = ShuffleSchedule(entries=((1 << 30, 2),), max_batch=2, word_bits=64)


def default_schedule(max_batch: int = 6) -> ShuffleSchedule:
    """shuffle.py:71-77."""
    if not 2 <= max_batch <= DEFAULT_SCHEDULE.max_batch:
        raise ValueError(f"max_batch must be in [2, {DEFAULT_SCHEDULE.max_batch}]")
    return ShuffleSchedule(DEFAULT_SCHEDULE.entries[: max_batch - 1], max_batch, DEFAULT_SCHEDULE.word_bits)


def _device_payload(z, torch):
    """(device tensor, finisher) for z: tensors/ndarrays of 4/8-byte items are shuffled in
    place; anything else is shuffled as an index vector and permuted on the way back."""
    import numpy as np

    if isinstance(z, torch.Tensor) and z.element_size() in (4, 8):
        if z.is_cuda and z.is_contiguous():
            return z.view(-1), lambda d: z
        dev = z.contiguous().view(-1).cuda()

        def fin(d):
            z.copy_(d.view(z.shape).to(z.device))
            return z

        return dev, fin
    if isinstance(z, np.ndarray) and z.dtype.itemsize in (4, 8):
        host = np.ascontiguousarray(z).reshape(-1)
        dev = torch.from_numpy(host.view(np.int32 if z.dtype.itemsize == 4 else np.int64)).cuda()

        def fin(d):
            out = d.cpu().numpy().view(z.dtype).reshape(z.shape)
            z[...] = out
            return z

        return dev, fin
    n = len(z)
    idx = torch.arange(n, dtype=torch.int32 if n < 1 << 31 else torch.int64, device="cuda")

    def fin(d):
        perm = d.cpu().tolist()
        vals = list(z)
        for i, p in enumerate(perm):
            z[i] = vals[p]
        return z

    return idx, fin


_TLS = threading.local()


def _call_scratch(torch):
    """Per-thread, per-device 16-word device scratch (state, words, rk) reused by the
    single-array calls; every such call ends with a synchronising state download, so the
    scratch is free again when the next call on this thread starts."""
    dev = torch.cuda.current_device()
    cache = getattr(_TLS, "scratch", None)
    if cache is None:
        cache = _TLS.scratch = {}
    t = cache.get(dev)
    if t is None:
        t = cache[dev] = torch.zeros(16, dtype=torch.int64, device="cuda")
    return t


def _host_array(z, torch):
    """A contiguous numpy view of a host array of 4/8-byte items (ndarray or CPU tensor), with
    a finisher that writes results back; None for device tensors and other containers."""
    import numpy as np

    if isinstance(z, np.ndarray) and z.dtype.itemsize in (4, 8):
        if z.flags.c_contiguous:
            return z.reshape(-1), lambda a: z
        a = np.ascontiguousarray(z).reshape(-1)

        def fin(b):
            z[...] = b.reshape(z.shape)
            return z

        return a, fin
    if isinstance(z, torch.Tensor) and not z.is_cuda and z.element_size() in (4, 8):
        t = z.contiguous()
        a = t.view(-1).numpy()
        if t.data_ptr() == z.data_ptr():
            return a, lambda b: z

        def fin(b):
            z.copy_(torch.from_numpy(b).view(z.shape))
            return z

        return a, fin
    return None


# one pinned host buffer and one device buffer per thread and device for the single-array
# calls on host arrays: [state (64 B) | words (8 B) | rk (8 B) | ... | payload from byte 128]
_STAGE_HDR = 128
_STAGE_MAX = 64 << 20  # larger host arrays take the unstaged path (no pinned buffer kept for them)


def _stage_buffers(torch, nbytes):
    dev = torch.cuda.current_device()
    cache = getattr(_TLS, "stage", None)
    if cache is None:
        cache = _TLS.stage = {}
    hb, db = cache.get(dev, (None, None))
    if hb is None or hb.numel() < nbytes:
        size = max(nbytes, 1 << 16)
        hb = torch.empty(size, dtype=torch.uint8).pin_memory()
        db = torch.empty(size, dtype=torch.uint8, device="cuda")
        cache[dev] = (hb, db)
    return hb, db


def _shuffle_stream_host(source, arr, fin, regimes, unbatched, segments, want_rk, naive, torch):
    """_shuffle_stream for a host array: state and payload go up in one copy and come back in
    one copy through pinned staging, with one stream synchronisation per call."""
    import numpy as np

    st = _state_struct(source)
    n = arr.size
    nbytes = _STAGE_HDR + arr.nbytes
    hb, db = _stage_buffers(torch, nbytes)
    hnp = hb.numpy()
    C.memmove(hnp.ctypes.data, C.addressof(st), C.sizeof(st))
    hnp[_STAGE_HDR:nbytes] = arr.view(np.uint8)
    db[:nbytes].copy_(hb[:nbytes], non_blocking=True)
    base = db.data_ptr()
    sp = _stream_ptr(torch)
    dz, dstate, dwords, drk = (C.c_void_p(base + _STAGE_HDR), C.c_void_p(base), C.c_void_p(base + 64),
                               C.c_void_p(base + 72))
    L = N.lib()
    if naive:
        N.check(L.br_shuffle_naive_stream(dz, arr.itemsize, n, dstate, dwords, sp), "shuffle")
    elif segments is None:
        regs = regimes if regimes is not None else (N.Regime * 1)()
        nreg = len(regimes) if regimes is not None else 0
        N.check(L.br_shuffle_stream(dz, arr.itemsize, n, dstate, regs, nreg, int(unbatched), dwords, sp), "shuffle")
    else:
        segs = (N.Segment * len(segments))()
        for i, (sn, k, cnt) in enumerate(segments):
            segs[i].start_n, segs[i].k, segs[i].count = sn, k, cnt
        N.check(L.br_shuffle_stream_segments(dz, arr.itemsize, n, dstate, segs, len(segments), dwords,
                                             drk if want_rk else None, sp), "shuffle")
    hb[:nbytes].copy_(db[:nbytes], non_blocking=True)
    torch.cuda.current_stream().synchronize()
    _apply_state(source, N.Pcg64State.from_buffer_copy(bytes(hnp[:C.sizeof(N.Pcg64State)])))
    arr[...] = hnp[_STAGE_HDR:nbytes].view(arr.dtype)
    out = fin(arr)
    if want_rk:
        return out, int(hnp[72:80].view(np.uint64)[0])
    return out


def _shuffle_stream(source, z, regimes, unbatched: bool, segments=None, want_rk=False, naive=False):
    torch = _torch()
    host = _host_array(z, torch)
    if host is not None and host[0].nbytes <= _STAGE_MAX:
        return _shuffle_stream_host(source, host[0], host[1], regimes, unbatched, segments, want_rk, naive, torch)
    st = _state_struct(source)
    dev, fin = _device_payload(z, torch)
    if _is_fixed(source) and dev.data_ptr() == getattr(z, "data_ptr", lambda: 0)():
        # a replayed sequence can be over-read: shuffle a copy of the caller's CUDA tensor and
        # copy back only on success, so SourceExhausted leaves the payload unchanged
        target, dev = dev, dev.clone()
        fin0 = fin

        def fin(d):
            target.copy_(d)
            return fin0(target)

    n = dev.numel()
    scratch = _call_scratch(torch)
    ds = DeviceStream.__new__(DeviceStream)
    ds._init(st, scratch[0:8])
    words = scratch[8:9]
    rk = scratch[9:10] if want_rk else None
    L = N.lib()
    if naive:
        N.check(L.br_shuffle_naive_stream(_ptr(dev), dev.element_size(), n, _ptr(ds.state), _ptr(words),
                                          _stream_ptr(torch)), "shuffle")
    elif segments is None:
        regs = regimes if regimes is not None else (N.Regime * 1)()
        nreg = len(regimes) if regimes is not None else 0
        N.check(L.br_shuffle_stream(_ptr(dev), dev.element_size(), n, _ptr(ds.state), regs, nreg, int(unbatched),
                                    _ptr(words), _stream_ptr(torch)), "shuffle")
    else:
        segs = (N.Segment * len(segments))()
        for i, (sn, k, cnt) in enumerate(segments):
            segs[i].start_n, segs[i].k, segs[i].count = sn, k, cnt
        N.check(L.br_shuffle_stream_segments(_ptr(dev), dev.element_size(), n, _ptr(ds.state), segs, len(segments),
                                             _ptr(words), _ptr(rk), _stream_ptr(torch)), "shuffle")
    ds.write_back(source)
    out = fin(dev)
    if want_rk:
        return out, int(rk.item()) & MASK64
    return out


def shuffle_batched(source, z, schedule: ShuffleSchedule = DEFAULT_SCHEDULE, check_bounds: bool = False):
    """shuffle.py:149-225 on the device.  z is permuted in place and returned.

    ``check_bounds`` is the reference's testing hook; the device plan uses exact per-batch
    thresholds, so there is no carried bound to re-validate and behaviour is identical.
    """
    if getattr(source, "word_bits", 64) != schedule.word_bits:
        raise ValueError(
            f"source emits {getattr(source, 'word_bits', 64)}-bit words but schedule expects {schedule.word_bits}"
        )
    if len(z) < 2:
        return z
    return _shuffle_stream(source, z, schedule._regimes(), False)


def shuffle_unbatched(source, z):
    """shuffle.py:80-97 on the device."""
    if len(z) < 2:
        return z
    return _shuffle_stream(source, z, None, True)


def shuffle_naive_batched(source, z):
    """shuffle.py:228-266 on the device: pairs (i, i-1) from one draw on (i+1)*i split by
    division, a single roll on 2 for a leftover index 1.  The division-based baseline."""
    bits = getattr(source, "word_bits", 64)
    i = len(z) - 1
    if i >= 2 and (i + 1) * i > 1 << bits:
        raise BoundOverflow(f"pair product {(i + 1) * i} exceeds 2**{bits}")
    if len(z) < 2:
        return z
    return _shuffle_stream(source, z, None, False, naive=True)


def partial_shuffle_batch(source, z, n: int, k: int, u: int) -> int:
    """shuffle.py:137-146: one batch of k dice on the first n elements; returns the bound
    to carry (u unchanged unless the first word's remainder fell below it)."""
    if not 1 <= k <= n or n > len(z):
        raise ValueError(f"need 1 <= k <= n <= len(z), got n={n} k={k}")
    ff = falling_factorial(n, k, getattr(source, "word_bits", 64))
    if u < ff:
        raise BoundOverflow(f"upper bound {u} below product {ff}")
    _, rk = _shuffle_stream(source, z, None, False, segments=[(n, k, 1)], want_rk=True)
    return ff if rk < u else u


# ---------------------------------------------------------------------------- bulk device API
class DeviceStream:
    """A PCG64 stream whose state lives in device memory, for chained bulk calls without a
    host round trip.  ``write_back(source)`` copies the advanced state to a host source."""

    def __init__(self, seed: int = 0, generator: str = "pcg64"):
        st = N.Pcg64State()
        if generator == "lehmer":
            N.lib().br_lehmer_seed(seed & MASK64, C.byref(st))
        elif generator == "pcg64":
            N.lib().br_pcg64_seed(seed & MASK64, C.byref(st))
        elif generator == "chacha":
            st = N.ChachaState()
            N.lib().br_chacha_seed(seed & MASK64, C.byref(st))
        else:
            raise UnknownGenerator(f"no device generator {generator!r}")
        self._init(st)

    @classmethod
    def from_source(cls, source) -> "DeviceStream":
        return cls.from_struct(_state_struct(source))

    @classmethod
    def from_struct(cls, st: N.Pcg64State) -> "DeviceStream":
        self = cls.__new__(cls)
        self._init(st)
        return self

    def _init(self, st, state=None):
        torch = _torch()
        self._keep = getattr(st, "_keep", None)  # device words of a replayed sequence
        # 8 words: a br_pcg64 head, then the ChaCha key (unused by PCG64 / Lehmer)
        self.state = torch.empty(8, dtype=torch.int64, device="cuda") if state is None else state
        self._workspace = None
        N.check(N.lib().br_state_upload(_ptr(self.state), C.byref(st), _stream_ptr(torch)), "state upload")

    @property
    def workspace(self):
        """Roll-kernel workspace (rejection bookkeeping), allocated on first bulk roll."""
        if self._workspace is None:
            torch = _torch()
            self._workspace = torch.zeros(N.lib().br_roll_workspace_bytes(), dtype=torch.uint8, device="cuda")
        return self._workspace

    def host_state(self) -> N.Pcg64State:
        torch = _torch()
        st = N.Pcg64State()
        N.check(N.lib().br_state_download(C.byref(st), _ptr(self.state), _stream_ptr(torch)), "state download")
        return st

    def write_back(self, source) -> None:
        _apply_state(source, self.host_state())


def _apply_state(source, st) -> None:
    """Advance the host source to the device state st (a br_pcg64 head)."""
    if _is_fixed(source):
        used = (st.state_hi << 64) | st.state_lo
        avail = len(source.words) - source.cursor
        if used > avail:
            source.cursor = len(source.words)
            raise SourceExhausted(f"sequence of {len(source.words)} words over-read")
        source.cursor += used
    elif _is_chacha(source):
        _chacha_set_position(source, (st.state_hi << 64) | st.state_lo)
    else:
        source.state = (st.state_hi << 64) | st.state_lo


class RollBatchesResult(NamedTuple):
    rolls: object
    words: object
    flags: object
    final_remainder: object


def roll_batches(stream, bounds, k: Optional[int] = None, *, flags: bool = False, final_remainder: bool = False,
                 out=None, check: bool = True, chunks: int = 16, naive: bool = False) -> RollBatchesResult:
    """Bulk roll_batch: batch i rolls the k dice bounds[i*k:(i+1)*k] (4-byte items, >= 1)
    from the PCG64 ``stream`` (a DeviceStream or a host PCG64 source, advanced in place).

    Device ``bounds`` give device results: rolls (int32 view of u32, len nb*k), words
    (uint8, len nb) and optionally flags (threshold_computed) and final_remainder (int64
    view of u64).  Host ``bounds`` (CPU tensor / ndarray, ideally pinned) give host results;
    the copies are pipelined in ``chunks`` pieces over two copy streams so host-to-device,
    rolling and device-to-host overlap.  ``check`` synchronises and raises ValueError /
    BoundOverflow like RadixBases.of.  ``naive`` takes the digits by division of one draw
    on the product (roll_batch_naive, batched.py:126-128) -- identical results, the
    division-based baseline."""
    torch = _torch()
    host_source = None
    if not isinstance(stream, DeviceStream):
        host_source = stream
        stream = DeviceStream.from_source(stream)
    if hasattr(bounds, "dim") and bounds.dim() == 2:
        k = bounds.shape[1] if k is None else k
    elif hasattr(bounds, "ndim") and bounds.ndim == 2:
        k = bounds.shape[1] if k is None else k
    if k is None:
        raise ValueError("k is required for flat bounds")
    if not (hasattr(bounds, "is_cuda") and bounds.is_cuda):
        res = _roll_batches_host(stream, bounds, k, flags, final_remainder, out, chunks, torch, naive)
    else:
        res = _roll_batches_dev(stream, bounds.reshape(-1), k, flags, final_remainder, out, torch, naive)
    if check:
        extra = C.c_uint64()
        N.check(N.lib().br_roll_check(_ptr(stream.workspace), _stream_ptr(torch), C.byref(extra)), "roll_batches")
    if host_source is not None:
        stream.write_back(host_source)
    return res


def _roll_fn(naive: bool):
    return N.lib().br_roll_batches_naive if naive else N.lib().br_roll_batches


def _roll_batches_dev(stream, b, k, flags, final_remainder, out, torch, naive=False):
    if b.element_size() != 4 or not b.is_contiguous():
        raise TypeError("bounds must be a contiguous tensor of 4-byte items")
    nb = b.numel() // k
    if out is None:
        rolls = torch.empty(nb * k, dtype=torch.int32, device="cuda")
        words = torch.empty(nb, dtype=torch.uint8, device="cuda")
    else:
        rolls, words = out[0], out[1]
    fl = torch.empty(nb, dtype=torch.uint8, device="cuda") if flags else None
    rk = torch.empty(nb, dtype=torch.int64, device="cuda") if final_remainder else None
    N.check(_roll_fn(naive)(_ptr(b), k, nb, _ptr(stream.state), _ptr(rolls), _ptr(words), _ptr(fl), _ptr(rk),
                            _ptr(stream.workspace), _stream_ptr(torch)), "roll_batches")
    return RollBatchesResult(rolls, words, fl, rk)


def _roll_batches_host(stream, bounds, k, flags, final_remainder, out, chunks, torch, naive=False):
    import numpy as np

    if isinstance(bounds, np.ndarray):
        bounds = torch.from_numpy(np.ascontiguousarray(bounds).view(np.int32))
    b = bounds.reshape(-1)
    if b.element_size() != 4:
        raise TypeError("bounds must have 4-byte items")
    nb = b.numel() // k
    pin = b.is_pinned()
    if out is None:
        rolls = torch.empty(nb * k, dtype=torch.int32, pin_memory=pin)
        words = torch.empty(nb, dtype=torch.uint8, pin_memory=pin)
    else:
        rolls, words = out[0], out[1]
    fl = torch.empty(nb, dtype=torch.uint8, pin_memory=pin) if flags else None
    rk = torch.empty(nb, dtype=torch.int64, pin_memory=pin) if final_remainder else None
    chunks = max(1, min(chunks, nb))
    per = -(-nb // chunks)
    per = (per + 3) & ~3
    comp = torch.cuda.current_stream()
    h2d, d2h = _copy_streams(torch)
    # the device buffers below may reuse memory the previous call's kernels (comp) were still
    # reading or writing when it returned: the copy streams start after that work
    h2d.wait_stream(comp)
    d2h.wait_stream(comp)
    dbufs = [torch.empty(per * k, dtype=torch.int32, device="cuda") for _ in range(2)]
    dro = [torch.empty(per * k, dtype=torch.int32, device="cuda") for _ in range(2)]
    dwo = [torch.empty(per, dtype=torch.uint8, device="cuda") for _ in range(2)]
    dfl = [torch.empty(per, dtype=torch.uint8, device="cuda") if flags else None for _ in range(2)]
    drk = [torch.empty(per, dtype=torch.int64, device="cuda") if final_remainder else None for _ in range(2)]
    freed = [None, None]
    L = N.lib()
    for c, lo in enumerate(range(0, nb, per)):
        hi = min(nb, lo + per)
        cnt = hi - lo
        slot = c & 1
        with torch.cuda.stream(h2d):
            if freed[slot] is not None:
                h2d.wait_event(freed[slot])
            dbufs[slot][: cnt * k].copy_(b[lo * k: hi * k], non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(h2d)
        comp.wait_event(ready)
        N.check(_roll_fn(naive)(_ptr(dbufs[slot]), k, cnt, _ptr(stream.state), _ptr(dro[slot]), _ptr(dwo[slot]),
                                _ptr(dfl[slot]), _ptr(drk[slot]), _ptr(stream.workspace),
                                C.c_void_p(comp.cuda_stream)), "roll_batches")
        done = torch.cuda.Event()
        done.record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(done)
            rolls[lo * k: hi * k].copy_(dro[slot][: cnt * k], non_blocking=True)
            words[lo:hi].copy_(dwo[slot][:cnt], non_blocking=True)
            if flags:
                fl[lo:hi].copy_(dfl[slot][:cnt], non_blocking=True)
            if final_remainder:
                rk[lo:hi].copy_(drk[slot][:cnt], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(d2h)
            freed[slot] = ev
    comp.wait_stream(d2h)
    comp.wait_stream(h2d)
    # freed device buffers are reused only after the copy streams are done with them
    for t in dbufs + dro + dwo + dfl + drk:
        if t is not None:
            t.record_stream(h2d)
            t.record_stream(d2h)
    return RollBatchesResult(rolls, words, fl, rk)


_COPY_STREAMS = {}


def _copy_streams(torch):
    dev = torch.cuda.current_device()
    if dev not in _COPY_STREAMS:
        _COPY_STREAMS[dev] = (torch.cuda.Stream(), torch.cuda.Stream())
    return _COPY_STREAMS[dev]


def digit_pass_many(words, bounds, k: int):
    """Device digit_pass for word i with bases bounds[i*k:(i+1)*k]; returns (digits, rk)."""
    torch = _torch()
    n = words.numel()
    digits = torch.empty(n * k, dtype=torch.int32, device="cuda")
    rk = torch.empty(n, dtype=torch.int64, device="cuda")
    N.check(N.lib().br_digit_pass(_ptr(words), _ptr(bounds), k, n, _ptr(digits), _ptr(rk), _stream_ptr(torch)),
            "digit_pass")
    return digits, rk


def pcg64_fill(source_or_seed, count: int, offset: int = 0, generator: str = "pcg64"):
    """count consecutive words (from word `offset`) of a PCG64, Lehmer or ChaCha stream, as an
    int64 CUDA tensor (bit pattern of the u64 words).  The source is not advanced."""
    torch = _torch()
    if isinstance(source_or_seed, int):
        st = N.Pcg64State()
        if generator == "lehmer":
            N.lib().br_lehmer_seed(source_or_seed & MASK64, C.byref(st))
        elif generator == "chacha":
            st = N.ChachaState()
            N.lib().br_chacha_seed(source_or_seed & MASK64, C.byref(st))
        elif generator == "pcg64":
            N.lib().br_pcg64_seed(source_or_seed & MASK64, C.byref(st))
        else:
            raise UnknownGenerator(f"no device generator {generator!r}")
    else:
        st = _state_struct(source_or_seed)
    out = torch.empty(count, dtype=torch.int64, device="cuda")
    N.check(N.lib().br_pcg64_fill(_ptr(out), count, C.byref(st), offset, _stream_ptr(torch)), "pcg64_fill")
    return out


def _segmented_call(flat, n, num_arrays, run_seed, base, schedule, gen_id, naive, words, stream_ptr):
    L = N.lib()
    if naive:
        return L.br_shuffle_naive_segmented(_ptr(flat), flat.element_size(), num_arrays, n, run_seed & MASK64, base,
                                            gen_id, _ptr(words), stream_ptr)
    regs = schedule._regimes()
    return L.br_shuffle_segmented(_ptr(flat), flat.element_size(), num_arrays, n, run_seed & MASK64, base, regs,
                                  len(regs), gen_id, _ptr(words), stream_ptr)


def _shuffle_many_host(flat, n, num_arrays, run_seed, base, schedule, gen_id, naive, words, chunks, torch):
    """shuffle_many on a host tensor (ideally pinned): the arrays go up, are shuffled and come
    back in ``chunks`` pieces, the copies on two copy streams overlapping the shuffles."""
    chunks = max(1, min(chunks, num_arrays))
    per = -(-num_arrays // chunks)
    comp = torch.cuda.current_stream()
    h2d, d2h = _copy_streams(torch)
    h2d.wait_stream(comp)
    d2h.wait_stream(comp)
    dbufs = [torch.empty(per * n, dtype=flat.dtype, device="cuda") for _ in range(min(2, chunks))]
    dwords = [torch.empty(per, dtype=torch.int32, device="cuda") if words is not None else None
              for _ in range(len(dbufs))]
    freed = [None] * len(dbufs)
    for c, a0 in enumerate(range(0, num_arrays, per)):
        na = min(per, num_arrays - a0)
        slot = c % len(dbufs)
        with torch.cuda.stream(h2d):
            if freed[slot] is not None:
                h2d.wait_event(freed[slot])
            dbufs[slot][: na * n].copy_(flat[a0 * n: (a0 + na) * n], non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(h2d)
        comp.wait_event(ready)
        N.check(_segmented_call(dbufs[slot][: na * n], n, na, run_seed, base + a0, schedule, gen_id, naive,
                                dwords[slot], C.c_void_p(comp.cuda_stream)), "shuffle_many")
        done = torch.cuda.Event()
        done.record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(done)
            flat[a0 * n: (a0 + na) * n].copy_(dbufs[slot][: na * n], non_blocking=True)
            if words is not None:
                words[a0: a0 + na].copy_(dwords[slot][:na], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(d2h)
            freed[slot] = ev
    comp.wait_stream(d2h)
    comp.wait_stream(h2d)
    for t in dbufs + dwords:
        if t is not None:
            t.record_stream(h2d)
            t.record_stream(d2h)


def shuffle_many(data, n: int, run_seed: int, array_index_base: int = 0,
                 schedule: ShuffleSchedule = DEFAULT_SCHEDULE, return_words: bool = False,
                 generator: str = "pcg64", naive: bool = False, chunks: int = 8, sync: bool = True):
    """Independent shuffles of the num_arrays = data.numel() // n contiguous arrays of a
    tensor (4- or 8-byte items), in place: array a is
    shuffle_batched(make_source(generator, array_seed(run_seed, array_index_base + a)), ...)
    with generator "pcg64", "lehmer" or "chacha" -- or, with ``naive``,
    shuffle_naive_batched(make_source(...), ...) (schedule ignored).

    A CUDA tensor is shuffled where it is (asynchronously on the current stream).  A host
    tensor (pinned for overlap) is copied up, shuffled and copied back in ``chunks`` pipelined
    pieces; with ``sync`` the call returns once the host data holds the result."""
    if generator not in _GENERATOR_IDS:
        raise UnknownGenerator(f"no device generator {generator!r}")
    torch = _torch()
    flat = data.view(-1)
    if flat.element_size() not in (4, 8):
        raise TypeError("data must be a tensor of 4- or 8-byte items")
    if n <= 0 or flat.numel() % n:
        raise ValueError("data length must be a multiple of n")
    num_arrays = flat.numel() // n
    gid = _GENERATOR_IDS[generator]
    if not flat.is_cuda:
        words = torch.empty(num_arrays, dtype=torch.int32, pin_memory=flat.is_pinned()) if return_words else None
        if num_arrays:
            _shuffle_many_host(flat, n, num_arrays, run_seed, array_index_base, schedule, gid, naive, words, chunks,
                               torch)
        if sync:
            torch.cuda.current_stream().synchronize()
        return (data, words) if return_words else data
    words = torch.empty(num_arrays, dtype=torch.int32, device="cuda") if return_words else None
    N.check(_segmented_call(flat, n, num_arrays, run_seed, array_index_base, schedule, gid, naive, words,
                            _stream_ptr(torch)), "shuffle_many")
    return (data, words) if return_words else data


def last_kernel() -> str:
    """Which kernel the last device call on this thread launched (diagnostics)."""
    return N.last_kernel()


__all__ = [
    "BatchRandError", "BatchResult", "BatchSpec", "BoundEncoding", "BoundOverflow", "DEFAULT_SCHEDULE",
    "RollOutcome", "roll_single", "roll_single_traced",
    "DigitOutOfRange", "DeviceStream", "FullProduct", "PAIR_SCHEDULE", "Pcg64Source", "RadixBases",
    "RollBatchesResult", "ShuffleSchedule", "SourceExhausted", "UnknownGenerator", "ValueOutOfRange",
    "WordSource", "array_seed", "default_schedule", "digit_pass", "digit_pass_many", "falling_factorial",
    "make_source", "mul_full", "LehmerSource", "ChaChaSource", "GENERATORS", "partial_shuffle_batch", "pcg64_fill", "roll_batch", "roll_batch_known_threshold",
    "roll_batch_naive", "shuffle_naive_batched", "encode", "decode", "chacha_block",
    "FixedSequenceSource", "ExhaustiveSource",
    "roll_batches", "shuffle_batched", "shuffle_many", "shuffle_unbatched", "splitmix64_stream", "threshold",
    "last_kernel",
]
