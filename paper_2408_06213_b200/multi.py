"""One job over several GPUs -- or several streams of one GPU -- from a single process
(the torchrun form, one process per GPU, is ``shard`` + ``bench.py --gpus N``).

* ``shuffle_many_sharded``: the arrays of a segmented shuffle (C3/C4/C5) are cut into S
  contiguous ranges; shard r runs ``shuffle_many`` on its range on ``devices[r]`` and its own
  stream, passing the range's first global index as ``array_index_base``.  Array a's seed
  depends only on (run_seed, global a), so the result equals the one-call result and there is
  no exchange between shards.
* ``roll_batches_sharded``: one global bulk-roll stream (C2) cut into S batch sections.  Shard
  r starts at word ``first_r`` (jump-ahead), speculating that no earlier section rejected a
  batch.  Each shard reports its extra words (``br_roll_check``); a section after a rejecting
  one is shifted by the sum of the earlier extras and re-rolled on its device, to the fixed
  point (``resolve_sections``; the same rule as ``shard.sharded_rolls``, which does it across
  processes with one all-gather).

Each shard's kernels are the product kernels; the host only splits ranges and orders
streams.  With ``devices=[0, 0, 0, 0]`` a single GPU runs four shards on four streams (how
the GPU tests cover the multi-shard path on a one-GPU box).
"""

from __future__ import annotations

import ctypes as C
from typing import Callable, List, Optional, Sequence

from . import _native as N
from . import batchrand as BR
from .shard import even_split

MASK64 = (1 << 64) - 1

_STREAMS = {}


def _shard_stream(torch, device: int, idx: int):
    """A cached side stream per (device, shard index)."""
    key = (device, idx)
    if key not in _STREAMS:
        _STREAMS[key] = torch.cuda.Stream(device=device)
    return _STREAMS[key]


def _devices(torch, devices: Optional[Sequence[int]]) -> List[int]:
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devices = [int(d) for d in devices]
    if not devices:
        raise ValueError("need at least one device")
    count = torch.cuda.device_count()
    for d in devices:
        if not 0 <= d < count:
            raise ValueError(f"no CUDA device {d} (have {count})")
    return devices


def resolve_sections(extras: List[int], reroll: Callable[[int, int], int]) -> List[int]:
    """Word shifts of S consecutive sections of one stream.

    ``extras[r]`` are the extra words section r drew when rolled with shift 0;
    ``reroll(r, d)`` re-rolls section r shifted by d words and returns its new extra words.
    Section r's shift is the sum of the (final) extras of the sections before it; a re-roll
    can change a section's own extras and so the shifts after it, hence the loop (at most S
    rounds: section 0 never moves).  Returns the final shifts."""
    S = len(extras)
    extras = list(extras)
    shifts = [0] * S
    for _ in range(S):
        moved = False
        acc = 0
        for r in range(S):
            if acc != shifts[r]:
                shifts[r] = acc
                extras[r] = reroll(r, acc)
                moved = True
            acc += extras[r]
        if not moved:
            break
    return shifts


def _to_device(torch, t, device, stream):
    if t.is_cuda and t.device.index == device:
        return t
    return t.to(device=torch.device("cuda", device), non_blocking=True)


def shuffle_many_sharded(data, n: int, run_seed: int, devices: Optional[Sequence[int]] = None,
                         array_index_base: int = 0, schedule=None, return_words: bool = False,
                         generator: str = "pcg64", naive: bool = False):
    """``shuffle_many`` with the arrays split over ``devices`` (one shard per entry, each on its
    own stream; repeat a device for several streams on it).

    ``data`` is a host tensor (pinned for overlapping copies) or a CUDA tensor; each shard's
    range is copied to its device when it lives elsewhere, shuffled there and copied back.
    Returns ``data`` (and the int32 words per array with ``return_words``), complete on return
    for host data and ordered before the current stream's later work for CUDA data."""
    torch = BR._torch()
    devices = _devices(torch, devices)
    schedule = BR.DEFAULT_SCHEDULE if schedule is None else schedule
    flat = data.view(-1)
    if flat.element_size() not in (4, 8):
        raise TypeError("data must be a tensor of 4- or 8-byte items")
    if n <= 0 or flat.numel() % n:
        raise ValueError("data length must be a multiple of n")
    num_arrays = flat.numel() // n
    words = None
    if return_words:
        words = (torch.empty(num_arrays, dtype=torch.int32, device=flat.device) if flat.is_cuda else
                 torch.empty(num_arrays, dtype=torch.int32, pin_memory=flat.is_pinned()))
    S = len(devices)
    src_ready = torch.cuda.current_stream(flat.device) if flat.is_cuda else None
    done = []
    for r, dev in enumerate(devices):
        first, count = even_split(num_arrays, S, r)
        if count == 0:
            continue
        st = _shard_stream(torch, dev, r)
        with torch.cuda.device(dev), torch.cuda.stream(st):
            if src_ready is not None:
                st.wait_stream(src_ready) if src_ready.device.index == dev else st.wait_event(_event(torch, src_ready))
            part = flat[first * n:(first + count) * n]
            local = _to_device(torch, part, dev, st)
            _, w = BR.shuffle_many(local, n, run_seed, array_index_base=array_index_base + first,
                                   schedule=schedule, return_words=True, generator=generator, naive=naive)
            if local.data_ptr() != part.data_ptr():
                part.copy_(local, non_blocking=True)
            if words is not None:
                words[first:first + count].copy_(w, non_blocking=True)
            for t in (local, w):
                t.record_stream(st)
            done.append((dev, st))
    if flat.is_cuda:
        cur = torch.cuda.current_stream(flat.device)
        for dev, st in done:
            cur.wait_event(_event(torch, st)) if dev != flat.device.index else cur.wait_stream(st)
    else:
        for _, st in done:
            st.synchronize()
    return (data, words) if return_words else data


def _event(torch, stream):
    ev = torch.cuda.Event()
    ev.record(stream)
    return ev


def roll_batches_sharded(source, bounds, k: int, devices: Optional[Sequence[int]] = None, naive: bool = False):
    """``roll_batches`` of one source over ``devices``: the batches are cut into S consecutive
    sections, each rolled on its device and stream from the source's word stream jumped ahead
    to the section's first batch; sections shifted by an earlier section's rejections are
    re-rolled (``resolve_sections``).  The results equal one sequential
    ``[roll_batch(source, ...) for each batch]``; the source (a PCG64/Lehmer/ChaCha source, or
    a seed for a fresh PCG64 stream) is advanced by the words consumed.

    ``bounds`` (4-byte items, batch-major) is a host or CUDA tensor; the results (rolls int32,
    words uint8) are host tensors for host bounds and tensors on the bounds' device otherwise.
    Returns (rolls, words, shifts) where shifts[r] is the word shift section r ended with."""
    torch = BR._torch()
    devices = _devices(torch, devices)
    import numpy as np

    if isinstance(bounds, np.ndarray):
        bounds = torch.from_numpy(np.ascontiguousarray(bounds).view(np.int32))
    b = bounds.reshape(-1)
    if b.element_size() != 4:
        raise TypeError("bounds must have 4-byte items")
    if k <= 0 or b.numel() % k:
        raise ValueError("bounds length must be a multiple of k")
    nb = b.numel() // k
    host_source = None
    if isinstance(source, int):
        st0 = N.Pcg64State()
        N.lib().br_pcg64_seed(source & MASK64, C.byref(st0))
    else:
        if BR._is_fixed(source):
            raise TypeError("a replayed word sequence cannot be cut into sections; use roll_batches")
        host_source = source
        st0 = BR._state_struct(source)
    S = len(devices)
    out_dev = b.device if b.is_cuda else None
    rolls = torch.empty(nb * k, dtype=torch.int32, device=out_dev, pin_memory=not b.is_cuda and b.is_pinned())
    words = torch.empty(nb, dtype=torch.uint8, device=out_dev, pin_memory=not b.is_cuda and b.is_pinned())
    src_ready = torch.cuda.current_stream(b.device) if b.is_cuda else None
    shards = []
    for r, dev in enumerate(devices):
        # sections in whole groups of 4 batches: every section's bounds and rolls start on a
        # 16-byte boundary (the roll kernels load and store 16-byte vectors)
        fu, cu = even_split((nb + 3) // 4, S, r)
        first = min(nb, 4 * fu)
        count = min(nb, 4 * (fu + cu)) - first
        st = _shard_stream(torch, dev, r)
        with torch.cuda.device(dev), torch.cuda.stream(st):
            if src_ready is not None:
                st.wait_stream(src_ready) if src_ready.device.index == dev else st.wait_event(_event(torch, src_ready))
            lb = _to_device(torch, b[first * k:(first + count) * k], dev, st)
            lb.record_stream(st)
            shards.append({"dev": dev, "stream": st, "first": first, "count": count, "bounds": lb})

    def roll(r: int, shift: int) -> int:
        sh = shards[r]
        if sh["count"] == 0:
            sh["ds"] = None
            return 0
        st = type(st0)()
        C.memmove(C.byref(st), C.byref(st0), C.sizeof(st0))
        N.lib().br_pcg64_advance(C.byref(st), (sh["first"] + shift) & MASK64)
        with torch.cuda.device(sh["dev"]), torch.cuda.stream(sh["stream"]):
            ds = BR.DeviceStream.from_struct(st)
            res = BR.roll_batches(ds, sh["bounds"], k, check=False, naive=naive)
            extra = C.c_uint64()
            N.check(N.lib().br_roll_check(BR._ptr(ds.workspace), BR._stream_ptr(torch), C.byref(extra)),
                    "roll_batches_sharded")
        sh["ds"], sh["res"] = ds, res
        return int(extra.value)

    extras = [roll(r, 0) for r in range(S)]
    shifts = resolve_sections(extras, roll)
    for sh in shards:
        if sh["count"] == 0:
            continue
        with torch.cuda.device(sh["dev"]), torch.cuda.stream(sh["stream"]):
            f, c = sh["first"], sh["count"]
            rolls[f * k:(f + c) * k].copy_(sh["res"].rolls, non_blocking=True)
            words[f:f + c].copy_(sh["res"].words, non_blocking=True)
    for sh in shards:
        sh["stream"].synchronize()
    if host_source is not None:
        last = [sh for sh in shards if sh["count"]]
        if last:
            with torch.cuda.device(last[-1]["dev"]), torch.cuda.stream(last[-1]["stream"]):
                last[-1]["ds"].write_back(host_source)
    return rolls, words, shifts
