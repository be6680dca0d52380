"""Host-side sharding logic for one job spread over several GPUs.

* Segmented shuffles (C3/C4/C5): arrays are independent; each rank takes a contiguous
  array range and passes its first global index as ``array_index_base``.  Seeds depend only
  on (run_seed, global array index), so there is no data-path collective.
* One bulk-roll stream (C2): rank r rolls the batches [first, first+count) of the global
  sequence, starting at word ``first + D_prefix`` where D_prefix counts the extra words drawn
  by rejections on earlier ranks.  Ranks speculate D_prefix = 0, exchange their own extra
  counts (the only exchange: one int64 per rank) and recompute only if an earlier rank
  rejected something (P ~ 2^-10 per 2^25 batches for C2).
"""

from __future__ import annotations

import ctypes as C
from typing import Callable, Sequence

from . import _native as N

MASK64 = (1 << 64) - 1


def even_split(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous (first, count) of rank's share of `total` units."""
    per, rem = divmod(total, world)
    first = rank * per + min(rank, rem)
    return first, per + (1 if rank < rem else 0)


def advanced_state(state: int, increment: int, words: int) -> tuple[int, int]:
    """PCG64 (state, increment) after `words` more words (native host jump-ahead)."""
    st = N.Pcg64State()
    st.state_hi, st.state_lo = (state >> 64) & MASK64, state & MASK64
    st.inc_hi, st.inc_lo = (increment >> 64) & MASK64, increment & MASK64
    N.lib().br_pcg64_advance(C.byref(st), words & MASK64)
    return (st.state_hi << 64) | st.state_lo, increment


def seeded_state(seed: int) -> tuple[int, int]:
    st = N.Pcg64State()
    N.lib().br_pcg64_seed(seed & MASK64, C.byref(st))
    return (st.state_hi << 64) | st.state_lo, (st.inc_hi << 64) | st.inc_lo


def rejection_prefix(extras: Sequence[int], rank: int) -> int:
    """Words by which rank's section is shifted: the extra words of all earlier ranks."""
    return int(sum(int(x) for x in extras[:rank]))


def all_gather_ints(value: int, group=None, device=None) -> list[int]:
    """One int64 per rank via torch.distributed (NCCL on GPUs, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = torch.tensor([value], dtype=torch.int64, device=device)
    out = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [int(x.item()) for x in out]


def sharded_rolls(seed_state: tuple[int, int], total_batches: int, world: int, rank: int,
                  roll: Callable[[tuple[int, int], int, int], tuple[object, int]], group=None, device=None):
    """Run this rank's section of one global roll stream.

    ``roll(state, first_batch, count) -> (result, extra_words)`` rolls `count` batches from
    the given generator state.  Returns (result, first_batch, count, d_prefix, recomputed).
    """
    first, count = even_split(total_batches, world, rank)
    state = advanced_state(seed_state[0], seed_state[1], first)
    res, extra = roll(state, first, count)
    d, recomputed = 0, False
    # A shifted rank re-rolls, which can change its own extra count and so the shift of the
    # ranks after it: iterate to the fixed point (at most `world` rounds; rank 0 never
    # moves, and each round fixes at least the next rank's prefix).  One round when nothing
    # was rejected.
    for _ in range(world):
        extras = all_gather_ints(extra, group, device)
        nd = rejection_prefix(extras, rank)
        moved = nd != d
        if moved:
            d = nd
            state = advanced_state(seed_state[0], seed_state[1], first + d)
            res, extra = roll(state, first, count)
            recomputed = True
        if not any(all_gather_ints(int(moved), group, device)):
            break
    return res, first, count, d, recomputed
