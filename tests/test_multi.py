"""World-size-2 tests of the multi-GPU host logic on CPU (gloo).  The rolls themselves are
computed by the oracle here (no GPU); the point is the sharding, the seed/offset bookkeeping
and the rejection-count exchange, which bench.py drives over NCCL on GPUs."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O

    from paper_2408_06213_b200 import shard

    if mode in ("rolls", "rolls3"):
        nb = 6000
        bounds = _roll_bounds(nb, mode == "rolls3")
        seed_state = shard.seeded_state(O.array_seed(7, 1))

        def roll(state, first, count):
            src = O.pcg64_from_state(*state)
            rolls, words, _, _ = O.roll_batches(src, bounds[2 * first: 2 * (first + count)], 2)
            return (rolls, words), int(words.astype(np.int64).sum()) - count

        (rolls, words), first, count, d, rec = shard.sharded_rolls(seed_state, nb, world, rank, roll)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), rolls=rolls, words=words, first=first, d=d, rec=rec)
    else:
        na, n = 37, 100
        first, count = shard.even_split(na, world, rank)
        data = np.tile(np.arange(n, dtype=np.uint32), count)
        O.shuffle_segmented(data, n, 1234, array_index_base=first)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), data=data, first=first)
    dist.barrier()
    dist.destroy_process_group()


def _roll_bounds(nb, cascade):
    rng = np.random.default_rng(0)
    bounds = rng.integers(2, 1 << 16, 2 * nb, dtype=np.uint32)
    # heavy batches (~30% rejection) on rank 0's section force cross-rank shifts; with
    # `cascade` the middle rank's section has them too, so its re-roll changes its own
    # rejection count and the last rank's shift needs a second round
    spans = [(0, 40)] + ([(2 * 3800, 2 * 3800 + 300)] if cascade else [])  # rank 1 re-rolls 58 -> 63 extra
    for a, b in spans:
        bounds[a:b:2] = 0xFFFFFFFF
        bounds[a + 1:b:2] = 3006477107
    return bounds


def _run(mode, tmp_path, world=2):
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, mode, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    return [np.load(tmp_path / f"r{r}.npz") for r in range(world)]


def test_even_split():
    from paper_2408_06213_b200.shard import even_split

    for total in (0, 1, 7, 256, 1000):
        for world in (1, 2, 3, 8):
            spans = [even_split(total, world, r) for r in range(world)]
            assert sum(c for _, c in spans) == total
            assert all(spans[r][0] + spans[r][1] == spans[r + 1][0] for r in range(world - 1))


def test_sharded_segmented_equals_single_process(tmp_path, O):
    parts = _run("arrays", tmp_path)
    got = np.concatenate([p["data"] for p in parts])
    ref = np.tile(np.arange(100, dtype=np.uint32), 37)
    O.shuffle_segmented(ref, 100, 1234)
    assert np.array_equal(got, ref)


def test_sharded_roll_stream_equals_single_stream(tmp_path, O):
    parts = _run("rolls", tmp_path)
    nb = 6000
    bounds = _roll_bounds(nb, False)
    rolls, words, _, _ = O.roll_batches(O.pcg64(O.array_seed(7, 1)), bounds, 2)
    assert int(parts[1]["d"]) > 0 and bool(parts[1]["rec"])  # rank 1 was shifted by rank 0's rejections
    assert np.array_equal(np.concatenate([p["rolls"] for p in parts]), rolls)
    assert np.array_equal(np.concatenate([p["words"] for p in parts]), words)


def test_sharded_roll_stream_cascading_shifts(tmp_path, O):
    """Three ranks, rejections in two sections: the shifted middle rank's re-roll changes its
    own extra count, and the last rank must follow (fixed-point rounds in sharded_rolls)."""
    parts = _run("rolls3", tmp_path, world=3)
    nb = 6000
    bounds = _roll_bounds(nb, True)
    rolls, words, _, _ = O.roll_batches(O.pcg64(O.array_seed(7, 1)), bounds, 2)
    assert all(bool(p["rec"]) for p in parts[1:])
    assert np.array_equal(np.concatenate([p["rolls"] for p in parts]), rolls)
    assert np.array_equal(np.concatenate([p["words"] for p in parts]), words)


# ------------------------------------------------------------- single-process sections (multi.py)
def _oracle_sections(O, bounds, nb, S):
    """resolve_sections driven by the oracle as the section roller (the GPU tests drive it with
    the device kernels): the concatenated sections equal one sequential stream."""
    from paper_2408_06213_b200 import multi, shard

    state, inc = shard.seeded_state(O.array_seed(7, 1))
    res = {}

    def roll(r, shift):
        first, count = shard.even_split(nb, S, r)
        st, _ = shard.advanced_state(state, inc, first + shift)
        rolls, words, _, _ = O.roll_batches(O.pcg64_from_state(st, inc), bounds[2 * first: 2 * (first + count)], 2)
        res[r] = (rolls, words)
        return int(words.astype(np.int64).sum()) - count

    extras = [roll(r, 0) for r in range(S)]
    shifts = multi.resolve_sections(extras, roll)
    return res, shifts


def test_resolve_sections_single_process(O):
    nb = 6000
    for S, cascade in ((2, False), (3, True), (5, True)):
        bounds = _roll_bounds(nb, cascade)
        res, shifts = _oracle_sections(O, bounds, nb, S)
        rolls, words, _, _ = O.roll_batches(O.pcg64(O.array_seed(7, 1)), bounds, 2)
        assert shifts[0] == 0 and shifts[1] > 0
        assert np.array_equal(np.concatenate([res[r][0] for r in range(S)]), rolls)
        assert np.array_equal(np.concatenate([res[r][1] for r in range(S)]), words)


def test_resolve_sections_fixed_point_rounds():
    """A re-roll that changes the section's own extras moves every later section again."""
    from paper_2408_06213_b200 import multi

    calls = []

    def reroll(r, d):
        calls.append((r, d))
        return {1: 5, 2: 0, 3: 1}.get(r, 0) if d else 0

    shifts = multi.resolve_sections([3, 0, 0, 0], reroll)
    assert shifts == [0, 3, 8, 8]
    assert (1, 3) in calls and (2, 8) in calls and (3, 8) in calls
