"""The single-process multi-shard entry points (paper_2408_06213_b200.multi) on one GPU: S
shards on S streams of device 0, against the oracle -- segmented shuffles (C3/C4/C5 shapes,
host and device data) and one bulk-roll stream cut into sections, including sections shifted
by an earlier section's rejections."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.fixture(scope="module")
def B():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2408_06213_b200 as B

    return B


@pytest.mark.parametrize("n,na,eb", [(64, 3001, 4), (4096, 301, 4), (70000, 7, 8), (1 << 20, 5, 8)])
@pytest.mark.parametrize("where", ["device", "host"])
def test_shuffle_many_sharded(B, O, n, na, eb, where):
    from paper_2408_06213_b200 import multi

    dt = np.uint32 if eb == 4 else np.uint64
    payload = np.arange(n * na, dtype=dt) * 7 + 3
    t = torch.from_numpy(payload.view(np.int32 if eb == 4 else np.int64).copy())
    t = t.cuda() if where == "device" else t.pin_memory()
    _, w = multi.shuffle_many_sharded(t, n, 77, devices=[0, 0, 0], array_index_base=11, return_words=True)
    torch.cuda.synchronize()
    ref = payload.copy()
    rw = O.shuffle_segmented(ref, n, 77, array_index_base=11)
    assert np.array_equal(t.cpu().numpy().view(dt), ref)
    assert np.array_equal(w.cpu().numpy().view(np.uint32), rw)


def _bounds(O, nb, heavy):
    b = O.gen_bounds(7, 2 * nb)
    for lo, hi in heavy:  # products near 2^64: ~30% of these batches are rejected
        b[2 * lo: 2 * hi: 2] = 0xFFFFFFFF
        b[2 * lo + 1: 2 * hi: 2] = 3006477107
    return b


@pytest.mark.parametrize("S,heavy", [(1, []), (4, []), (4, [(0, 50)]), (3, [(0, 40), (40000, 40300)]),
                                     (8, [(1000, 1200), (90000, 90100)])])
@pytest.mark.parametrize("where", ["device", "host"])
def test_roll_batches_sharded(B, O, S, heavy, where):
    """One stream over S sections; rejections in early sections shift the later ones, which
    are re-rolled on the device; results and the advanced source equal one sequential stream."""
    from paper_2408_06213_b200 import multi

    nb = 120_000
    b = _bounds(O, nb, heavy)
    tb = torch.from_numpy(b.view(np.int32))
    tb = tb.cuda() if where == "device" else tb.pin_memory()
    src = B.Pcg64Source(O.array_seed(7, 1))
    rolls, words, shifts = multi.roll_batches_sharded(src, tb, 2, devices=[0] * S)
    o = O.pcg64(O.array_seed(7, 1))
    rr, wr, _, _ = O.roll_batches(o, b, 2)
    assert np.array_equal(rolls.cpu().numpy().view(np.uint32), rr)
    assert np.array_equal(words.cpu().numpy(), wr)
    assert src.state == o.state
    if heavy and S > 1:
        assert shifts[-1] > 0


def test_roll_batches_sharded_generators(B, O):
    from paper_2408_06213_b200 import multi

    nb = 50_000
    b = _bounds(O, nb, [(100, 160)])
    for gen in ("lehmer", "chacha"):
        src = B.make_source(gen, 5)
        rolls, words, _ = multi.roll_batches_sharded(src, torch.from_numpy(b.view(np.int32)).cuda(), 2,
                                                     devices=[0, 0, 0])
        o = O.GENERATOR_MAKERS[gen](5)
        rr, wr, _, _ = O.roll_batches(o, b, 2)
        assert np.array_equal(rolls.cpu().numpy().view(np.uint32), rr), gen
        assert np.array_equal(words.cpu().numpy(), wr), gen
