"""The stage-pipeline shuffle kernel (csrc/stage_shuffle.cuh) against the oracle: forced through
BR_SHUFFLE_KERNEL=stage on lengths around the block size and far beyond it, u32 and u64,
PCG64 and Lehmer, batched and naive plans, several schedules; every array compared bit-exactly
with the oracle's sequential shuffle, plus the words consumed per array."""

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


def _run(B, O, n, na, eb, gen, naive=False, schedule=None, seed=4321, base=17):
    dt = np.uint32 if eb == 4 else np.uint64
    payload = np.arange(n * na, dtype=dt) * 3 + 1
    dev = torch.from_numpy(payload.view(np.int32 if eb == 4 else np.int64).copy()).cuda()
    kw = {} if schedule is None else {"schedule": schedule}
    _, w = B.shuffle_many(dev, n, seed, array_index_base=base, return_words=True, generator=gen, naive=naive, **kw)
    kern = B.last_kernel()
    ref = payload.copy()
    if naive:
        rw = O.shuffle_naive_segmented(ref, n, seed, array_index_base=base, generator=gen)
    elif schedule is None:
        rw = O.shuffle_segmented(ref, n, seed, array_index_base=base, generator=gen)
    else:
        rw = O.shuffle_segmented(ref, n, seed, array_index_base=base, generator=gen, entries=schedule.entries)
    got = dev.cpu().numpy().view(dt)
    return kern, got, ref, w.cpu().numpy().view(np.uint32), rw


@pytest.mark.parametrize("gen", ["pcg64", "lehmer"])
@pytest.mark.parametrize("eb", [4, 8])
@pytest.mark.parametrize("n", [2, 3, 64, 1000, 4095, 4096, 4097, 8197, 70000, 300001])
def test_stage_forced(B, O, monkeypatch, n, eb, gen):
    monkeypatch.setenv("BR_SHUFFLE_KERNEL", "stage")
    na = max(3, min(40, (1 << 21) // n))
    for naive in (False, True):
        kern, got, ref, w, rw = _run(B, O, n, na, eb, gen, naive)
        assert "shuffle_stage_kernel" in kern, kern
        bad = [a for a in range(na) if not np.array_equal(got[a * n:(a + 1) * n], ref[a * n:(a + 1) * n])]
        assert not bad, (n, eb, gen, naive, bad[:5])
        assert np.array_equal(w, rw)


@pytest.mark.parametrize("maxb", [2, 3, 6])
def test_stage_schedules(B, O, monkeypatch, maxb):
    monkeypatch.setenv("BR_SHUFFLE_KERNEL", "stage")
    sched = B.default_schedule(maxb)
    for n in (5000, 123457):
        kern, got, ref, w, rw = _run(B, O, n, 6, 8, "pcg64", schedule=sched, seed=99)
        assert "shuffle_stage_kernel" in kern and np.array_equal(got, ref) and np.array_equal(w, rw), (maxb, n)
    # a schedule with 8 dice per word at the bottom (ring room for the largest generation step)
    s8 = B.ShuffleSchedule(entries=((1 << 30, 2), (1 << 19, 3), (1 << 14, 4), (1 << 11, 5), (1 << 9, 6), (200, 7),
                                    (120, 8)), max_batch=8, word_bits=64)
    kern, got, ref, w, rw = _run(B, O, 33333, 5, 4, "lehmer", schedule=s8, seed=5)
    assert "shuffle_stage_kernel" in kern and np.array_equal(got, ref) and np.array_equal(w, rw)


def test_stage_c5_shape(B, O, monkeypatch):
    """C5 shape (u64[2^20]), 12 arrays, every one bit-exact (each has ~172 rejected words, so the
    realignment runs inside every array)."""
    monkeypatch.setenv("BR_SHUFFLE_KERNEL", "stage")
    n, na = 1 << 20, 12
    kern, got, ref, w, rw = _run(B, O, n, na, 8, "pcg64", seed=5, base=100)
    assert "shuffle_stage_kernel" in kern, kern
    assert np.array_equal(got, ref) and np.array_equal(w, rw)
    assert (w.astype(np.int64) - 435422 > 100).all()  # rejections happened in every array
