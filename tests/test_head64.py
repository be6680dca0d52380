"""Arrays of 2^32 or more elements (shuffle.py:175-190): the single-roll head above 2^32 - 1
runs in shuffle_head64_kernel (csrc/head64.cuh), the rest continues on the 32-bit kernels.

* Exactness of the head kernel against the oracle on small arrays, with the split lowered by
  BR_HEAD64_STOP (every generator, u32 and u64, unbatched and a schedule whose top regime is
  below the split, and replayed words with forced rejections).
* The real single-roll head of the default schedule at n = 2^30 + 4097 (u32), every element
  against the oracle.
* A real n = 2^32 + 2^16 (16 GiB): the head positions against a sparse replay of the
  reference's head loop, the rest by permutation checksums, and the stream's next word.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

MASK = (1 << 64) - 1


@pytest.fixture(scope="module")
def B():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2408_06213_b200 as B

    return B


def _dev(n, eb):
    if eb == 4:
        return torch.arange(n, dtype=torch.int32, device="cuda")
    return torch.arange(n, dtype=torch.int64, device="cuda") * 3 + 1


def _host(t, eb):
    return t.cpu().numpy().view(np.uint32 if eb == 4 else np.uint64)


@pytest.mark.parametrize("gen", ["pcg64", "lehmer", "chacha"])
@pytest.mark.parametrize("eb", [4, 8])
def test_head64_forced(B, O, monkeypatch, gen, eb):
    monkeypatch.setenv("BR_HEAD64_STOP", "3000")
    sched = B.ShuffleSchedule(entries=((1000, 2), (100, 3)), max_batch=3, word_bits=64)
    for n, schedule in ((9000, None), (20000, sched), (3001, None), (4024, sched)):
        z = _dev(n, eb)
        ref0 = _host(z, eb).copy()
        src = B.make_source(gen, 77 + n)
        o = O.GENERATOR_MAKERS[gen](77 + n)
        if schedule is None:
            B.shuffle_unbatched(src, z)
            ref = O.shuffle_unbatched(o, ref0)
        else:
            B.shuffle_batched(src, z, schedule)
            ref = O.shuffle_batched(o, ref0, entries=schedule.entries)
        assert "shuffle_head64_kernel" in B.last_kernel(), B.last_kernel()
        assert np.array_equal(_host(z, eb), ref), (gen, eb, n)
        assert src.next_word() == O.next_word(o)


def test_head64_rejections(B, O, monkeypatch):
    """Replayed words with zeros in the head: each zero is rejected (lo = 0 < 2^64 mod b) and
    the step re-drawn from the next word, shifting every later step (shuffle.py:181-186)."""
    monkeypatch.setenv("BR_HEAD64_STOP", "1000")
    n = 5000
    rng = np.random.default_rng(3)
    words = [int(w) for w in rng.integers(1, 1 << 63, size=n + 64, dtype=np.int64)]
    for p in (0, 1, 2, 700, 1023, 1024, 1025, 2047, 3000, 3998):  # group edges and runs
        words.insert(p, 0)
    z = _dev(n, 4)
    src = B.FixedSequenceSource(words, 64)
    B.shuffle_unbatched(src, z)
    o = O.fixed(words)
    ref = O.shuffle_unbatched(o, np.arange(n, dtype=np.uint32))
    assert "shuffle_head64_kernel" in B.last_kernel()
    assert np.array_equal(_host(z, 4), ref)
    assert src.cursor == n - 1 + 10


def _sparse_head(O, o, n, stop):
    """The reference's single-roll loop (shuffle.py:175-190) for positions n-1 .. stop on a
    sparse array (position -> original index); returns the final index at each position."""
    cur = {}
    for i in range(n - 1, stop - 1, -1):
        b = i + 1
        p = b * O.next_word(o)
        lo = p & MASK
        if lo < b:
            t = ((1 << 64) - b) % b
            while lo < t:
                p = b * O.next_word(o)
                lo = p & MASK
        j = p >> 64
        ci, cj = cur.get(i, i), cur.get(j, j)
        cur[i], cur[j] = cj, ci
    return cur


def test_single_roll_head_2p30(B, O):
    """Default schedule at n = 2^30 + 4097 (u32): 4097 single rolls above 2^30, then the k=2
    regime; every element and the stream's next word against the oracle."""
    n = (1 << 30) + 4097
    z = torch.arange(n, dtype=torch.int32, device="cuda")
    src = B.make_source("pcg64", 11)
    B.shuffle_batched(src, z)
    got = z.cpu().numpy().view(np.uint32)
    del z
    torch.cuda.empty_cache()
    o = O.pcg64(11)
    ref = O.shuffle_batched(o, np.arange(n, dtype=np.uint32))
    assert np.array_equal(got, ref)
    assert src.next_word() == O.next_word(o)


@pytest.mark.slow
def test_array_of_2p32_plus(B, O):
    """n = 2^32 + 2^16 u32 through the drop-in shuffle_batched: the head kernel, then the
    32-bit path on 2^32 - 1 elements.  The head positions (final after the head) against a
    sparse replay of the reference loop; the whole array by permutation checksums."""
    n = (1 << 32) + (1 << 16)
    stop = (1 << 32) - 1
    free, _ = torch.cuda.mem_get_info()
    if free < n * 4 + (2 << 30):
        pytest.skip("not enough device memory")
    z = torch.empty(n, dtype=torch.int32, device="cuda")
    idx = torch.arange(n, dtype=torch.int64, device="cuda")
    z.copy_(idx.to(torch.int32))  # values = index mod 2^32
    del idx

    def sums(t):
        v = t.to(torch.int64) & 0xFFFFFFFF
        return int(v.sum().item()), int((v * v).sum().item()) & MASK

    s0 = [0, 0]
    for c in torch.split(z, 1 << 28):
        a, b = sums(c)
        s0[0] += a
        s0[1] = (s0[1] + b) & MASK
    src = B.make_source("pcg64", 23)
    B.shuffle_batched(src, z)
    assert "shuffle_head64_kernel" in B.last_kernel()
    s1 = [0, 0]
    for c in torch.split(z, 1 << 28):
        a, b = sums(c)
        s1[0] += a
        s1[1] = (s1[1] + b) & MASK
    assert s0 == s1
    o = O.pcg64(23)
    head = _sparse_head(O, o, n, stop)
    top = z[stop:].cpu().numpy().view(np.uint32)
    want = np.array([head.get(i, i) & 0xFFFFFFFF for i in range(stop, n)], dtype=np.uint32)
    assert np.array_equal(top, want)
