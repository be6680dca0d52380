"""Parity of the CUDA path (through the C ABI) against the oracle and the golden vectors.

Bit-exact for everything: rolls, words consumed, threshold flags, final remainders,
permutations and the advanced generator state.  Sizes are the BASELINE.json configs where
the oracle finishes in seconds (C2 prefix + 2^22 batches, all of C3, C1, samples of C4);
size-independent properties (permutation of the input, word counts) cover the rest.
"""

import hashlib
import os

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


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def dev_u32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def sha_u32(a):
    return hashlib.sha256(np.asarray(a, dtype="<u4").tobytes()).hexdigest()


# ------------------------------------------------------------------ generator
def test_pcg64_fill_matches_oracle(B, O):
    for seed, offset, count in ((0, 0, 1), (5, 0, 100000), (42, 12345, 77777), (7, (1 << 40) + 3, 4096)):
        got = u64(B.pcg64_fill(seed, count, offset))
        ref = O.pcg64_fill(O.pcg64(seed), offset, count)
        assert np.array_equal(got, ref), (seed, offset)
    assert "pcg_fill_kernel" in B.last_kernel()


# ------------------------------------------------------------------ batched rolls
def run_rolls(B, O, seed, bounds, k, flags=True, rk=True):
    src = O.pcg64(seed)
    ref = O.roll_batches(src, bounds, k)
    ds = B.DeviceStream(seed)
    r = B.roll_batches(ds, dev_u32(bounds), k, flags=flags, final_remainder=rk)
    st = ds.host_state()
    return r, ref, src, (st.state_hi << 64) | st.state_lo


def test_roll_batches_c2_prefix_golden(B, O, golden, golden_arrays):
    bounds = golden_arrays["c2_bounds"]
    ds = B.DeviceStream(golden["c2"]["roll_seed"])
    r = B.roll_batches(ds, dev_u32(bounds), 2)
    assert np.array_equal(u32(r.rolls), golden_arrays["c2_rolls"])
    assert np.array_equal(r.words.cpu().numpy(), golden_arrays["c2_words"])
    st = ds.host_state()
    assert (st.state_hi << 64 | st.state_lo) == golden["c2"]["state_after"]
    assert "roll_fast_kernel<2>" in B.last_kernel()


def test_roll_batches_c2_large_vs_oracle(B, O):
    nb = 1 << 22
    bounds = O.gen_bounds(7, 2 * nb)
    r, (rolls, words, flags, rk), src, st = run_rolls(B, O, O.array_seed(7, 1), bounds, 2)
    assert np.array_equal(u32(r.rolls), rolls)
    assert np.array_equal(r.words.cpu().numpy(), words)
    assert np.array_equal(r.flags.cpu().numpy(), flags)
    assert np.array_equal(u64(r.final_remainder), rk)
    assert st == src.state


def test_roll_batches_c2_full_size(B, O):
    """The whole C2 workload (BASELINE configs[1]: 2^25 batches, the bench's bounds and stream)
    bit-exact against the oracle, through the production call (no flags requested)."""
    nb = 1 << 25
    bounds = O.gen_bounds(7, 2 * nb)
    src = O.pcg64(O.array_seed(7, 1))
    rolls, words, _, _ = O.roll_batches(src, bounds, 2)
    ds = B.DeviceStream(O.array_seed(7, 1))
    r = B.roll_batches(ds, dev_u32(bounds), 2)
    assert "roll_fast_kernel<2>" in B.last_kernel()
    st = ds.host_state()
    assert np.array_equal(u32(r.rolls), rolls) and np.array_equal(r.words.cpu().numpy(), words)
    assert (st.state_hi << 64 | st.state_lo) == src.state


def test_one_huge_array(B, O):
    """A single array of 2^25 elements (128 MiB) through the stream call, bit-exact against the
    oracle (hundreds of rejected batches at these lengths exercise the realignment)."""
    n = 1 << 25
    s = B.Pcg64Source(2026)
    z = torch.arange(n, dtype=torch.int32, device="cuda")
    B.shuffle_batched(s, z)
    o = O.pcg64(2026)
    ref = O.shuffle_batched(o, np.arange(n, dtype=np.uint32))
    assert np.array_equal(u32(z), ref) and s.state == o.state, B.last_kernel()
    assert o.drawn > len(O.shuffle_trace(n)[0]) + 100  # the rejection path was exercised


@pytest.mark.parametrize("heavy_fraction", [0.001, 0.05, 1.0])
def test_roll_batches_forced_rejections(B, O, heavy_fraction):
    """Products near 0.7*2^64 reject ~30% of words: exercises the exact fixup path."""
    rng = np.random.default_rng(int(heavy_fraction * 1000) + 1)
    nb = 20000
    bounds = rng.integers(2, 1 << 16, 2 * nb, dtype=np.uint32)
    heavy = rng.random(nb) < heavy_fraction
    bounds[0::2][heavy] = 0xFFFFFFFF
    bounds[1::2][heavy] = 3006477107
    r, (rolls, words, flags, rk), src, st = run_rolls(B, O, 99, bounds, 2)
    assert words.max() > 1 or heavy_fraction < 0.01
    assert np.array_equal(u32(r.rolls), rolls)
    assert np.array_equal(r.words.cpu().numpy(), words)
    assert np.array_equal(r.flags.cpu().numpy(), flags)
    assert np.array_equal(u64(r.final_remainder), rk)
    assert st == src.state


@pytest.mark.parametrize("gen", ["pcg64", "lehmer", "chacha"])
def test_roll_batches_dense_rejections(B, O, gen):
    """Thousands of rejected batches spread over a long run (k = 5, bounds up to 4000: about
    one batch in 1100 rejects), three calls in a row on one workspace: each fixup iteration
    resolves one rejection and re-rolls the tail front first.  Bit-exact (the time per
    rejection is measured by tools/fixup_cost.py, not asserted here)."""
    k, nb = 5, 1 << 21
    maker = {"pcg64": O.pcg64, "lehmer": O.lehmer, "chacha": O.chacha}[gen]
    src = maker(77)
    ds = B.DeviceStream(77, generator=gen)
    for call in range(3):
        bounds = np.random.default_rng(call).integers(2, 4002, k * nb, dtype=np.uint32)
        rolls, words, flags, rk = O.roll_batches(src, bounds, k)
        r = B.roll_batches(ds, dev_u32(bounds), k, flags=True, final_remainder=True)
        assert int(words.sum()) - nb > 1000  # the rejections happened
        assert np.array_equal(u32(r.rolls), rolls) and np.array_equal(r.words.cpu().numpy(), words), (gen, call)
        assert np.array_equal(r.flags.cpu().numpy(), flags) and np.array_equal(u64(r.final_remainder), rk)
        st = ds.host_state()
        pos = (st.state_hi << 64) | st.state_lo
        assert pos == (O.chacha_position(src) if gen == "chacha" else src.state), (gen, call)


@pytest.mark.parametrize("k,nb", [(1, 50000), (1, 1 << 20), (1, 513), (2, 50001), (2, 255), (2, 1), (3, 50000),
                                  (4, 50000), (5, 50000), (6, 50000), (7, 50000), (8, 50000)])
def test_roll_batches_k_variants(B, O, k, nb):
    rng = np.random.default_rng(k * 1000 + nb)
    hi = {1: 1 << 32, 2: 1 << 32, 3: 1 << 21, 4: 1 << 16, 5: 1 << 12, 6: 1 << 10, 7: 1 << 9, 8: 1 << 8}[k]
    bounds = rng.integers(1, hi, k * nb, dtype=np.uint64).astype(np.uint32)
    if k == 3 and nb >= 50:  # some products exactly 2^64 (always accepted, threshold 0)
        bounds[: 3 * 50] = np.tile(np.array([1 << 31, 1 << 31, 4], dtype=np.uint32), 50)
    r, (rolls, words, flags, rk), src, st = run_rolls(B, O, 1000 + k, bounds, k)
    assert np.array_equal(u32(r.rolls), rolls)
    assert np.array_equal(r.words.cpu().numpy(), words)
    assert np.array_equal(r.flags.cpu().numpy(), flags)
    assert np.array_equal(u64(r.final_remainder), rk)
    assert st == src.state


def test_roll_batches_invalid_bounds(B, O):
    ds = B.DeviceStream(3)
    st0 = ds.host_state()
    bounds = np.full(2 * 1000, 6, dtype=np.uint32)
    bounds[777] = 0
    with pytest.raises(ValueError):
        B.roll_batches(ds, dev_u32(bounds), 2)
    st1 = ds.host_state()
    assert (st1.state_hi, st1.state_lo) == (st0.state_hi, st0.state_lo)
    bounds = np.full(3 * 100, 1 << 22, dtype=np.uint32)
    with pytest.raises(B.BoundOverflow):
        B.roll_batches(ds, dev_u32(bounds), 3)
    # the workspace is clean again afterwards
    r = B.roll_batches(ds, dev_u32(np.full(2 * 10, 6, dtype=np.uint32)), 2)
    assert r.words.cpu().numpy().tolist() == [1] * 10


def test_roll_batch_dropin_golden(B, golden):
    for rec in golden["roll_batch"]:
        s = B.Pcg64Source(rec["seed"])
        spec = B.BatchSpec(B.RadixBases.of(rec["bases"]))
        for digits, words, tc, rk in rec["results"][:8]:
            r = B.roll_batch(s, spec)
            assert (list(r.digits), r.words_consumed, int(r.threshold_computed), r.final_remainder) == (
                digits, words, tc, rk)
        rest = rec["results"][8:]
        k = len(rec["bases"])
        res = B.roll_batches(s, dev_u32(np.tile(np.asarray(rec["bases"], dtype=np.uint32), len(rest))), k,
                             flags=True, final_remainder=True)
        assert u32(res.rolls).reshape(-1, k).tolist() == [x[0] for x in rest]
        assert res.words.cpu().tolist() == [x[1] for x in rest]
        assert res.flags.cpu().tolist() == [x[2] for x in rest]
        assert u64(res.final_remainder).tolist() == [x[3] for x in rest]
        assert s.state == rec["state_after"]


def test_roll_batch_known_threshold(B, O):
    """batched.py:85-99 against the oracle's restatement (or_roll_batch_known_threshold), on
    streams that include rejected words (products near 2^64) and k > 8 bases."""
    cases = [(52, 51), (6,) * 6, (0xFFFFFFFF, 3006477107), (3,) * 40, ((1 << 40) + 7,), (1 << 31, 1 << 31, 4)]
    a, o = B.Pcg64Source(5), O.pcg64(5)
    seen_reject = False
    for rep in range(40):
        for bases in cases:
            spec = B.BatchSpec.with_threshold(B.RadixBases.of(bases))
            r = B.roll_batch_known_threshold(a, spec)
            ref = O.roll_batch_known_threshold(o, bases)
            assert (tuple(r.digits), r.words_consumed, r.threshold_computed, r.final_remainder) == ref, (rep, bases)
            seen_reject |= r.words_consumed > 1
    assert a.state == o.state and seen_reject
    with pytest.raises(ValueError):
        B.roll_batch_known_threshold(a, B.BatchSpec(B.RadixBases.of((52, 51))))


def test_roll_batch_words_beyond_255(B, O):
    """A FixedSequenceSource whose first 300 words are all rejected: words_consumed is exact
    (not the saturating u8 counter of the bulk kernel)."""
    bases = (0xFFFFFFFF, 3006477107)
    words = [0] * 300 + [2**64 - 1, 12345]
    s = B.FixedSequenceSource(words)
    r = B.roll_batch(s, B.BatchSpec(B.RadixBases.of(bases)))
    ref = O.roll_batch(O.fixed(words), bases)
    assert (tuple(r.digits), r.words_consumed, r.threshold_computed, r.final_remainder) == ref
    assert r.words_consumed == 301 and s.cursor == 301


def test_digit_pass_vs_oracle(B, O, golden):
    for rec in golden["digit_pass"][:40]:
        if max(rec["bases"]) < 1 << 32:
            assert B.digit_pass(rec["r0"], B.RadixBases.of(rec["bases"])) == (tuple(rec["digits"]), rec["rk"])
    rng = np.random.default_rng(3)
    n, k = 1 << 20, 4
    words = rng.integers(0, 2**63, n, dtype=np.int64)
    bounds = rng.integers(1, 1 << 16, n * k, dtype=np.uint32)
    d, rk = B.digit_pass_many(torch.from_numpy(words).cuda(), dev_u32(bounds), k)
    d = u32(d).reshape(n, k)
    rk = u64(rk)
    # Theorem 1 reconstruction (test_acceptance.py:72-99): encode(digits)*2^64 + rk == prod*r0
    for i in rng.integers(0, n, 2000):
        bs = [int(x) for x in bounds[i * k:(i + 1) * k]]
        enc = 0
        for dig, base in zip(d[i].tolist(), bs):
            enc = enc * base + dig
        prod = bs[0] * bs[1] * bs[2] * bs[3]
        assert enc * (1 << 64) + int(rk[i]) == prod * int(words[i])


# ------------------------------------------------------------------ segmented shuffles
def test_c3_every_array(B, O, golden, golden_arrays):
    n, na = 64, 1 << 20
    data = torch.arange(n, dtype=torch.int32, device="cuda").repeat(na)
    _, words = B.shuffle_many(data, n, 1234, return_words=True)
    assert "shuffle_small" in B.last_kernel()
    got = u32(data)
    ref = np.tile(np.arange(n, dtype=np.uint32), na)
    ref_words = O.shuffle_segmented(ref, n, 1234)
    assert np.array_equal(got, ref)
    assert np.array_equal(u32(words), ref_words)
    assert np.array_equal(got[: 256 * 64].reshape(256, 64), golden_arrays["c3_perm_first256"].astype(np.uint32))
    for rec in golden["c3_high"]:
        assert got[rec["a"] * 64:(rec["a"] + 1) * 64].tolist() == rec["perm"]


def test_c4_sample(B, O, golden):
    n, na = 4096, 1 << 16
    data = torch.arange(n, dtype=torch.int32, device="cuda").repeat(na)
    _, words = B.shuffle_many(data, n, 99, return_words=True)
    assert "shuffle_idx_kernel" in B.last_kernel()
    got = u32(data).reshape(na, n)
    w = u32(words)
    for rec in golden["c4"]:
        assert sha_u32(got[rec["a"]]) == rec["sha"] and int(w[rec["a"]]) == rec["words"]
    rng = np.random.default_rng(4)
    for start in rng.integers(0, na - 256, 8):
        ref = np.tile(np.arange(n, dtype=np.uint32), 256)
        rw = O.shuffle_segmented(ref, n, 99, array_index_base=int(start))
        assert np.array_equal(got[start:start + 256].reshape(-1), ref)
        assert np.array_equal(w[start:start + 256], rw)
    # every array is a permutation
    assert np.array_equal(np.sort(got[::97], axis=1), np.tile(np.arange(n, dtype=np.uint32), (len(got[::97]), 1)))


KERNEL_CASES = {  # forced kernel -> (name in last_kernel, lengths it can take)
    "small": ("shuffle_small", (2, 5, 33, 64, 100)),
    "resolve": ("shuffle_resolve_kernel", (2, 3, 64, 100, 1000, 4096, 4097, 10000)),
    "hash": ("shuffle_cta_hash_kernel", (2, 64, 1000, 4096, 10000, 20000)),
    "mid": ("shuffle_mid_kernel", (2, 64, 1000, 4096, 10000)),
    "large": ("shuffle_cta_large_kernel", (2, 64, 1000, 4096, 70000)),
    "global": ("shuffle_large_gen_kernel", (2, 64, 1000, 4096, 70000)),
    "warp": ("shuffle_warp_kernel", (2, 33, 64, 1000, 4096, 6000, 12000)),
    "idx": ("shuffle_idx_kernel", (2, 33, 64, 65, 127, 1000, 4096, 4097, 6000, 12000)),
}


@pytest.mark.parametrize("kernel", sorted(KERNEL_CASES))
@pytest.mark.parametrize("gen", ["pcg64", "chacha"])
def test_every_shuffle_kernel(B, O, monkeypatch, kernel, gen):
    """Each shuffle kernel (forced through BR_SHUFFLE_KERNEL) against the oracle, segmented and
    stream form, u32 and u64, default and naive plans."""
    monkeypatch.setenv("BR_SHUFFLE_KERNEL", kernel)
    name, lengths = KERNEL_CASES[kernel]
    for n in lengths:
        for eb in (4, 8):
            if kernel == "mid" and n * eb + n > 200 * 1024:
                continue
            na = max(2, min(64, (1 << 19) // n))
            dt = np.uint32 if eb == 4 else np.uint64
            payload = np.arange(n * na, dtype=dt)
            for naive in (False, True):
                dev = torch.from_numpy(payload.view(np.int32 if eb == 4 else np.int64).copy()).cuda()
                _, w = B.shuffle_many(dev, n, 4321, array_index_base=17, return_words=True, generator=gen,
                                      naive=naive)
                kern = B.last_kernel()
                ref = payload.copy()
                if naive:
                    rw = O.shuffle_naive_segmented(ref, n, 4321, array_index_base=17, generator=gen)
                else:
                    rw = O.shuffle_segmented(ref, n, 4321, array_index_base=17, generator=gen)
                assert np.array_equal(dev.cpu().numpy().view(dt), ref), (kernel, n, eb, naive, kern)
                assert np.array_equal(u32(w), rw)
                if n > 2 and not (kernel == "small" and eb == 8 and n >= 64) and not (kernel.startswith("warp") and n * eb > 48 * 1024):
                    assert name in kern, (kernel, n, eb, kern)
        if kernel != "small":  # stream form (one array from a caller's source)
            s = B.make_source(gen, 900 + n)
            z = torch.arange(n, dtype=torch.int32, device="cuda")
            B.shuffle_batched(s, z)
            o = O.GENERATOR_MAKERS[gen](900 + n)
            zr = O.shuffle_batched(o, np.arange(n, dtype=np.uint32))
            assert np.array_equal(u32(z), zr), (kernel, n, B.last_kernel())


DISPATCH = [  # (n, item bytes, arrays, kernel the default dispatch picks)
    (64, 4, 2048, "shuffle_small_idx_kernel"),
    (1000, 4, 2048, "shuffle_warp_kernel"),
    (2048, 4, 2048, "shuffle_warp_kernel"),
    (4096, 4, 4096, "shuffle_idx_kernel"),
    (4096, 8, 2048, "shuffle_idx_kernel"),
    (8192, 4, 1024, "shuffle_idx_kernel"),
    (12000, 4, 512, "shuffle_cta_hash_kernel"),
    (20000, 4, 256, "shuffle_cta_hash_kernel"),
    (70000, 8, 8, "shuffle_stage_kernel"),
    (300001, 4, 4, "shuffle_stage_kernel"),
]


@pytest.mark.parametrize("n,eb,na,kernel", DISPATCH)
def test_default_dispatch(B, O, n, eb, na, kernel):
    """The size-based kernel choice (measured crossovers) and its result on sampled arrays."""
    dt = np.uint32 if eb == 4 else np.uint64
    payload = np.arange(n * na, dtype=dt)
    dev = torch.from_numpy(payload.view(np.int32 if eb == 4 else np.int64).copy()).cuda()
    _, w = B.shuffle_many(dev, n, 606, array_index_base=9, return_words=True)
    assert kernel in B.last_kernel(), (n, eb, B.last_kernel())
    got = dev.cpu().numpy().view(dt).reshape(na, n)
    for a in (0, na // 2, na - 1):
        ref = np.arange(a * n, (a + 1) * n, dtype=dt)
        rw = O.shuffle_segmented(ref, n, 606, array_index_base=9 + a)
        assert np.array_equal(got[a], ref) and int(u32(w)[a]) == int(rw[0]), (n, eb, a)


def test_idx_staging_queue_under_pressure(B, O, monkeypatch):
    """The index kernel's staging hand-off with its queues saturated: the holder of buffer 0 sleeps
    (BR_IDX_HOLD_US), so nearly every warp of a CTA ends up waiting on that one buffer.  A single
    ring of 32 ticket slots over both buffers let a second warp into a held buffer here."""
    monkeypatch.setenv("BR_SHUFFLE_KERNEL", "idx")
    monkeypatch.setenv("BR_IDX_HOLD_US", "40")
    n, na = 2048, 148 * 24 * 5
    dev = torch.arange(n, dtype=torch.int32, device="cuda").repeat(na)
    B.shuffle_many(dev, n, 31337, array_index_base=1)
    torch.cuda.synchronize()
    assert "shuffle_idx_kernel" in B.last_kernel()
    got = u32(dev).reshape(na, n)
    assert np.array_equal(np.sort(got, axis=1), np.tile(np.arange(n, dtype=np.uint32), (na, 1)))
    for a in list(range(0, na, 997)) + [na - 1]:
        ref = np.arange(n, dtype=np.uint32)
        O.shuffle_segmented(ref, n, 31337, array_index_base=1 + a)
        assert np.array_equal(got[a], ref), a


@pytest.mark.parametrize("kernel", ["idx", "warp", "hash", "small", "large"])
def test_unaligned_payload(B, O, monkeypatch, kernel):
    """Payload starting 4 bytes past a 16-byte boundary: the kernels fall back from bulk (TMA)
    copies and 16-byte stores to element copies; results unchanged."""
    monkeypatch.setenv("BR_SHUFFLE_KERNEL", kernel)
    for n in ((64, 100) if kernel == "small" else (1000, 4096)):
        na = 40 if kernel == "small" else 24  # a full warp of arrays: the 8-byte vector path must step aside
        payload = np.arange(n * na, dtype=np.uint32) ^ 0x5A5A
        big = torch.zeros(n * na + 4, dtype=torch.int32, device="cuda")
        big[1:1 + n * na] = torch.from_numpy(payload.view(np.int32).copy()).cuda()
        view = big[1:1 + n * na]
        assert view.data_ptr() % 16 == 4
        B.shuffle_many(view, n, 99, array_index_base=3)
        ref = payload.copy()
        O.shuffle_segmented(ref, n, 99, array_index_base=3)
        assert np.array_equal(view.cpu().numpy().view(np.uint32), ref), (kernel, n, B.last_kernel())
        assert int(big[0]) == 0 and int(big[-1]) == 0 and int(big[-2]) == 0 and int(big[-3]) == 0


@pytest.mark.parametrize("kernel", ["idx", "warp", "hash", "small"])
def test_lehmer_segmented_kernels(B, O, monkeypatch, kernel):
    """Lehmer128 streams (increment 0) through the shared-memory shuffle kernels, u32 and u64,
    including partial last groups and arrays whose index permutation spans every group."""
    monkeypatch.setenv("BR_SHUFFLE_KERNEL", kernel)
    for n in ((33, 100, 127) if kernel == "small" else (33, 1000, 4096, 5003)):
        for eb in (4, 8):
            na = max(2, min(40, (1 << 18) // n))
            dt = np.uint32 if eb == 4 else np.uint64
            payload = np.arange(n * na, dtype=dt) * 3 + 1
            dev = torch.from_numpy(payload.view(np.int32 if eb == 4 else np.int64).copy()).cuda()
            _, w = B.shuffle_many(dev, n, 2718, array_index_base=5, return_words=True, generator="lehmer")
            ref = payload.copy()
            rw = O.shuffle_segmented(ref, n, 2718, array_index_base=5, generator="lehmer")
            assert np.array_equal(dev.cpu().numpy().view(dt), ref), (kernel, n, eb, B.last_kernel())
            assert np.array_equal(u32(w), rw), (kernel, n, eb)


@pytest.mark.parametrize("eb", [4, 8])
@pytest.mark.parametrize("n", [2, 3, 5, 7, 8, 9, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129, 255, 256, 257, 511,
                               512, 513, 1000, 2047, 2048, 2049, 4095, 4097, 10000, 16384])
def test_shuffle_many_lengths_and_payloads(B, O, n, eb):
    na = max(2, min(3000, (1 << 21) // n))
    rng = np.random.default_rng(n * 10 + eb)
    dt = np.uint32 if eb == 4 else np.uint64
    payload = rng.integers(0, np.iinfo(dt).max, na * n, dtype=dt)
    dev = torch.from_numpy(payload.view(np.int32 if eb == 4 else np.int64).copy()).cuda()
    _, words = B.shuffle_many(dev, n, 777, array_index_base=123, return_words=True)
    ref = payload.copy()
    rw = O.shuffle_segmented(ref, n, 777, array_index_base=123)
    got = dev.cpu().numpy().view(dt)
    assert np.array_equal(got, ref), (n, eb, B.last_kernel())
    assert np.array_equal(u32(words), rw)


def test_shuffle_many_custom_schedules(B, O, golden):
    for name in ("pair", "max3", "head", "wide"):
        entries = [tuple(e) for e in golden["schedules"][name]["entries"]]
        sched = B.ShuffleSchedule(tuple(entries), golden["schedules"][name]["max_batch"])
        for n in (5, 64, 300, 1000, 4097):
            na = 64
            data = torch.arange(n, dtype=torch.int32, device="cuda").repeat(na)
            B.shuffle_many(data, n, 5, schedule=sched)
            ref = np.tile(np.arange(n, dtype=np.uint32), na)
            from oracle import shuffle_segmented

            shuffle_segmented(ref, n, 5, entries=entries)
            assert np.array_equal(u32(data), ref), (name, n)


# ------------------------------------------------------------------ single stream / drop-in
def test_c1_stream_golden(B, golden, golden_arrays):
    s = B.Pcg64Source(42)
    z = np.arange(10000, dtype=np.uint32)
    B.shuffle_batched(s, z)
    assert np.array_equal(z, golden_arrays["c1_batched"])
    o = B.Pcg64Source(42)
    o.advance(golden["c1"]["batched"]["words"])
    assert s.state == o.state
    s = B.Pcg64Source(42)
    z = np.arange(10000, dtype=np.uint32)
    B.shuffle_unbatched(s, z)
    assert np.array_equal(z, golden_arrays["c1_unbatched"])
    o = B.Pcg64Source(42)
    o.advance(9999)
    assert s.state == o.state


def test_dropin_shuffle_batched_golden(B, golden):
    scheds = {k: B.ShuffleSchedule(tuple(tuple(e) for e in v["entries"]), v["max_batch"])
              for k, v in golden["schedules"].items()}
    for rec in golden["shuffle_batched"]:
        s = B.Pcg64Source(rec["seed"])
        z = list(range(rec["n"]))
        out = B.shuffle_batched(s, z, scheds[rec["schedule"]])
        assert out is z
        assert sha_u32(z) == rec["sha"], rec["n"]
        o = B.Pcg64Source(rec["seed"])
        o.advance(rec["words"])
        assert s.state == o.state


def test_dropin_unbatched_golden(B, golden):
    for rec in golden["shuffle_unbatched"]:
        s = B.Pcg64Source(rec["seed"])
        z = B.shuffle_unbatched(s, list(range(rec["n"])))
        assert sha_u32(z) == rec["sha"]


def test_partial_shuffle_batch_golden(B, golden):
    for rec in golden["partial_shuffle_batch"]:
        s = B.Pcg64Source(rec["seed"])
        z = list(range(rec["n"]))
        u = B.partial_shuffle_batch(s, z, rec["n"], rec["k"], rec["u_in"])
        assert z == rec["perm"] and u == rec["u_out"]


def test_dropin_payload_types(B, O):
    s1, s2, s3 = B.Pcg64Source(9), B.Pcg64Source(9), B.Pcg64Source(9)
    objs = [f"item{i}" for i in range(777)]
    a = B.shuffle_batched(s1, list(objs))
    b = B.shuffle_batched(s2, np.arange(777, dtype=np.uint64))
    c = B.shuffle_batched(s3, torch.arange(777, dtype=torch.int32, device="cuda"))
    assert a == [objs[i] for i in b.tolist()]
    assert c.cpu().tolist() == b.tolist()
    assert s1.state == s2.state == s3.state
    ref = O.shuffle_batched(O.pcg64(9), np.arange(777, dtype=np.uint32))
    assert b.tolist() == ref.tolist()
    # multiset preservation with duplicates (test_shuffle.py:248-257)
    d = [3, 1, 3, 3, 7, 1] * 50
    out = B.shuffle_batched(B.Pcg64Source(1), list(d))
    assert sorted(out) == sorted(d)


def test_dropin_accepts_reference_style_source(B, O):
    class RefLike:  # duck-typed like the reference Pcg64Source
        word_bits = 64

        def __init__(self, seed):
            o = O.pcg64(seed)
            self.state, self.increment = o.state, o.increment

    s = RefLike(31)
    z = B.shuffle_batched(s, list(range(1000)))
    o = O.pcg64(31)
    assert z == O.shuffle_batched(o, np.arange(1000, dtype=np.uint32)).tolist()
    assert s.state == o.state
    with pytest.raises(TypeError):
        class Mystery:  # neither a PCG64 (state+increment) nor a Lehmer source
            word_bits = 64
            state = 5

        B.shuffle_batched(Mystery(), list(range(10)))


def test_short_arrays_finish_in_one_batch(B):
    # test_shuffle.py:223-235: n=5 under the default schedule is one batch of four dice
    for seed in range(20):
        s = B.Pcg64Source(seed)
        z = B.shuffle_batched(s, list(range(5)))
        o = B.Pcg64Source(seed)
        o.advance(1)
        assert s.state == o.state and sorted(z) == list(range(5))


def test_native_library_is_the_one_loaded(B):
    import paper_2408_06213_b200._native as N

    maps = open("/proc/self/maps").read()
    assert N.LIB_PATH in maps


# ------------------------------------------------------------------ large arrays (global-memory path)
def test_c5_sample_vs_golden_and_oracle(B, O, golden):
    n, na = 1 << 20, 8
    payload = O.pcg64_fill(O.pcg64(5), 0, n * na)  # C5 payload convention: words of pcg64(5)
    dev = torch.from_numpy(payload.view(np.int64).copy()).cuda()
    _, words = B.shuffle_many(dev, n, 5, return_words=True)
    assert "shuffle_stage_kernel" in B.last_kernel()
    got = dev.cpu().numpy().view(np.uint64)
    ref = payload.copy()
    rw = O.shuffle_segmented(ref, n, 5)
    assert np.array_equal(got, ref)
    assert np.array_equal(u32(words), rw)
    # golden (reference-run) index permutations of arrays 0 and 255
    for rec in golden["c5"]:
        idx = torch.arange(n, dtype=torch.int32, device="cuda")
        _, w = B.shuffle_many(idx, n, 5, array_index_base=rec["a"], return_words=True)
        assert sha_u32(u32(idx)) == rec["sha"] and int(u32(w)[0]) == rec["words"]


@pytest.mark.parametrize("n", [16385, 20000, 65536, 100003, 1 << 18])
def test_large_stream_and_segmented_vs_oracle(B, O, n):
    s = B.Pcg64Source(n)
    z = np.arange(n, dtype=np.uint32)
    B.shuffle_batched(s, z)
    o = O.pcg64(n)
    ref = O.shuffle_batched(o, np.arange(n, dtype=np.uint32))
    assert np.array_equal(z, ref) and s.state == o.state
    s = B.Pcg64Source(n + 1)
    z = np.arange(n, dtype=np.uint64)
    B.shuffle_unbatched(s, z)
    o = O.pcg64(n + 1)
    assert np.array_equal(z, O.shuffle_unbatched(o, np.arange(n, dtype=np.uint64))) and s.state == o.state
    data = torch.arange(n, dtype=torch.int32, device="cuda").repeat(3)
    _, w = B.shuffle_many(data, n, 11, array_index_base=7, return_words=True)
    ref = np.tile(np.arange(n, dtype=np.uint32), 3)
    rw = O.shuffle_segmented(ref, n, 11, array_index_base=7)
    assert np.array_equal(u32(data), ref) and np.array_equal(u32(w), rw)


def test_roll_single_dropin(B, O):  # bounded.py:73-104 via the k=1 batch kernel
    for seed, bound in ((1, 6), (2, 52), (3, (1 << 32) - 1), (4, 3 << 30), (5, 1)):
        s, o = B.Pcg64Source(seed), O.pcg64(seed)
        for _ in range(20):
            v, w, ro = O.roll_single(o, bound)
            r = B.roll_single_traced(s, bound)
            assert (r.value, r.words_consumed, r.remainder_ops) == (v, w, ro)
        assert s.state == o.state
    with pytest.raises(B.BoundOverflow):
        B.roll_single(B.Pcg64Source(1), 0)


# ------------------------------------------------------------------ Lehmer128
def test_lehmer_fill_and_dropin_shuffles(B, O, golden):
    got = u64(B.pcg64_fill(77, 5000, 123, generator="lehmer"))
    o = O.lehmer(77)
    O.words(o, 123)
    assert got.tolist() == O.words(o, 5000)
    scheds = {k: B.ShuffleSchedule(tuple(tuple(e) for e in v["entries"]), v["max_batch"])
              for k, v in golden["schedules"].items()}
    for rec in golden["shuffle_batched_lehmer"]:
        s = B.LehmerSource(rec["seed"])
        z = np.arange(rec["n"], dtype=np.uint32)
        B.shuffle_batched(s, z, scheds[rec["schedule"]])
        o = O.lehmer(rec["seed"])
        O.shuffle_batched(o, np.arange(rec["n"], dtype=np.uint32), [tuple(e) for e in golden["schedules"][rec["schedule"]]["entries"]])
        assert sha_u32(z) == rec["sha"] and s.state == o.state, rec["n"]
    for rec in golden["shuffle_unbatched_lehmer"]:
        s = B.LehmerSource(rec["seed"])
        z = B.shuffle_unbatched(s, list(range(rec["n"])))
        assert sha_u32(z) == rec["sha"]
    # test_shuffle.py:154-161 word budget on the reference's own Lehmer seed
    s = B.LehmerSource(31337)
    B.shuffle_batched(s, list(range(1000)))
    o = O.lehmer(31337)
    O.words(o, golden["lehmer_31337_n1000_words"])
    assert s.state == o.state


@pytest.mark.parametrize("n,eb", [(64, 4), (100, 8), (4096, 4), (20000, 8), (70000, 4)])
def test_lehmer_segmented(B, O, n, eb):
    na = max(2, min(500, (1 << 20) // n))
    dt = np.uint32 if eb == 4 else np.uint64
    payload = np.arange(n * na, dtype=dt)
    dev = torch.from_numpy(payload.view(np.int32 if eb == 4 else np.int64).copy()).cuda()
    _, w = B.shuffle_many(dev, n, 4242, array_index_base=9, return_words=True, generator="lehmer")
    ref = payload.copy()
    rw = O.shuffle_segmented(ref, n, 4242, array_index_base=9, generator="lehmer")
    assert np.array_equal(dev.cpu().numpy().view(dt), ref), B.last_kernel()
    assert np.array_equal(u32(w), rw)


def test_lehmer_rolls(B, O, golden):
    for rec in golden["roll_batch_lehmer"]:
        s = B.LehmerSource(rec["seed"])
        k = len(rec["bases"])
        res = B.roll_batches(s, dev_u32(np.tile(np.asarray(rec["bases"], dtype=np.uint32), len(rec["results"]))), k,
                             flags=True, final_remainder=True)
        assert u32(res.rolls).reshape(-1, k).tolist() == [x[0] for x in rec["results"]]
        assert res.words.cpu().tolist() == [x[1] for x in rec["results"]]
        assert u64(res.final_remainder).tolist() == [x[3] for x in rec["results"]]
        assert s.state == rec["state_after"]
    nb = 300000
    bounds = O.gen_bounds(8, 2 * nb)
    bounds[:1000:2] = 0xFFFFFFFF
    bounds[1:1000:2] = 3006477107
    src = O.lehmer(5)
    rolls, words, _, _ = O.roll_batches(src, bounds, 2)
    ds = B.DeviceStream(5, generator="lehmer")
    r = B.roll_batches(ds, dev_u32(bounds), 2)
    st = ds.host_state()
    assert np.array_equal(u32(r.rolls), rolls) and np.array_equal(r.words.cpu().numpy(), words)
    assert (st.state_hi << 64 | st.state_lo) == src.state


# ------------------------------------------------------------------ ChaCha20
def test_chacha_fill(B, O):
    for seed, offset, count in ((0, 0, 1), (3, 5, 20), (77, 123, 50001), (9, (1 << 40) + 3, 4096)):
        got = u64(B.pcg64_fill(seed, count, offset, generator="chacha"))
        assert np.array_equal(got, O.pcg64_fill(O.chacha(seed), offset, count)), (seed, offset)
    assert "cha_fill_kernel" in B.last_kernel()
    s = B.ChaChaSource(77)
    [s.next_word() for _ in range(5)]  # mid-block source: fill starts at its position
    o = O.chacha(77)
    O.words(o, 5)
    assert u64(B.pcg64_fill(s, 30)).tolist() == O.words(o, 30)


def test_chacha_dropin_shuffles_golden(B, O, golden):
    scheds = {k: B.ShuffleSchedule(tuple(tuple(e) for e in v["entries"]), v["max_batch"])
              for k, v in golden["schedules"].items()}
    for rec in golden["shuffle_batched_chacha"]:
        s = B.make_source("chacha", rec["seed"])
        for _ in range(rec["pre"]):
            s.next_word()
        z = np.arange(rec["n"], dtype=np.uint32)
        B.shuffle_batched(s, z, scheds[rec["schedule"]])
        assert sha_u32(z) == rec["sha"], (rec["n"], rec["schedule"], B.last_kernel())
        assert (s.counter, s._pos) == (rec["counter_after"], rec["pos_after"])
        if s._pos < 16:  # the refilled buffer is the block the reference would hold
            o = O.chacha(rec["seed"])
            O.words(o, rec["pre"] + rec["words"])
            assert s._buffer == list(o.buf)
    for rec in golden["shuffle_unbatched_chacha"]:
        s = B.ChaChaSource(rec["seed"])
        z = B.shuffle_unbatched(s, list(range(rec["n"])))
        assert sha_u32(z) == rec["sha"]


def test_chacha_counter_wrap(B, O):
    """A ChaCha source two blocks before its 64-bit block counter wraps (wordsource.py:160
    masks the counter): words, shuffles and rolls cross the wrap like the reference."""
    for pre, n in ((0, 1000), (5, 1000), (3, 70000)):
        s = B.ChaChaSource(77)
        s.counter, s._pos = (1 << 64) - 2, 16
        o = O.chacha(77)
        o.counter, o.pos = (1 << 64) - 2, 16
        for _ in range(pre):
            assert s.next_word() == O.next_word(o)
        z = torch.arange(n, dtype=torch.int32, device="cuda")
        B.shuffle_batched(s, z)
        zr = O.shuffle_batched(o, np.arange(n, dtype=np.uint32))
        assert np.array_equal(u32(z), zr) and (s.counter, s._pos) == (o.counter, o.pos), (pre, n, B.last_kernel())
        assert s.counter < 1 << 20  # wrapped
        assert [s.next_word() for _ in range(9)] == O.words(o, 9)
    s = B.ChaChaSource(9)
    s.counter, s._pos = (1 << 64) - 1, 16
    o = O.chacha(9)
    o.counter, o.pos = (1 << 64) - 1, 16
    bounds = O.gen_bounds(3, 2 * 5000)
    r = B.roll_batches(s, dev_u32(bounds), 2)
    rolls, words, _, _ = O.roll_batches(o, bounds, 2)
    assert np.array_equal(u32(r.rolls), rolls) and (s.counter, s._pos) == (o.counter, o.pos)
    assert u64(B.pcg64_fill(s, 20)).tolist() == O.words(o, 20)


@pytest.mark.parametrize("n,eb", [(64, 4), (100, 8), (4096, 4), (20000, 8), (70000, 4), (1 << 20, 8)])
def test_chacha_segmented(B, O, n, eb):
    na = max(2, min(400, (1 << 20) // n))
    dt = np.uint32 if eb == 4 else np.uint64
    payload = np.arange(n * na, dtype=dt)
    dev = torch.from_numpy(payload.view(np.int32 if eb == 4 else np.int64).copy()).cuda()
    _, w = B.shuffle_many(dev, n, 777, array_index_base=3, return_words=True, generator="chacha")
    ref = payload.copy()
    rw = O.shuffle_segmented(ref, n, 777, array_index_base=3, generator="chacha")
    assert np.array_equal(dev.cpu().numpy().view(dt), ref), B.last_kernel()
    assert np.array_equal(u32(w), rw)


@pytest.mark.parametrize("n", [1000, 70000])
def test_chacha_wide_schedule_paths(B, O, n):
    """k = 16 in the tail regime: n=1000 runs in the warp kernel and n=70000 in
    the global-target fallback, in both the segmented and the stream form."""
    entries = ((1 << 30, 2), (17, 16))
    sched = B.ShuffleSchedule(entries, 16)
    na = 6
    payload = np.arange(n * na, dtype=np.uint32)
    dev = torch.from_numpy(payload.view(np.int32).copy()).cuda()
    B.shuffle_many(dev, n, 31, schedule=sched, generator="chacha")
    kern = B.last_kernel()
    ref = payload.copy()
    O.shuffle_segmented(ref, n, 31, entries=list(entries), generator="chacha")
    assert np.array_equal(u32(dev), ref), kern
    assert ("mid" in kern) if n == 1000 else ("large_gen" in kern)
    s = B.ChaChaSource(55)
    z = torch.arange(n, dtype=torch.int32, device="cuda")
    B.shuffle_batched(s, z, sched)
    o = O.chacha(55)
    zr = O.shuffle_batched(o, np.arange(n, dtype=np.uint32), list(entries))
    assert np.array_equal(u32(z), zr) and (s.counter, s._pos) == (o.counter, o.pos)


def test_chacha_rolls(B, O, golden):
    for rec in golden["roll_batch_chacha"]:
        s = B.ChaChaSource(rec["seed"])
        k = len(rec["bases"])
        res = B.roll_batches(s, dev_u32(np.tile(np.asarray(rec["bases"], dtype=np.uint32), len(rec["results"]))), k,
                             flags=True, final_remainder=True)
        assert u32(res.rolls).reshape(-1, k).tolist() == [x[0] for x in rec["results"]]
        assert res.words.cpu().tolist() == [x[1] for x in rec["results"]]
        assert res.flags.cpu().tolist() == [x[2] for x in rec["results"]]
        assert u64(res.final_remainder).tolist() == [x[3] for x in rec["results"]]
        assert (s.counter, s._pos) == (rec["counter_after"], rec["pos_after"])
    for k, nb in ((2, 300000), (1, 100003), (3, 50001)):
        bounds = O.gen_bounds(8, k * nb)
        if k == 2:  # products near 2^64: rejections at the head of the run
            bounds[:1000:2] = 0xFFFFFFFF
            bounds[1:1000:2] = 3006477107
        src = O.chacha(5)
        rolls, words, flags, rk = O.roll_batches(src, bounds, k)
        ds = B.DeviceStream(5, generator="chacha")
        r = B.roll_batches(ds, dev_u32(bounds), k, flags=True, final_remainder=True)
        st = ds.host_state()
        assert np.array_equal(u32(r.rolls), rolls) and np.array_equal(r.words.cpu().numpy(), words), k
        assert np.array_equal(r.flags.cpu().numpy(), flags) and np.array_equal(u64(r.final_remainder), rk)
        assert (st.state_hi << 64 | st.state_lo) == O.chacha_position(src)
        if k == 2:
            assert int(words.sum()) > nb  # the forced rejections happened


def test_roll_kernel_choice_is_only_a_hint(B, O):
    """The host picks the main roll kernel from the kind recorded at br_state_upload; a state
    written behind its back (stale or unknown kind) is still rolled exactly by the fixup."""
    nb, k = 70001, 2
    bounds = O.gen_bounds(12, k * nb)
    db = dev_u32(bounds)
    for first, second in (("chacha", "pcg64"), ("pcg64", "chacha"), ("lehmer", "chacha")):
        ds = B.DeviceStream(3, generator=first)  # kind recorded for ds.state: `first`
        other = B.DeviceStream(4, generator=second)
        ds.state.copy_(other.state)  # now holds a `second` stream; the record still says `first`
        src = O.GENERATOR_MAKERS[second](4)
        rolls, words, _, _ = O.roll_batches(src, bounds, k)
        r = B.roll_batches(ds, db, k)
        st = ds.host_state()
        assert np.array_equal(u32(r.rolls), rolls) and np.array_equal(r.words.cpu().numpy(), words), (first, second)
        pos = (st.state_hi << 64) | st.state_lo
        assert pos == (O.chacha_position(src) if second == "chacha" else src.state)
    # an unrecorded buffer (a clone) takes the default guess and the same fallback
    ds = B.DeviceStream(8, generator="chacha")
    ds.state = ds.state.clone()
    src = O.chacha(8)
    rolls, words, _, _ = O.roll_batches(src, bounds, k)
    r = B.roll_batches(ds, db, k)
    assert np.array_equal(u32(r.rolls), rolls)
    ds = B.DeviceStream(8, generator="chacha")
    B.roll_batches(ds, db, k)
    assert "roll_cha_kernel" in B.last_kernel()


# ------------------------------------------------------------------ division-based baselines (8(f) row 3)
def test_naive_shuffle_dropin_golden(B, O, golden):
    for rec in golden["shuffle_naive_batched"]:
        s = B.make_source(rec["gen"], rec["seed"])
        z = B.shuffle_naive_batched(s, list(range(rec["n"])))
        assert sha_u32(z) == rec["sha"], (rec["gen"], rec["n"], B.last_kernel())
        o = O.GENERATOR_MAKERS[rec["gen"]](rec["seed"])
        O.words(o, rec["words"])
        if rec["gen"] == "chacha":
            assert B.batchrand._chacha_position(s) == O.chacha_position(o)
        else:
            assert s.state == o.state
    with pytest.raises(B.BoundOverflow):
        class Narrow:
            word_bits = 8
        B.shuffle_naive_batched(Narrow(), list(range(17)))


@pytest.mark.parametrize("gen", ["pcg64", "chacha"])
@pytest.mark.parametrize("n,eb", [(64, 4), (101, 8), (4096, 4), (20001, 8), (70000, 4)])
def test_naive_shuffle_segmented(B, O, gen, n, eb):
    na = max(2, min(300, (1 << 20) // n))
    dt = np.uint32 if eb == 4 else np.uint64
    payload = np.arange(n * na, dtype=dt)
    dev = torch.from_numpy(payload.view(np.int32 if eb == 4 else np.int64).copy()).cuda()
    _, w = B.shuffle_many(dev, n, 2024, array_index_base=5, return_words=True, generator=gen, naive=True)
    ref = payload.copy()
    rw = O.shuffle_naive_segmented(ref, n, 2024, array_index_base=5, generator=gen)
    assert np.array_equal(dev.cpu().numpy().view(dt), ref), B.last_kernel()
    assert np.array_equal(u32(w), rw)


def test_naive_rolls(B, O, golden):
    for rec in golden["roll_batch_naive"]:
        s = B.Pcg64Source(rec["seed"])
        rb = B.RadixBases.of(tuple(rec["bases"]))
        assert [list(B.roll_batch_naive(s, rb)) for _ in range(len(rec["digits"]))] == rec["digits"]
        o = O.pcg64(rec["seed"])
        O.words(o, rec["words"])
        assert s.state == o.state
    for k, nb in ((2, 300000), (3, 50001), (5, 20000)):
        bounds = O.gen_bounds(9, k * nb) if k < 5 else O.gen_bounds(9, k * nb, 2, 4000)
        if k == 2:
            bounds[:1000:2] = 0xFFFFFFFF
            bounds[1:1000:2] = 3006477107
        src = O.pcg64(6)
        rolls, words, flags, rk = O.roll_batches(src, bounds, k)
        ds = B.DeviceStream(6)
        r = B.roll_batches(ds, dev_u32(bounds), k, flags=True, final_remainder=True, naive=True)
        st = ds.host_state()
        assert np.array_equal(u32(r.rolls), rolls) and np.array_equal(r.words.cpu().numpy(), words), k
        assert np.array_equal(r.flags.cpu().numpy(), flags) and np.array_equal(u64(r.final_remainder), rk)
        assert (st.state_hi << 64 | st.state_lo) == src.state


def test_cli_bench_and_shuffle(B, O, tmp_path):
    import io
    import contextlib

    from paper_2408_06213_b200 import cli

    recs = cli.bench("pcg64", (64, 4096), ("shuffle_6_b200", "many_6_b200"), budget_ns=200_000)
    assert [(r[0], r[2]) for r in recs] == [("shuffle_6_b200", 64), ("shuffle_6_b200", 4096),
                                            ("many_6_b200", 64), ("many_6_b200", 4096)]
    assert all(r[3] >= r[4] > 0 for r in recs)
    inp = tmp_path / "lines.txt"
    inp.write_text("\n".join(f"line{i}" for i in range(500)) + "\n")
    out = io.StringIO()
    with contextlib.redirect_stdout(out):
        assert cli.main(["shuffle", str(inp), "--seed", "7"]) == 0
    got = out.getvalue().splitlines()
    perm = O.shuffle_batched(O.pcg64(7), np.arange(500, dtype=np.uint32)).tolist()
    assert got == [f"line{p}" for p in perm]


# ------------------------------------------------------------------ C-ABI argument errors
def test_abi_error_paths(B):
    """Status codes of the device entry points on bad arguments (no launch happens) and the
    edge cases that need no work (n < 2, zero arrays, zero batches)."""
    import ctypes as C

    from paper_2408_06213_b200 import _native as N

    L = N.lib()
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    z = torch.zeros(64, dtype=torch.int32, device="cuda")
    st = torch.zeros(8, dtype=torch.int64, device="cuda")
    w64 = torch.full((1,), 7, dtype=torch.int64, device="cuda")
    zp, stp, wp = (C.c_void_p(t.data_ptr()) for t in (z, st, w64))
    regs = B.DEFAULT_SCHEDULE._regimes()
    assert L.br_shuffle_stream(zp, 2, 64, stp, regs, len(regs), 0, None, sp) == N.BR_E_UNSUPPORTED  # elem size
    # n >= 2^32: the stream form takes it (tests/test_head64.py); the segmented form does not,
    # and the naive form overflows its pair product (shuffle.py:240-241); no launch happens
    assert L.br_shuffle_segmented(zp, 4, 1, 1 << 32, 1, 0, regs, len(regs), 0, None, sp) == N.BR_E_UNSUPPORTED
    assert L.br_shuffle_naive_stream(zp, 4, (1 << 32) + 1, stp, None, sp) == N.BR_E_BOUND_OVERFLOW
    assert L.br_shuffle_stream(None, 4, 64, stp, regs, len(regs), 0, None, sp) == N.BR_E_INVALID
    assert L.br_shuffle_stream(zp, 4, 64, None, regs, len(regs), 0, None, sp) == N.BR_E_INVALID
    assert L.br_shuffle_segmented(zp, 4, 1, 64, 1, 0, regs, len(regs), 3, None, sp) == N.BR_E_UNSUPPORTED  # generator
    assert L.br_shuffle_segmented(zp, 4, -1, 64, 1, 0, regs, len(regs), 0, None, sp) == N.BR_E_INVALID
    bad = (N.Segment * 1)()
    bad[0].start_n, bad[0].k, bad[0].count = 64, 5, 13  # 65 steps on 64 positions
    assert L.br_shuffle_stream_segments(zp, 4, 64, stp, bad, 1, None, None, sp) == N.BR_E_INVALID
    # n < 2: nothing to do, zero words reported, data untouched
    assert L.br_shuffle_stream(zp, 4, 1, stp, regs, len(regs), 0, wp, sp) == N.BR_OK
    assert int(w64.item()) == 0
    assert L.br_shuffle_segmented(zp, 4, 0, 64, 1, 0, regs, len(regs), 0, None, sp) == N.BR_OK
    ws = torch.zeros(L.br_roll_workspace_bytes(), dtype=torch.uint8, device="cuda")
    b = torch.ones(16, dtype=torch.int32, device="cuda")
    r = torch.zeros(16, dtype=torch.int32, device="cuda")
    wd = torch.zeros(16, dtype=torch.uint8, device="cuda")
    bp, rp, wdp, wsp = (C.c_void_p(t.data_ptr()) for t in (b, r, wd, ws))
    assert L.br_roll_batches(bp, 0, 8, stp, rp, wdp, None, None, wsp, sp) == N.BR_E_INVALID  # k < 1
    assert L.br_roll_batches(bp, 9, 1, stp, rp, wdp, None, None, wsp, sp) == N.BR_E_UNSUPPORTED  # k > 8
    assert L.br_roll_batches(bp, 2, -1, stp, rp, wdp, None, None, wsp, sp) == N.BR_E_INVALID
    assert L.br_roll_batches(C.c_void_p(b.data_ptr() + 4), 2, 4, stp, rp, wdp, None, None, wsp, sp) == N.BR_E_INVALID
    assert L.br_roll_batches(bp, 2, 0, stp, rp, wdp, None, None, wsp, sp) == N.BR_OK  # zero batches
    assert L.br_roll_batches_phase(bp, 2, 4, stp, rp, wdp, None, None, wsp, 4, sp) == N.BR_E_INVALID
    assert L.br_pcg64_fill(None, 5, C.byref(N.Pcg64State()), 0, sp) == N.BR_E_INVALID
    assert L.br_state_upload(None, C.byref(N.Pcg64State()), sp) == N.BR_E_INVALID
    assert "null" in N.last_error() or N.last_error()


def test_dropin_edge_cases(B, O):
    """Empty and single-element inputs consume nothing (test_shuffle.py:61-67); k = n batch;
    bounds of 1 (a die with one face) and a product of exactly 2^64."""
    for gen in ("pcg64", "lehmer", "chacha"):
        s = B.make_source(gen, 3)
        before = B.batchrand._state_struct(s)
        assert B.shuffle_batched(s, []) == [] and B.shuffle_unbatched(s, [5]) == [5]
        assert B.shuffle_naive_batched(s, [9]) == [9]
        after = B.batchrand._state_struct(s)
        assert (before.state_hi, before.state_lo) == (after.state_hi, after.state_lo)
    s = B.Pcg64Source(4)
    r = B.roll_batch(s, B.BatchSpec(B.RadixBases.of((1, 1, 1))))
    assert r.digits == (0, 0, 0) and r.words_consumed == 1
    o = O.pcg64(4)
    ro = O.roll_batch(o, (1 << 16, 1 << 16, 1 << 16, 1 << 16))  # product exactly 2^64: never rejected
    s = B.Pcg64Source(4)
    r = B.roll_batch(s, B.BatchSpec(B.RadixBases.of((1 << 16,) * 4)))
    assert r == B.BatchResult(ro[0], ro[1], ro[2], ro[3]) and s.state == o.state


# ------------------------------------------------------------------ replayed word sequences
def test_fixed_sequence_source(B, O):
    """FixedSequenceSource with 64-bit words on the device (wordsource.py:191-207): the
    reference's own cases (test_shuffle.py:70-100), long sequences against the oracle's fixed
    source, cursor accounting, and SourceExhausted on an over-read."""
    z = B.shuffle_unbatched(B.FixedSequenceSource([5], 64), [0, 1])  # test_shuffle.py:68-74
    assert z == [1, 0]
    assert B.shuffle_unbatched(B.FixedSequenceSource([1 << 63], 64), [0, 1]) == [0, 1]
    s = B.FixedSequenceSource([1], 64)  # test_shuffle.py:83-92: k = n = 3 ends with a self-swap
    z = [0, 1, 2]
    assert B.partial_shuffle_batch(s, z, 3, 3, 6) == 6 and z == [1, 2, 0] and s.cursor == 1
    s = B.FixedSequenceSource([(1 << 64) - 1], 64)
    assert B.shuffle_batched(s, [0, 1]) == O.shuffle_batched(O.fixed([(1 << 64) - 1]),
                                                              np.arange(2, dtype=np.uint32)).tolist()
    assert s.cursor == 1
    words = O.pcg64_fill(O.pcg64(99), 0, 5000).tolist()
    for n, sched in ((1000, None), (4000, None), (3000, "pair")):
        s = B.FixedSequenceSource(words, 64)
        s.next_word()  # start one word in
        o = O.fixed(words)
        O.next_word(o)
        entries = [(1 << 30, 2)] if sched == "pair" else None
        z = np.arange(n, dtype=np.uint32)
        if entries:
            B.shuffle_batched(s, z, B.PAIR_SCHEDULE)
            ref = O.shuffle_batched(o, np.arange(n, dtype=np.uint32), entries)
        else:
            B.shuffle_batched(s, z)
            ref = O.shuffle_batched(o, np.arange(n, dtype=np.uint32))
        assert np.array_equal(z, ref) and s.cursor == o.cursor, (n, B.last_kernel())
    # bulk rolls and fill from a replayed sequence
    s = B.FixedSequenceSource(words, 64)
    o = O.fixed(words)
    bounds = O.gen_bounds(4, 2 * 1500)
    r = B.roll_batches(s, dev_u32(bounds), 2)
    rolls, wds, _, _ = O.roll_batches(o, bounds, 2)
    assert np.array_equal(u32(r.rolls), rolls) and s.cursor == o.cursor
    # over-read: SourceExhausted, host payload untouched, cursor at the end (wordsource.py:203-204)
    s = B.FixedSequenceSource(words[:100], 64)
    z = list(range(1000))
    with pytest.raises(B.SourceExhausted):
        B.shuffle_batched(s, z)
    assert z == list(range(1000)) and s.cursor == 100
    # the same with a caller's CUDA tensor (large enough to skip the host staging path)
    s = B.FixedSequenceSource(words[:100], 64)
    zt = torch.arange(20000, dtype=torch.int32, device="cuda")
    with pytest.raises(B.SourceExhausted):
        B.shuffle_batched(s, zt)
    assert torch.equal(zt, torch.arange(20000, dtype=torch.int32, device="cuda")) and s.cursor == 100
    s = B.FixedSequenceSource(words, 64)
    zt = torch.arange(3000, dtype=torch.int32, device="cuda")
    B.shuffle_batched(s, zt)
    o = O.fixed(words)
    assert np.array_equal(u32(zt), O.shuffle_batched(o, np.arange(3000, dtype=np.uint32))) and s.cursor == o.cursor
    with pytest.raises(TypeError):
        B.shuffle_batched(B.FixedSequenceSource([1, 2, 3], 16), [1, 2, 3], B.ShuffleSchedule(((1 << 4, 2),), 2, 16))
    with pytest.raises(TypeError):
        B.shuffle_batched(B.ExhaustiveSource(8), [1, 2, 3], B.ShuffleSchedule(((8, 2),), 2, 8))


def test_wide_bases_single_batches(B, O):
    """roll_single / roll_batch / digit_pass with bases at or above 2^32, up to the full range
    2^64 (bounded.py:35-104, batched.py:69-123): the one-thread 64-bit path."""
    cases = [(1 << 40,), ((1 << 64) - 1,), (1 << 63, 2), (3 << 33, 1 << 20, 7), ((1 << 32) + 15, (1 << 31) - 1)]
    for seed, bases in enumerate(cases):
        s, o = B.Pcg64Source(seed), O.pcg64(seed)
        spec = B.BatchSpec(B.RadixBases.of(bases))
        for _ in range(30):
            r = B.roll_batch(s, spec)
            ro = O.roll_batch(o, bases)
            assert (r.digits, r.words_consumed, r.threshold_computed, r.final_remainder) == ro, (bases, r, ro)
        assert s.state == o.state
        for r0 in (0, 1, (1 << 64) - 1, 0x123456789ABCDEF0):
            assert B.digit_pass(r0, B.RadixBases.of(bases)) == O.digit_pass(r0, bases)
    for gen in ("pcg64", "lehmer", "chacha"):  # bound 2^64 is the full range (the word itself)
        s, o = B.make_source(gen, 5), O.GENERATOR_MAKERS[gen](5)
        for bound in (1 << 33, (1 << 64) - 12345, 1 << 64):
            for _ in range(10):
                v, w, ro = O.roll_single(o, bound)
                r = B.roll_single_traced(s, bound)
                assert (r.value, r.words_consumed, r.remainder_ops) == (v, w, ro)
    # heavy rejection: 2^63 + 1 rejects about half of all words
    s, o = B.Pcg64Source(77), O.pcg64(77)
    rej = 0
    for _ in range(50):
        v, w, ro = O.roll_single(o, (1 << 63) + 1)
        r = B.roll_single_traced(s, (1 << 63) + 1)
        assert (r.value, r.words_consumed, r.remainder_ops) == (v, w, ro)
        rej += w - 1
    assert rej > 5 and s.state == o.state
