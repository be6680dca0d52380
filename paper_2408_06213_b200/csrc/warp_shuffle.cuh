// warp_shuffle.cuh -- one warp per shared-memory-resident array, 32 Fisher-Yates steps per
// warp step, for the many-arrays calls of moderate length (C4: 65,536 x u32[4096]).
//
// Same algorithm as shuffle.cuh (shuffle.py:100-225: batches of k dice, rejection re-draws
// the batch from the next word), built for few instructions per element:
//   * per-batch records {threshold, n_b, k_b} (plan.brec) replace the segment walk;
//   * targets go into a 512-entry u16 ring just ahead of the groups that read them;
//   * a group of 32 steps i_l = top - l (lane l) is applied as independent swaps, except
//     for "dirty" lanes, which are then replayed one at a time in step order.  Lane l is
//     dirty iff its target is shared with another lane (match.any), lies inside the group
//     (another lane's position), or some other lane targets i_l.  A clean lane's two
//     positions are touched by no other lane, so applying the clean lanes first and the
//     dirty ones sequentially equals the sequential loop.  For n = 4096 about one lane in
//     sixty is dirty.
#pragma once
#include "shuffle.cuh"

namespace br {

static constexpr uint32_t WRING = 512;

struct WarpGen {
    u128 s, inc, A32, C32;
    u128 W0;                  // ChaCha: origin of the warp's keystream window
    uint32_t B0, D, frontier; // frontier: lowest position whose target is committed
};

// 32 batches B0 + lane on words B0 + D + lane; the accepted prefix is committed
template <bool CHA>
__device__ __forceinline__ void warp_gen_step(WarpGen &g, const DevPlan &plan, uint16_t *ring, int lane,
                                              uint64_t *rk_first, uint64_t *chawin, const ChaKey &ck) {
    const bool lh = is_lehmer(g.inc);
    const uint32_t nb = plan.nbatches;
    const uint32_t b = g.B0 + lane;
    bool fail = false;
    uint32_t low = 0xFFFFFFFFu;
    uint64_t rc = 0;
    if constexpr (CHA) rc = cha_warp_word(chawin, ck, g.W0, cha_prev(g.s), lane);  // warp-collective
    if (b < nb) {
        const uint4 rec = __ldg(plan.brec + b);
        const uint64_t t = ((uint64_t)rec.y << 32) | rec.x;
        const uint32_t nbb = rec.z, k = rec.w;
        uint64_t r = CHA ? rc : gen_out(g.s, lh);
        const uint32_t pos = nbb - 1;
        if (plan.naive && k == 2) {
            uint32_t j1, j2;
            naive_pair(nbb, r, j1, j2);
            ring[pos & (WRING - 1)] = (uint16_t)j1;
            ring[(pos - 1) & (WRING - 1)] = (uint16_t)j2;
        } else {
            for (uint32_t m = 0; m < k; ++m) ring[(pos - m) & (WRING - 1)] = (uint16_t)die(nbb - m, r);
        }
        low = nbb - k;
        fail = r < t;
        if (rk_first && b == 0 && g.D == 0) *rk_first = r;
    }
    const unsigned fm = __ballot_sync(FULL, fail);
    const unsigned active = __ballot_sync(FULL, b < nb);
    const unsigned commit = fm ? (active & ((fm & (0u - fm)) - 1u)) : active;
    if (commit) g.frontier = __shfl_sync(FULL, low, 31 - __clz(commit));
    __syncwarp();
    if (fm == 0) {
        g.B0 += 32;
        if constexpr (CHA) g.s = cha_add(g.s, 32);
        else g.s = mad128(g.s, g.A32, g.C32);
    } else {
        const int l = __ffs(fm) - 1;
        g.B0 += l;
        g.D += 1;
        if constexpr (CHA) g.s = cha_add(g.s, (uint64_t)l + 1);
        else g.s = gen_jump_small(g.s, g.inc, l + 1, lh);
    }
}

// steps top, top-1, ..., max(top-31, lim) of z[i] <-> z[J[i]] (i descending)
template <typename T>
__device__ __forceinline__ void warp_apply_group(T *z, const uint16_t *ring, uint32_t top, uint32_t lim, int lane) {
    const bool act = (uint32_t)lane <= top - lim;
    const uint32_t i = top - lane;
    const uint32_t lo = top - lim >= 31 ? top - 31 : lim;
    uint32_t j = 0;
    T vi = T(0), vj = T(0);
    if (act) {
        j = ring[i & (WRING - 1)];
        vi = z[i];
        vj = z[j];
    }
    const unsigned same = __match_any_sync(FULL, act ? j : 0x10000u + lane);
    const bool inr = act && j >= lo && j != i;  // the target is another lane's position
    const unsigned hit = __reduce_or_sync(FULL, inr ? 1u << (top - j) : 0u);
    const bool dirty = act && (same != (1u << lane) || inr || ((hit >> lane) & 1u));
    const unsigned dm = __ballot_sync(FULL, dirty);
    if (act && !dirty) {
        z[i] = vj;
        z[j] = vi;
    }
    if (dm) {
        __syncwarp();
        for (unsigned m = dm; m; m &= m - 1) {
            if (lane == __ffs(m) - 1) {
                const T a = z[i], c = z[j];
                z[i] = c;
                z[j] = a;
            }
            __syncwarp();
        }
    }
    __syncwarp();
}

template <typename T, bool SEGMENTED, bool CHA>
__device__ __forceinline__ void shuffle_warp_body(T *__restrict__ data, int64_t num_arrays, const DevPlan &plan,
                                                  uint64_t run_seed, int64_t base, uint32_t *__restrict__ words32,
                                                  uint64_t *state_io, uint64_t *words64, uint64_t *rk_first,
                                                  int use_tma, int gen, T *z, uint16_t *ring, uint64_t &bar,
                                                  uint64_t *chawin) {
    const int lane = threadIdx.x & 31;
    if (use_tma && lane == 0) mbar_init(&bar, 1);
    __syncwarp();
    const uint32_t n = plan.n;
    const uint32_t bytes = n * (uint32_t)sizeof(T);
    const uint32_t lim = plan.lo > 1 ? plan.lo : 1;
    uint32_t parity = 0;
    for (int64_t a = blockIdx.x; a < num_arrays; a += gridDim.x) {
        T *g = data + a * (int64_t)n;
        if (use_tma) {
            if (lane == 0) {
                bulk_wait_read();  // the previous array's bulk store has read z
                fence_proxy_async();
                mbar_arrive_expect_tx(&bar, bytes);
                bulk_load(z, g, bytes, &bar);
            }
        } else {
            warp_copy(z, g, n, lane);
        }
        u128 s0, inc;
        bool lh;
        ChaKey ck;
        if constexpr (SEGMENTED) {
            lh = gen == 1;
            const uint64_t seed = array_seed(run_seed, (uint64_t)(base + a));
            if constexpr (CHA) {
                chacha_seed(seed, ck);
                s0 = mk128(0, 0);
                inc = mk128(ck.nonce, CHACHA_TAG);
            } else {
                gen_seed(seed, s0, inc, lh);
            }
        } else {
            s0 = mk128(state_io[0], state_io[1]);
            inc = mk128(state_io[2], state_io[3]);
            lh = is_lehmer(inc);
            if constexpr (CHA) ck = cha_key_of_state(state_io);
        }
        WarpGen gs;
        gs.inc = inc;
        if constexpr (CHA) {
            gs.s = cha_add(s0, (uint64_t)lane + 1);
            gs.W0 = cha_win_unset(s0);
        } else {
            gs.s = gen_jump_small(s0, inc, lane + 1, lh);
            gs.A32 = gen_SA(lh, 32);
            gs.C32 = mul128(g_SG[32], inc);
        }
        gs.B0 = 0;
        gs.D = 0;
        gs.frontier = n;
        uint64_t *rkf = SEGMENTED ? nullptr : rk_first;
        // the first targets are generated while the payload streams in
        if (plan.nbatches) warp_gen_step<CHA>(gs, plan, ring, lane, rkf, chawin, ck);
        if (use_tma) {
            mbar_wait(&bar, parity);
            parity ^= 1u;
        }
        __syncwarp();
        for (uint32_t top = n - 1; n > lim; top -= 32) {
            const uint32_t need = top - lim >= 31 ? top - 31 : lim;
            while (gs.frontier > need && gs.B0 < plan.nbatches) warp_gen_step<CHA>(gs, plan, ring, lane, rkf, chawin, ck);
            warp_apply_group<T>(z, ring, top, lim, lane);
            if (top < lim + 32) break;
        }
        // finish the word accounting (a trailing rejection can follow the last position)
        while (gs.B0 < plan.nbatches) warp_gen_step<CHA>(gs, plan, ring, lane, rkf, chawin, ck);
        if (use_tma) {
            if (lane == 0) {
                fence_proxy_async();
                bulk_store(g, z, bytes);
            }
        } else {
            warp_copy(g, z, n, lane);
        }
        const uint64_t words = (uint64_t)plan.nbatches + gs.D;
        if (lane == 0) {
            if constexpr (SEGMENTED) {
                if (words32) words32[a] = (uint32_t)words;
            } else {
                const u128 sf = CHA ? cha_add(s0, words) : gen_jump(s0, inc, words, lh);
                state_io[0] = sf.hi;
                state_io[1] = sf.lo;
                if (words64) words64[0] = words;
            }
        }
        __syncwarp();
    }
    if (use_tma && lane == 0) bulk_wait_all();
}

// CM as in shuffle_mid_kernel: 0 = PCG64/Lehmer, 1 = ChaCha, 2 = from the stream state's tag
template <typename T, bool SEGMENTED, int CM>
__global__ void __launch_bounds__(32) shuffle_warp_kernel(T *__restrict__ data, int64_t num_arrays, DevPlan plan,
                                                          uint64_t run_seed, int64_t base,
                                                          uint32_t *__restrict__ words32, uint64_t *state_io,
                                                          uint64_t *words64, uint64_t *rk_first, int use_tma,
                                                          int gen) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(16) uint16_t ring[WRING];
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(16) uint64_t chawin[CM ? 256 : 2];
    T *z = reinterpret_cast<T *>(smem_raw);
    bool cha = CM == 1;
    if constexpr (CM == 2) cha = is_posgen(mk128(state_io[2], state_io[3]));
    if (CM != 0 && cha)
        shuffle_warp_body<T, SEGMENTED, CM != 0>(data, num_arrays, plan, run_seed, base, words32, state_io, words64,
                                                 rk_first, use_tma, gen, z, ring, bar, chawin);
    else if (CM != 1)
        shuffle_warp_body<T, SEGMENTED, false>(data, num_arrays, plan, run_seed, base, words32, state_io, words64,
                                               rk_first, use_tma, gen, z, ring, bar, chawin);
}

}  // namespace br
