// warp_shuffle.cuh -- one warp per shared-memory-resident array, 32 Fisher-Yates steps per
// warp step, in two kernels:
//   * shuffle_warp_kernel: the array itself in shared memory, one warp per CTA (many arrays
//     of up to 16 KB);
//   * shuffle_idx_kernel: a u16 index permutation per warp, NW warps per CTA, the payload
//     applied at the end through shared staging buffers (C4: 65,536 x u32[4096], 20 arrays
//     per SM instead of 12).
//
// Same algorithm as shuffle.cuh (shuffle.py:100-225: batches of k dice, rejection re-draws
// the batch from the next word), built for few instructions and short dependency chains:
//   * per-batch records {threshold, n_b, k_b} (plan.brec) replace the segment walk;
//   * targets go into a 256-entry u16 ring just ahead of the groups that read them;
//   * a group of 32 steps i_l = top - l (lane l) is resolved exactly in registers
//     (warp_apply_group_exact): equal targets through a byte table instead of MATCH.ANY,
//     predecessor chains through 32 bytes of shared memory and shuffles, no serial replay;
//   * the next group's targets and equality mask are prepared around the current group.
#pragma once
#include "shuffle.cuh"
#include <type_traits>

namespace br {

// 256 entries hold the current and next group and one generation step for k <= 6 (the
// default schedule); with the 1 KB target table that keeps 12 arrays of 16 KB per SM
static constexpr uint32_t WRING = 256;

struct WarpGen {
    u128 s, inc, A32, C32;
    u128 W0;                  // ChaCha: origin of the warp's keystream window
    uint32_t B0, D, frontier; // frontier: lowest position whose target is committed
};

// 32 batches B0 + lane on words B0 + D + lane; the accepted prefix is committed
template <bool CHA, uint32_t RS = WRING>
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
            ring[pos & (RS - 1)] = (uint16_t)j1;
            ring[(pos - 1) & (RS - 1)] = (uint16_t)j2;
        } else {
            // unrolled for the default schedule's k (k changes only at regime edges)
            auto dice = [&](auto K) {
#pragma unroll
                for (uint32_t m = 0; m < decltype(K)::value; ++m)
                    ring[(pos - m) & (RS - 1)] = (uint16_t)die(nbb - m, r);
            };
            switch (k) {
            case 2: dice(std::integral_constant<uint32_t, 2>{}); break;
            case 3: dice(std::integral_constant<uint32_t, 3>{}); break;
            case 4: dice(std::integral_constant<uint32_t, 4>{}); break;
            case 5: dice(std::integral_constant<uint32_t, 5>{}); break;
            case 6: dice(std::integral_constant<uint32_t, 6>{}); break;
            default:
                for (uint32_t m = 0; m < k; ++m) ring[(pos - m) & (RS - 1)] = (uint16_t)die(nbb - m, r);
            }
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
        else g.s = mad128_wide(g.s, g.A32, g.C32);  // 17 SASS instructions against 25
    } else {
        const int l = __ffs(fm) - 1;
        g.B0 += l;
        g.D += 1;
        if constexpr (CHA) g.s = cha_add(g.s, (uint64_t)l + 1);
        else g.s = gen_jump_small(g.s, g.inc, l + 1, lh);
    }
}

// Shared-memory accesses of the group loop through 32-bit shared addresses: with generic
// pointers ptxas re-forms the shared window base (S2R SR_CgaCtaId + LEA) inside the loop,
// and every swap waits on that S2R.  The base is laundered through a volatile move once.
__device__ __forceinline__ uint32_t smem_base(const void *p) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(p), b;
    asm volatile("mov.b32 %0, %1;" : "=r"(b) : "r"(a));
    return b;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void lds_v(uint32_t a, uint16_t &v) {
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
}
__device__ __forceinline__ void sts_v(uint32_t a, uint16_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(v) : "memory");
}
__device__ __forceinline__ void lds_v(uint32_t a, uint32_t &v) {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
}
__device__ __forceinline__ void lds_v(uint32_t a, uint64_t &v) {
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
}
__device__ __forceinline__ void sts_v(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_v(uint32_t a, uint64_t v) {
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ int lds_s8(uint32_t a) {
    int16_t v;
    asm volatile("ld.shared.s8 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_s8(uint32_t a, int v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "h"((int16_t)v) : "memory");
}

// The caller loads group g+1's targets and their equality mask ahead of group g's swaps.
// same = the lanes whose target equals this lane's.  MATCH.ANY computes it in one
// instruction but is slow on sm_100 (C4: 2.18 ms with it, 1.41 ms with the mask stubbed
// out), so lanes write their id into a 1024-slot byte table at j mod 1024 and read the slot
// back: a lane that reads another id shares a slot, and only then are the slot's lanes
// split by exact target, one ballot per distinct target.  Stale slots are never read (a
// lane reads only the slot it has just written).
static constexpr uint32_t WTBL = 1024;

// issue: targets and the slot read-back (consumed after the current group's swaps).
// FG: the group is full (top - lim >= 31), so every lane is active.
template <bool FG = false>
__device__ __forceinline__ void warp_group_targets(uint32_t ring, uint32_t tbl, uint32_t top, uint32_t lim,
                                                   int lane, uint32_t &j, bool &shared_slot) {
    // branch-free (every lane loads and stores; a branch here costs reconvergence and a
    // divergence check before each of the group's warp intrinsics): an inactive lane reads
    // a wrapped ring entry it ignores and writes its own private byte after the table
    const bool act = FG || (uint32_t)lane <= top - lim;
    const uint32_t jr = lds_u16(ring + 2u * ((top - lane) & (WRING - 1)));
    j = act ? jr : 0u;
    const uint32_t slot = act ? tbl + (jr & (WTBL - 1)) : tbl + WTBL + (uint32_t)lane;
    sts_s8(slot, lane);
    __syncwarp();
    shared_slot = lds_s8(slot) != lane;
}

// finish: split the lanes of shared slots by exact target
template <bool FG = false>
__device__ __forceinline__ unsigned warp_group_same(uint32_t top, uint32_t lim, int lane, uint32_t j, bool shared_slot) {
    const bool act = FG || (uint32_t)lane <= top - lim;
    unsigned pending = __ballot_sync(FULL, shared_slot);
    unsigned same = 1u << lane;
    while (pending) {
        const uint32_t jf = __shfl_sync(FULL, j, __ffs(pending) - 1);
        const unsigned S = __ballot_sync(FULL, act && j == jf);
        if ((S >> lane) & 1u) same = S;
        pending &= ~S;
    }
    return same;
}

// steps top, top-1, ..., max(top-31, lim) of z[i] <-> z[J[i]] (i descending), resolved
// exactly in registers (the warp form of apply_group_cta_global):
//   lane l owns step i_l = top - l with target j_l <= i_l; all values are loaded first;
//   T(l)    = latest earlier lane with target j_l           (equality mask below l)
//   Pred(l) = latest earlier lane whose target is i_l       (one byte per lane in P)
//   A_l = A_Pred(l), else z[i_l]    -- the value step l moves to j_l
//   B_l = A_T(l),    else z[j_l]    -- the value step l leaves at i_l (final: no later step
//                                      of the group can target i_l, all j are <= their i)
// z[j_l] = A_l is written by the last lane of each target below the group; targets inside
// the group are positions whose own lane writes B.  No lane is replayed serially.
template <typename T, bool FG = false>
__device__ __forceinline__ void warp_apply_group_exact(uint32_t z, uint32_t P, uint32_t top, uint32_t lim, int lane,
                                                       uint32_t j, unsigned same) {
    constexpr uint32_t E = sizeof(T);
    const bool act = FG || (uint32_t)lane <= top - lim;
    const uint32_t i = top - lane;
    const uint32_t lo = (FG || top - lim >= 31) ? top - 31 : lim;
    T vi, vj;
    lds_v(z + E * (act ? i : top), vi);  // inactive lanes (j = 0) load values nobody uses
    lds_v(z + E * j, vj);
    const unsigned below = same & ((1u << lane) - 1u);
    const unsigned above = same & ~((2u << lane) - 1u);  // later lanes (lane 31: 2u << 31 == 0)
    const bool inr = act && j >= lo && j != i;            // j = i_l' of a later lane l' = top - j
    T A = vi;
    if (__ballot_sync(FULL, inr)) {
        // P[l] is -1 on entry (set once per kernel, restored below after each use)
        // the latest lane before l' = top - j targeting i_l' (l' itself may target it: a self-swap)
        if (inr && (above & ~(1u << (top - j))) == 0) sts_s8(P + (top - j), lane);
        __syncwarp();
        const int p = lds_s8(P + lane);
        sts_s8(P + lane, -1);  // ordered before the next group's writes by the syncwarps between
        int r = p >= 0 ? p : lane;
        for (;;) {  // pointer jumping to the root of the Pred chain (Pred(l) < l)
            const int rr = __shfl_sync(FULL, r, r);
            if (!__ballot_sync(FULL, rr != r)) break;
            r = rr;
        }
        A = shfl_t<T>(vi, r);
        __syncwarp();
    }
    const int tl = below ? 31 - __clz(below) : lane;
    const T Bt = shfl_t<T>(A, tl);
    if (act) sts_v(z + E * i, below ? Bt : vj);
    if (act && !above && j < lo) sts_v(z + E * j, A);
    __syncwarp();
}

// IDX: the warp shuffles a u16 index permutation of the array (2 bytes per element in shared
// memory instead of sizeof(T)), then applies it to the payload through one of the CTA's
// shared staging buffers: more arrays per SM (shuffle_idx_kernel).
template <typename T, bool SEGMENTED, bool CHA, bool IDX = false>
__device__ __forceinline__ void shuffle_warp_body(T *__restrict__ data, int64_t num_arrays, const DevPlan &plan,
                                                  uint64_t run_seed, int64_t base, uint32_t *__restrict__ words32,
                                                  uint64_t *state_io, uint64_t *words64, uint64_t *rk_first,
                                                  int use_tma, int gen, std::conditional_t<IDX, uint16_t, T> *z,
                                                  uint16_t *ring, int8_t *P, int8_t *tbl, uint64_t &bar,
                                                  uint64_t *chawin, T *stage = nullptr, uint32_t *locks = nullptr,
                                                  int nstage = 0, uint32_t stage_elems = 0) {
    using E = std::conditional_t<IDX, uint16_t, T>;  // element type of the array being permuted
    const int lane = threadIdx.x & 31;
    // test knob (BR_IDX_HOLD_US, bits 8.. of use_tma): the holder of staging buffer 0 sleeps that
    // long, which piles the warps up on one buffer's queue (tests/test_gpu.py ticket stress)
    const int hold_us = use_tma >> 8;
    use_tma &= 1;
    if (!IDX && use_tma && lane == 0) mbar_init(&bar, 1);
    P[lane] = -1;  // warp_apply_group_exact's invariant
    __syncwarp();
    const uint32_t n = plan.n;
    const uint32_t bytes = n * (uint32_t)sizeof(T);
    const uint32_t lim = plan.lo > 1 ? plan.lo : 1;
    uint32_t parity = 0;
    const int64_t a0 = IDX ? (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5) : blockIdx.x;
    const int64_t astep = IDX ? (int64_t)gridDim.x * (blockDim.x >> 5) : gridDim.x;
    for (int64_t a = a0; a < num_arrays; a += astep) {
        T *g = data + a * (int64_t)n;
        if constexpr (IDX) {
            // identity permutation (an L2 prefetch of the payload here or later measured no gain)
            for (uint32_t p = lane; 2 * p < n; p += 32)
                reinterpret_cast<uint32_t *>(z)[p] = (2 * p) | ((2 * p + 1) << 16);
        } else if (use_tma) {
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
        if (plan.nbatches) warp_gen_step<CHA, WRING>(gs, plan, ring, lane, rkf, chawin, ck);
        if (!IDX && use_tma) {
            mbar_wait(&bar, parity);
            parity ^= 1u;
        }
        __syncwarp();
        if (n > lim) {
            // software-pipelined: group g+1's targets and equality mask are prepared around
            // group g's swaps
            uint32_t top = n - 1, j;
            unsigned same;
            const uint32_t need0 = top - lim >= 31 ? top - 31 : lim;
            while (gs.frontier > need0 && gs.B0 < plan.nbatches) warp_gen_step<CHA, WRING>(gs, plan, ring, lane, rkf, chawin, ck);
            __syncwarp();
            const uint32_t zs = smem_base(z), rs = smem_base(ring), ps = smem_base(P), ts = smem_base(tbl);
            bool sh;
            warp_group_targets(rs, ts, top, lim, lane, j, sh);
            same = warp_group_same(top, lim, lane, j, sh);
            // one group: issue the next group's targets into jn, swap this one, then finish
            // the next group's equality mask sn (its table read-back hides behind the swaps)
            // FG: this group and the next are full (t >= lim + 63): no partial-group predicates
            auto group = [&](auto FG, uint32_t t, uint32_t jc, unsigned sc, uint32_t &jn, unsigned &sn) -> bool {
                constexpr bool F = decltype(FG)::value;
                const bool last = !F && t < lim + 32;
                const uint32_t nt = t - 32;
                bool shn = false;
                if (!last) {
                    const uint32_t need = (F || nt - lim >= 31) ? nt - 31 : lim;
                    // the ring has room for the current group, the next and one generation step;
                    // the common case (targets already there) costs one compare
                    if (gs.frontier > need) {
                        do {
                            warp_gen_step<CHA, WRING>(gs, plan, ring, lane, rkf, chawin, ck);
                        } while (gs.frontier > need && gs.B0 < plan.nbatches);
                    }
                    __syncwarp();
                    warp_group_targets<F>(rs, ts, nt, lim, lane, jn, shn);
                }
                warp_apply_group_exact<E, F>(zs, ps, t, lim, lane, jc, sc);
                if (!last) sn = warp_group_same<F>(nt, lim, lane, jn, shn);
                return last;
            };
            uint32_t j2;
            unsigned same2;
            using Full = std::true_type;
            using Part = std::false_type;
            // unrolled by two: the prefetched values are never copied
            while (top >= lim + 95) {  // both groups of the pair and their successors are full
                group(Full{}, top, j, same, j2, same2);
                top -= 32;
                group(Full{}, top, j2, same2, j, same);
                top -= 32;
            }
            for (;;) {
                if (group(Part{}, top, j, same, j2, same2)) break;
                top -= 32;
                if (group(Part{}, top, j2, same2, j, same)) break;
                top -= 32;
            }
        }
        // finish the word accounting (a trailing rejection can follow the last position)
        while (gs.B0 < plan.nbatches) warp_gen_step<CHA, WRING>(gs, plan, ring, lane, rkf, chawin, ck);
        if constexpr (IDX) {
            // take a staging buffer in ticket order (FIFO hand-off): ticket t uses buffer
            // t % nstage and is number t / nstage in that buffer's queue; its predecessor in the
            // queue hands the buffer over by arriving on the mbarrier of the queue's slot
            // (t / nstage) % 32.  A queue's waiters are consecutive and at most one per warp
            // (<= 24), so a slot's barrier is never two phases away from its waiter; the
            // waiter sleeps in mbarrier.try_wait instead of polling a lock
            uint64_t *slotbar = reinterpret_cast<uint64_t *>(locks + 32);
            int sb = 0;
            uint32_t tk = 0, ph = 0;
            if (lane == 0) {
                tk = atomicAdd(&locks[0], 1u);
                sb = (int)(tk % (uint32_t)nstage);
                const uint32_t sq = tk / (uint32_t)nstage;  // position in the buffer's own queue
                mbar_wait(slotbar + (uint32_t)sb * 32u + (sq & 31u), (sq >> 5) & 1u);  // (the first holder: handed over at start)
                ph = locks[8 + sb];  // the buffer's load phase, read once by the lane that flips it
            }
            sb = __shfl_sync(FULL, sb, 0);
            ph = __shfl_sync(FULL, ph, 0);
            __syncwarp();
            T *buf = stage + (size_t)sb * stage_elems;
            if (hold_us && sb == 0)
                for (int h = 0; h < hold_us; ++h) __nanosleep(1000);
            if (use_tma) {  // one bulk copy; the stage's mbarrier phase lives next to its lock
                uint64_t *sbar = reinterpret_cast<uint64_t *>(locks + 16) + sb;
                if (lane == 0) {
                    fence_proxy_async();  // the previous holder's generic reads of buf come first
                    mbar_arrive_expect_tx(sbar, bytes);
                    bulk_load(buf, g, bytes, sbar);
                }
                mbar_wait(sbar, ph);
                if (lane == 0) locks[8 + sb] = ph ^ 1u;
            } else {
                warp_copy(buf, g, n, lane);
            }
            __syncwarp();
            if (use_tma && (n & 3u) == 0) {  // 16-byte aligned payload: 4 elements per lane step
#pragma unroll 4
                for (uint32_t q = lane; 4 * q < n; q += 32) {
                    const uint2 iv = reinterpret_cast<const uint2 *>(z)[q];
                    const T v0 = buf[iv.x & 0xFFFFu], v1 = buf[iv.x >> 16], v2 = buf[iv.y & 0xFFFFu], v3 = buf[iv.y >> 16];
                    if constexpr (sizeof(T) == 4) {
                        reinterpret_cast<uint4 *>(g)[q] = make_uint4((uint32_t)v0, (uint32_t)v1, (uint32_t)v2, (uint32_t)v3);
                    } else {
                        reinterpret_cast<ulonglong2 *>(g)[2 * q] = make_ulonglong2((uint64_t)v0, (uint64_t)v1);
                        reinterpret_cast<ulonglong2 *>(g)[2 * q + 1] = make_ulonglong2((uint64_t)v2, (uint64_t)v3);
                    }
                }
            } else {
                for (uint32_t p = lane; p < n; p += 32) g[p] = buf[z[p]];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(slotbar + (uint32_t)sb * 32u + ((tk / (uint32_t)nstage + 1u) & 31u));
        } else if (use_tma) {
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
    if (!IDX && use_tma && lane == 0) bulk_wait_all();
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
    __shared__ int8_t P[32];
    __shared__ int8_t tbl[WTBL + 32];
    __shared__ __align__(16) uint64_t chawin[CM ? 256 : 2];
    T *z = reinterpret_cast<T *>(smem_raw);
    bool cha = CM == 1;
    if constexpr (CM == 2) cha = is_posgen(mk128(state_io[2], state_io[3]));
    if (CM != 0 && cha)
        shuffle_warp_body<T, SEGMENTED, CM != 0>(data, num_arrays, plan, run_seed, base, words32, state_io, words64,
                                                 rk_first, use_tma, gen, z, ring, P, tbl, bar, chawin);
    else if (CM != 1)
        shuffle_warp_body<T, SEGMENTED, false>(data, num_arrays, plan, run_seed, base, words32, state_io, words64,
                                               rk_first, use_tma, gen, z, ring, P, tbl, bar, chawin);
}

// Many arrays, u16 index permutations (IDX mode of shuffle_warp_body): one CTA per SM of NW
// warps, each warp its own arrays; dynamic shared memory = nstage staging buffers (payload
// of one array each, shared by the CTA's warps under a lock) + 16 B of locks + per warp
// { u16 index array, target ring, equality table, Pred bytes, ChaCha window }.
constexpr uint32_t idx_warp_fixed(int cm) { return 2 * WRING + WTBL + 32 + 32 + (cm ? 256 * 8 : 0); }
// ticket, 8 load phases, 8 load mbarriers, then 32 ticket-slot mbarriers PER BUFFER (8 buffers): a
// buffer's waiters are consecutive in its own queue, so 32 slots cover any 24 warps.  (One ring of
// 32 slots over all buffers let ticket t + 32 pass while t still waited once 17 or more warps
// queued on one buffer: two holders of one buffer.)
constexpr uint32_t IDX_CTL_BYTES = 128 + 8 * 32 * 8;


template <typename T, int CM>
__global__ void __launch_bounds__(768, 1) shuffle_idx_kernel(T *__restrict__ data, int64_t num_arrays, DevPlan plan,
                                                           uint64_t run_seed, int64_t base,
                                                           uint32_t *__restrict__ words32, int use_tma, int gen,
                                                           int nstage) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t n = plan.n;
    const uint32_t selems = (n + 3u) & ~3u;
    const uint32_t sbytes = (uint32_t)(((uint64_t)selems * sizeof(T) + 15u) & ~15ull);
    const uint32_t ibytes = (2u * n + 15u) & ~15u;
    unsigned char *p = smem_raw;
    T *stage = reinterpret_cast<T *>(p);
    p += (size_t)nstage * sbytes;
    // locks[0..7], mbarrier phases [8..15], mbarriers (u64) from word 16
    uint32_t *locks = reinterpret_cast<uint32_t *>(p);
    p += IDX_CTL_BYTES;
    unsigned char *mine = p + (size_t)(threadIdx.x >> 5) * (ibytes + idx_warp_fixed(CM));
    uint16_t *idx = reinterpret_cast<uint16_t *>(mine);
    uint16_t *ring = reinterpret_cast<uint16_t *>(mine + ibytes);
    int8_t *tbl = reinterpret_cast<int8_t *>(mine + ibytes + 2 * WRING);
    int8_t *P = tbl + WTBL + 32;  // the table's last 32 bytes: inactive lanes' private slots
    uint64_t *chawin = reinterpret_cast<uint64_t *>(P + 32);
    if (threadIdx.x < (unsigned)nstage) {
        locks[threadIdx.x] = 0u;  // locks[0]: the staging-buffer ticket counter
        locks[8 + threadIdx.x] = 0u;
        mbar_init(reinterpret_cast<uint64_t *>(locks + 16) + threadIdx.x, 1);  // bulk load done
    }
    for (uint32_t i = threadIdx.x; i < (uint32_t)nstage * 32u; i += blockDim.x) {
        // ticket hand-off; the first ticket of each buffer is handed its buffer now
        mbar_init(reinterpret_cast<uint64_t *>(locks + 32) + i, 1);
        if ((i & 31u) == 0) mbar_arrive(reinterpret_cast<uint64_t *>(locks + 32) + i);
    }
    __syncthreads();
    uint64_t bar = 0;
    if constexpr (CM == 1)
        shuffle_warp_body<T, true, true, true>(data, num_arrays, plan, run_seed, base, words32, nullptr, nullptr,
                                                   nullptr, use_tma, gen, idx, ring, P, tbl, bar, chawin, stage,
                                                   locks, nstage, selems);
    else
        shuffle_warp_body<T, true, false, true>(data, num_arrays, plan, run_seed, base, words32, nullptr,
                                                    nullptr, nullptr, use_tma, gen, idx, ring, P, tbl, bar, chawin,
                                                    stage, locks, nstage, selems);
}

}  // namespace br
