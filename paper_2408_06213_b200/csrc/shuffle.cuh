// shuffle.cuh -- segmented Fisher-Yates shuffles with batched dice (shuffle.py:100-225).
//
// A compiled plan (capi.cu get_plan) lists the batches of shuffle_batched for one length n; batch b
// has remaining length n_b, size k_b and exact threshold t_b = 2^64 mod ff(n_b, k_b).
// A batch is accepted iff its final remainder r_k >= t_b.  This is exactly the
// reference's acceptance: the carried bound u of _run_batches (shuffle.py:118-128) only
// decides WHEN the threshold is computed, never WHETHER a batch is accepted (SURVEY
// finding 3; re-checked by tests/test_oracle.py, whose oracle keeps the literal u logic).
// Swaps of batch b: z[n_b-1-m] <-> z[d_m], m = 0..k_b-1, in that order.
//
// Work units sized to the array (north star item 3; dispatch in capi.cu launch_shuffle):
//   shuffle_small_kernel     one THREAD per array (small n), the block's arrays staged in
//                            shared memory with an odd row stride (conflict-free coalesced
//                            staging and uniform-position accesses);
//   shuffle_cta_hash_kernel  one CTA per shared-memory-resident array: TMA bulk copies in
//                            and out, targets generated just in time 32*W batches at a
//                            time, swaps applied 32*W steps at a time with an exact
//                            intra-group resolution (lane-chain hash + pointer jumping);
//   shuffle_cta_large_kernel the same groups on arrays in global memory (HBM-resident);
//   shuffle_mid_kernel / shuffle_large_gen+apply  warp-group forms for schedules with
//                            large k; shuffle_resolve_kernel (closed-form, whole array)
//                            serves single-array stream calls.
// Words: lane = batch, jump-ahead per lane, a CTA-wide vote on the rare rejection.
#pragma once
#include "chacha.cuh"
#include "jump.cuh"
#include "tma.cuh"

namespace br {

struct DevSeg {
    uint32_t start_n, k, count, first_batch;
};

static constexpr int MAX_SEGS = 40;

// Device plan header; thresholds follow in the same allocation.
struct DevPlan {
    uint32_t n, nbatches, nseg, max_k;
    uint32_t lo;              // lowest position that has a step (0 or 1 for full plans)
    uint32_t naive;           // pairs split by division (shuffle_naive_batched), see naive_pair
    const DevSeg *segs;       // [nseg]     (device)
    const uint64_t *thresh;   // [nbatches] (device)
    const uint4 *brec;        // [nbatches] {threshold lo, hi, n_b, k_b} (device; plans with n < 2^16 only)
};

// shuffle.py:242-253 (shuffle_naive_batched): the pair (i, i-1), i = nb - 1, takes ONE
// Lemire draw v = hi(b*w) on b = (i+1)*i and splits it by division, (j1, j2) = divmod(v, i).
// The acceptance (lo = b*w mod 2^64 >= 2^64 mod b) is the batched one (Theorem 1:
// r_2 == b*w mod 2^64), so the naive shuffle is the PAIR plan with division digits; the
// 64-by-32-bit division per pair is the cost this baseline exists to measure.
__device__ __forceinline__ void naive_pair(uint32_t nb, uint64_t &r, uint32_t &j1, uint32_t &j2) {
    const uint64_t i = nb - 1;
    const uint64_t b = (uint64_t)nb * i;
    const uint64_t v = __umul64hi(b, r);
    r = b * r;
    const uint64_t q = v / i;
    j1 = (uint32_t)q;
    j2 = (uint32_t)(v - q * i);
}

template <typename T>
__device__ __forceinline__ void swap_sm(T *p, uint32_t i, uint32_t j) {
    T x = p[i], y = p[j];
    p[i] = y;
    p[j] = x;
}

// -------------------------------------------------------------------------------------
// one thread per array
// -------------------------------------------------------------------------------------
// Run `count` consecutive batches of K dice (the first at remaining length nb) on one
// thread's array z (row of the block's shared buffer).  Fully unrolled per K.
template <int K, typename T, bool CHA>
__device__ __forceinline__ void small_segment(T *z, uint32_t nb, uint32_t count, const uint64_t *thresh, u128 &s,
                                              u128 inc, uint32_t &words, bool lh, const ChaKey &ck,
                                              ChaCursor &cur, bool naive) {
    for (uint32_t c = 0; c < count; ++c, nb -= K) {
        const uint64_t t = __ldg(thresh + c);
        uint32_t d[K];
        uint64_t r;
        do {
            if constexpr (CHA) {
                s = cha_add(s, 1);
                r = cha_out_cached(ck, cur, s);
            } else {
                r = gen_next(s, inc, lh);
            }
            ++words;
            if (K == 2 && naive) {
                naive_pair(nb, r, d[0], d[K - 1]);
            } else {
#pragma unroll
                for (int m = 0; m < K; ++m) d[m] = die(nb - m, r);
            }
        } while (r < t);  // reject: re-draw the whole batch (shuffle.py:121-128)
#pragma unroll
        for (int m = 0; m < K; ++m) swap_sm(z, nb - 1 - m, d[m]);
    }
}

template <typename T, bool CHA>
__device__ __forceinline__ void small_segment_any(T *z, uint32_t k, uint32_t nb, uint32_t count,
                                                  const uint64_t *thresh, u128 &s, u128 inc, uint32_t &words,
                                                  bool lh, const ChaKey &ck, ChaCursor &cur, bool naive) {
    switch (k) {
        case 1: small_segment<1, T, CHA>(z, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 2: small_segment<2, T, CHA>(z, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 3: small_segment<3, T, CHA>(z, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 4: small_segment<4, T, CHA>(z, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 5: small_segment<5, T, CHA>(z, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 6: small_segment<6, T, CHA>(z, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 7: small_segment<7, T, CHA>(z, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        default: small_segment<8, T, CHA>(z, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
    }
}

// Shared-memory layout: array t of the block at buf[t*stride + e], stride odd, so a warp's
// lanes touching the same position of 32 different arrays hit 32 different banks, and the
// coalesced copies (lanes = consecutive elements of one array) are conflict free too.
// Copies move the warp's own 32 arrays (a contiguous 32*n span) in 16-byte pieces when n
// is a multiple of 16/sizeof(T), else element by element; q / n uses a magic multiplier.
template <typename T>
__device__ __forceinline__ void small_copy(T *buf, T *g, uint32_t span, uint32_t n, uint32_t stride, uint32_t t0,
                                           uint32_t magic, int lane, bool to_smem, bool vec_ok) {
    constexpr uint32_t V = 16 / sizeof(T);
    constexpr int U = 8;  // half a warp span (n=64 u32) in flight per round
    if (vec_ok) {
        const uint32_t nv = span / V;
        for (uint32_t q0 = 0; q0 < nv; q0 += 32 * U) {
            uint4 v[U];
            if (to_smem) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t q = q0 + 32 * u + lane;
                    if (q < nv) v[u] = reinterpret_cast<const uint4 *>(g)[q];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t q = q0 + 32 * u + lane;
                if (q < nv) {
                    const uint32_t e0 = q * V;
                    const uint32_t t = __umulhi(e0, magic);
                    T *row = buf + (t0 + t) * stride + (e0 - t * n);
                    T *vv = reinterpret_cast<T *>(&v[u]);
                    if (to_smem) {
#pragma unroll
                        for (int x = 0; x < (int)V; ++x) row[x] = vv[x];
                    } else {
#pragma unroll
                        for (int x = 0; x < (int)V; ++x) vv[x] = row[x];
                        reinterpret_cast<uint4 *>(g)[q] = v[u];
                    }
                }
            }
        }
    } else {
        for (uint32_t q0 = 0; q0 < span; q0 += 32 * U) {
            T v[U];
            if (to_smem) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t q = q0 + 32 * u + lane;
                    if (q < span) v[u] = g[q];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t q = q0 + 32 * u + lane;
                if (q < span) {
                    const uint32_t t = __umulhi(q, magic);
                    T *p = buf + (t0 + t) * stride + (q - t * n);
                    if (to_smem) *p = v[u];
                    else g[q] = *p;
                }
            }
        }
    }
}

template <typename T, bool CHA>
__global__ void __launch_bounds__(128) shuffle_small_kernel(T *__restrict__ data, int64_t num_arrays,
                                                           DevPlan plan, uint32_t stride, uint32_t magic,
                                                           int vec_ok, uint64_t run_seed, int64_t base,
                                                           uint32_t *__restrict__ words_out, int gen) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ DevSeg segs[MAX_SEGS];
    T *buf = reinterpret_cast<T *>(smem_raw);
    const uint32_t n = plan.n;
    const int tid = threadIdx.x;
    const int64_t a0 = (int64_t)blockIdx.x * blockDim.x;
    const int na = (int)min((int64_t)blockDim.x, num_arrays - a0);
    if (tid < (int)plan.nseg) segs[tid] = plan.segs[tid];
    // each warp stages exactly the 32 arrays its lanes shuffle
    const int lane = tid & 31, wid = tid >> 5;
    const uint32_t t0 = wid * 32;
    const int tcount = max(0, min(32, na - (int)t0));
    T *g = data + (a0 + t0) * (int64_t)n;
    small_copy<T>(buf, g, (uint32_t)tcount * n, n, stride, t0, magic, lane, true, vec_ok != 0);
    __syncthreads();
    if (tid < na) {
        u128 s, inc;
        const bool lh = gen == 1;
        ChaKey ck;
        ChaCursor cur;
        cur.valid = false;
        const uint64_t seed = array_seed(run_seed, (uint64_t)(base + a0 + tid));
        if constexpr (CHA) {
            chacha_seed(seed, ck);
            s = mk128(0, 0);
            inc = mk128(ck.nonce, CHACHA_TAG);
        } else {
            gen_seed(seed, s, inc, lh);
        }
        T *z = buf + tid * stride;
        uint32_t words = 0;
        for (uint32_t sg = 0; sg < plan.nseg; ++sg) {
            const DevSeg S = segs[sg];
            small_segment_any<T, CHA>(z, S.k, S.start_n, S.count, plan.thresh + S.first_batch, s, inc, words, lh,
                                      ck, cur, plan.naive != 0);
        }
        if (words_out) words_out[a0 + tid] = words;
    }
    __syncwarp();
    small_copy<T>(buf, g, (uint32_t)tcount * n, n, stride, t0, magic, lane, false, vec_ok != 0);
}

// One thread per array on a u8 INDEX permutation (n <= 64).  Each thread shuffles the
// identity 0..n-1 as bytes, the same dice and swaps as shuffle_small_kernel, in a TRANSPOSED
// layout: byte j of lane l sits in word (j/4)*32 + l, i.e. every lane owns one bank, so the
// random swaps are conflict-free (the row layout measured ~3.5-way conflicts, the bound of
// shuffle_small_kernel).  The warp then turns its 32 permutations into rows (odd stride) and
// applies them to the payload one array at a time: lane l loads items l and l+32 (coalesced),
// fetches item row[p] from its owner lane with shuffles, and stores positions l and l+32.
// The payload never enters shared memory.
template <typename T>
struct alignas(2 * sizeof(T)) SmiPair {
    T a, b;
};

static constexpr int SMI_T = 128;  // 4 warps: 0.117 ms on C3 (8 warps: 0.121, 2 warps: 0.117)
#ifndef SMI_MINB
#define SMI_MINB 8
#endif
#ifndef SMI_U
#define SMI_U 8
#endif
static constexpr int SMI_WW = 32 * 17;  // words per warp: 16 transposed words x 32 lanes, or 32 rows of 17

__device__ __forceinline__ uint32_t smi_pos(uint32_t j) { return j + (j >> 2) * 124u; }  // (j/4)*128 + j%4

template <typename T>
__device__ __forceinline__ T smi_shfl(T v, int src) {
    if constexpr (sizeof(T) == 8) {
        const uint64_t x = (uint64_t)v;
        const uint32_t lo = __shfl_sync(0xFFFFFFFFu, (uint32_t)x, src), hi = __shfl_sync(0xFFFFFFFFu, (uint32_t)(x >> 32), src);
        return (T)(((uint64_t)hi << 32) | lo);
    } else {
        return (T)__shfl_sync(0xFFFFFFFFu, (uint32_t)v, src);
    }
}

// The K swaps of a batch at remaining length nb = 4a + R (za: row a of the lane's column):
// position nb-1-m = 4a + e, e = R-1-m, lies floor(e/4) rows away at byte e mod 4.
template <int K, int R>
__device__ __forceinline__ void smi_swaps(uint8_t *zt, uint8_t *za, const uint32_t (&d)[K]) {
#pragma unroll
    for (int m = 0; m < K; ++m) {
        const int e = R - 1 - m;
        const int row = (e >= 0) ? e / 4 : -((3 - e) / 4), byte = e - 4 * row;
        uint8_t *pi = za + (row * 128 + byte), *pj = zt + smi_pos(d[m]);
        const uint8_t x = *pi, y = *pj;
        *pi = y;
        *pj = x;
    }
}

template <int K, bool CHA>
__device__ __forceinline__ void smi_segment(uint8_t *zt, uint32_t nb, uint32_t count, const uint64_t *thresh, u128 &s,
                                            u128 inc, uint32_t &words, bool lh, const ChaKey &ck, ChaCursor &cur,
                                            bool naive) {
    // ub, the product of the segment's first K bounds, bounds every later batch's product and so
    // its threshold: the exact threshold is read only below it (the carried bound of
    // shuffle.py:118-128); n <= 64 and K <= 8 keep it below 2^48
    uint64_t ub = 1;
#pragma unroll
    for (int m = 0; m < K; ++m) ub *= (uint64_t)(nb - m);
    words += count;
    for (uint32_t c = 0; c < count; ++c, nb -= K) {
        uint32_t d[K];
        uint64_t r;
        auto draw = [&]() {
            if constexpr (CHA) {
                s = cha_add(s, 1);
                r = cha_out_cached(ck, cur, s);
            } else {
                s = mad128_wide(s, gen_mult(lh), inc);  // 17 SASS instead of mad128's 25
                r = gen_out(s, lh);
            }
            if (K == 2 && naive) {
                naive_pair(nb, r, d[0], d[K - 1]);
            } else {
#pragma unroll
                for (int m = 0; m < K; ++m) d[m] = die(nb - m, r);
            }
        };
        draw();
        if (r < ub) {
            const uint64_t t = __ldg(thresh + c);
            while (r < t) {  // reject: re-draw the whole batch (shuffle.py:121-128)
                draw();
                ++words;
            }
        }
        // nb = 4a + R: the batch's own positions are constant offsets from row a once R is known
        uint8_t *za = zt + (nb >> 2) * 128u;
        switch (nb & 3u) {
            case 0: smi_swaps<K, 0>(zt, za, d); break;
            case 1: smi_swaps<K, 1>(zt, za, d); break;
            case 2: smi_swaps<K, 2>(zt, za, d); break;
            default: smi_swaps<K, 3>(zt, za, d); break;
        }
    }
}

template <bool CHA>
__device__ __forceinline__ void smi_segment_any(uint8_t *zt, uint32_t k, uint32_t nb, uint32_t count,
                                                const uint64_t *thresh, u128 &s, u128 inc, uint32_t &words, bool lh,
                                                const ChaKey &ck, ChaCursor &cur, bool naive) {
    switch (k) {
        case 1: smi_segment<1, CHA>(zt, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 2: smi_segment<2, CHA>(zt, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 3: smi_segment<3, CHA>(zt, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 4: smi_segment<4, CHA>(zt, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 5: smi_segment<5, CHA>(zt, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 6: smi_segment<6, CHA>(zt, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        case 7: smi_segment<7, CHA>(zt, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
        default: smi_segment<8, CHA>(zt, nb, count, thresh, s, inc, words, lh, ck, cur, naive); break;
    }
}

template <typename T, bool CHA, int NF = 0, int TB = SMI_T>  // NF: n known at compile time (0: runtime); TB: threads
__global__ void __launch_bounds__(TB, SMI_MINB * SMI_T / TB) shuffle_small_idx_kernel(T *__restrict__ data, int64_t num_arrays,
                                                                 DevPlan plan, uint64_t run_seed, int64_t base,
                                                                 uint32_t *__restrict__ words_out, int gen) {
    __shared__ __align__(16) uint32_t wr[TB / 32][SMI_WW];
    __shared__ DevSeg segs[MAX_SEGS];
    const uint32_t n = plan.n;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t *W = wr[wid];
    const int64_t a = (int64_t)blockIdx.x * TB + tid;
    if (tid < (int)plan.nseg) segs[tid] = plan.segs[tid];
#pragma unroll
    for (int w = 0; w < 16; ++w)  // NF == 64: token j names its owner lane j / 2 and half j & 1 (bit 5)
        W[w * 32 + lane] = NF == 64 ? 0x21012000u + 0x02020202u * (uint32_t)w : 0x03020100u + 0x04040404u * (uint32_t)w;
    {  // the warp's payload span (32 arrays) is pulled into L2 while the permutations are built
        const int64_t aw0 = (int64_t)blockIdx.x * TB + wid * 32;
        const int64_t cnt0 = min((int64_t)32, num_arrays - aw0);
        if (cnt0 > 0) {
            const char *p0 = reinterpret_cast<const char *>(data + aw0 * (int64_t)n);
            const uint64_t span = (uint64_t)cnt0 * n * sizeof(T);
            for (uint64_t off = (uint64_t)lane * 128; off < span; off += 32 * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p0 + off));
        }
    }
    __syncthreads();
    if (a < num_arrays) {
        u128 s, inc;
        const bool lh = gen == 1;
        ChaKey ck;
        ChaCursor cur;
        cur.valid = false;
        const uint64_t seed = array_seed(run_seed, (uint64_t)(base + a));
        if constexpr (CHA) {
            chacha_seed(seed, ck);
            s = mk128(0, 0);
            inc = mk128(ck.nonce, CHACHA_TAG);
        } else {
            gen_seed(seed, s, inc, lh);
        }
        uint8_t *zt = reinterpret_cast<uint8_t *>(W) + lane * 4;
        uint32_t words = 0;
        for (uint32_t sg = 0; sg < plan.nseg; ++sg) {
            const DevSeg S = segs[sg];
            smi_segment_any<CHA>(zt, S.k, S.start_n, S.count, plan.thresh + S.first_batch, s, inc, words, lh, ck, cur,
                                 plan.naive != 0);
        }
        if (words_out) words_out[a] = words;
    }
    __syncwarp();
    {  // transposed -> rows: lane l's permutation at W[17 l ..]
        uint32_t mine[16];
#pragma unroll
        for (int w = 0; w < 16; ++w) mine[w] = W[w * 32 + lane];
        __syncwarp();
#pragma unroll
        for (int w = 0; w < 16; ++w) W[17 * lane + w] = mine[w];
        __syncwarp();
    }
    const int64_t aw = (int64_t)blockIdx.x * TB + wid * 32;
    const int cnt = (int)min((int64_t)32, num_arrays - aw);
    const uint32_t l0 = (uint32_t)lane, l1 = (uint32_t)lane + 32;
    constexpr int U = SMI_U;
    if (NF == 64 && cnt == 32 && (reinterpret_cast<uintptr_t>(data) & (2 * sizeof(T) - 1)) == 0) {
        // the C3 shape: lane l moves items 2l, 2l+1 as one vector; SHFL reads the token's low 5 bits
        using P = SmiPair<T>;
        constexpr int UF = sizeof(T) == 4 ? 4 : 2;  // arrays per step, loaded one step ahead
        P *gw = reinterpret_cast<P *>(data + aw * 64) + lane;
        P v[2][UF];
        auto load = [&](P (&b)[UF], int t0) {
#pragma unroll
            for (int u = 0; u < UF; ++u) b[u] = gw[(t0 + u) * 32];
        };
        auto apply = [&](P (&b)[UF], int t0) {
#pragma unroll
            for (int u = 0; u < UF; ++u) {
                const uint32_t xx = reinterpret_cast<const uint16_t *>(W + 17 * (t0 + u))[lane];
                const uint32_t x0 = xx, x1 = xx >> 8;
                const T a0 = smi_shfl(b[u].a, (int)x0), b0 = smi_shfl(b[u].b, (int)x0);
                const T a1 = smi_shfl(b[u].a, (int)x1), b1 = smi_shfl(b[u].b, (int)x1);
                P o;
                o.a = (x0 & 32) ? b0 : a0;
                o.b = (x1 & 32) ? b1 : a1;
                gw[(t0 + u) * 32] = o;
            }
        };
        load(v[0], 0);
#pragma unroll 1
        for (int t0 = 0; t0 < 32; t0 += 2 * UF) {
            load(v[1], t0 + UF);
            apply(v[0], t0);
            if (t0 + 2 * UF < 32) load(v[0], t0 + 2 * UF);
            apply(v[1], t0 + UF);
        }
        return;
    }
    const bool in0 = l0 < n, in1 = l1 < n;
    T *gw = data + aw * (int64_t)n;  // the warp's 32 arrays, contiguous
    for (int t0 = 0; t0 < cnt; t0 += U, gw += (int64_t)U * n) {
        T v0[U], v1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const T *g = gw + u * n;
            const bool ok = t0 + u < cnt;
            v0[u] = ok && in0 ? g[l0] : T(0);
            v1[u] = ok && in1 ? g[l1] : T(0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint8_t *row = reinterpret_cast<const uint8_t *>(W + 17 * (t0 + u));
            uint32_t x0 = row[l0], x1 = row[l1];  // (bytes past n are never used)
            if (NF == 64) {  // undo the (lane, half) token form
                x0 = ((x0 & 31) << 1) | (x0 >> 5);
                x1 = ((x1 & 31) << 1) | (x1 >> 5);
            }
            const T a0 = smi_shfl(v0[u], (int)(x0 & 31)), b0 = smi_shfl(v1[u], (int)(x0 & 31));
            const T a1 = smi_shfl(v0[u], (int)(x1 & 31)), b1 = smi_shfl(v1[u], (int)(x1 & 31));
            T *g = gw + u * n;
            if (t0 + u < cnt) {
                if (in0) g[l0] = (x0 & 32) ? b0 : a0;
                if (in1) g[l1] = (x1 & 32) ? b1 : a1;
            }
        }
    }
}

// -------------------------------------------------------------------------------------
// one warp per array
// -------------------------------------------------------------------------------------
static constexpr unsigned FULL = 0xFFFFFFFFu;

template <typename T>
__device__ __forceinline__ T shfl_t(T v, int src) {
    if constexpr (sizeof(T) == 8) {
        uint64_t x = (uint64_t)v;
        uint32_t lo = __shfl_sync(FULL, (uint32_t)x, src), hi = __shfl_sync(FULL, (uint32_t)(x >> 32), src);
        return (T)(((uint64_t)hi << 32) | lo);
    } else {
        return (T)__shfl_sync(FULL, (uint32_t)v, src);
    }
}

// warp copy (fallback when the array is not 16-byte sized/aligned for the bulk engine):
// U independent loads in flight per lane before the stores
template <typename T>
__device__ __forceinline__ void warp_copy(T *__restrict__ dst, const T *__restrict__ src, uint32_t n, int lane) {
    constexpr int U = 8;
    for (uint32_t e0 = 0; e0 < n; e0 += 32 * U) {
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t e = e0 + 32 * u + lane;
            if (e < n) v[u] = src[e];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t e = e0 + 32 * u + lane;
            if (e < n) dst[e] = v[u];
        }
    }
}

// Word/target generator of one array for the warp-per-array kernel.  Lane l evaluates
// batch B0+l on word B0+D+l; a rejected batch shifts every later batch by one word
// (shuffle.py:121-128), handled by realigning the lane states.  Targets are written into a
// ring indexed by position (RING entries), just ahead of the groups that consume them.
static constexpr uint32_t RING = 1024;

struct GenState {
    u128 s, inc, A32, C32;
    u128 W0;                        // ChaCha: origin of the warp's keystream window
    uint32_t B0, D, seg, frontier;  // frontier: lowest position whose target is committed
};

template <bool CHA>
__device__ __forceinline__ void gen_init(GenState &g, u128 s0, u128 inc, uint32_t n, int lane) {
    const bool lh = is_lehmer(inc);
    g.inc = inc;
    if constexpr (CHA) {
        g.s = cha_add(s0, (uint64_t)lane + 1);
        g.W0 = cha_win_unset(s0);
    } else {
        g.s = gen_jump_small(s0, inc, lane + 1, lh);
        g.A32 = gen_SA(lh, 32);
        g.C32 = mul128(g_SG[32], inc);
    }
    g.B0 = 0;
    g.D = 0;
    g.seg = 0;
    g.frontier = n;
}

// One generation step: 32 batches evaluated, the accepted prefix committed.
template <bool CHA, typename Sink>
__device__ __forceinline__ void gen_step(GenState &g, const DevPlan &plan, const DevSeg *segs, Sink sink, int lane,
                                         uint64_t *rk_first, uint64_t *chawin, const ChaKey &ck) {
    const bool lh = is_lehmer(g.inc);
    const uint32_t nb = plan.nbatches;
    const uint32_t b = g.B0 + lane;
    bool fail = false;
    uint32_t low = 0xFFFFFFFFu;  // lowest position this lane's batch covers
    uint64_t rc = 0;
    if constexpr (CHA) rc = cha_warp_word(chawin, ck, g.W0, cha_prev(g.s), lane);  // warp-collective
    if (b < nb) {
        uint32_t sg = g.seg;
        while (sg + 1 < plan.nseg && segs[sg + 1].first_batch <= b) ++sg;
        const DevSeg S = segs[sg];
        const uint32_t nbb = S.start_n - (b - S.first_batch) * S.k;
        const uint64_t t = __ldg(plan.thresh + b);
        uint64_t r = CHA ? rc : gen_out(g.s, lh);
        const uint32_t pos = nbb - 1;
        if (plan.naive && S.k == 2) {
            uint32_t j1, j2;
            naive_pair(nbb, r, j1, j2);
            sink(pos, j1);
            sink(pos - 1, j2);
        } else {
            for (uint32_t m = 0; m < S.k; ++m) sink(pos - m, die(nbb - m, r));
        }
        low = nbb - S.k;
        fail = r < t;
        if (rk_first && b == 0 && g.D == 0) *rk_first = r;
    }
    const unsigned fm = __ballot_sync(FULL, fail);
    const unsigned active = __ballot_sync(FULL, b < nb);
    // committed lanes: all active ones, or those before the first rejection
    const unsigned commit = fm ? (active & ((fm & (0u - fm)) - 1u)) : active;
    if (commit) {
        const int lastc = 31 - __clz(commit);
        g.frontier = __shfl_sync(FULL, low, lastc);
    }
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
    while (g.seg + 1 < plan.nseg && segs[g.seg + 1].first_batch <= g.B0) ++g.seg;
}

// Apply the steps at positions top, top-1, ..., top-31 (>= lim) of the sequential
// Fisher-Yates z[i] <-> z[J[i]] (i descending) as one warp step.  Lane l owns step
// i_l = top-l with target j_l <= i_l.  Within the group:
//   A_l = value at i_l just before step l = A_{Pred(l)} if some earlier lane m targeted
//         i_l (Pred(l) = latest such m) else z[i_l];
//   B_l = value at j_l just before step l = A_{T(l)} if some earlier lane targeted j_l
//         (T(l) = latest such) else z[j_l];
//   final z[i_l] = B_l; positions below the group receive A of their last toucher.
// Positions above the group are final and positions inside it are finalised here, so the
// result equals the sequential loop (checked bit-exactly against the oracle).
// Most groups have neither an in-group target (one vote) nor a repeated target (exact
// check through the per-array lane-id table H indexed by target): they take the direct
// path.  The rest resolve Pred chains with ballots + pointer jumping and T with a
// radix ballot over the bits of j.
template <typename T, uint32_t RSIZE = RING>
__device__ __forceinline__ void apply_group(T *z, const uint16_t *ring, uint8_t *H, int8_t *P, uint32_t top,
                                            uint32_t lim, int jbits, int lane) {
    const int64_t i64 = (int64_t)top - lane;
    const bool act = i64 >= (int64_t)lim;
    const uint32_t i = act ? (uint32_t)i64 : 0;
    const uint32_t j = act ? (uint32_t)ring[i & (RSIZE - 1)] : 0;
    const T vi = act ? z[i] : T(0);
    const T vj = act ? z[j] : T(0);
    const uint32_t lo_pos = top >= lim + 31 ? top - 31 : lim;
    // round 1: every lane claims H[j]; the survivor of a repeated target is arbitrary
    if (act) H[j] = (uint8_t)lane;
    P[lane] = -1;
    const bool inrange = act && j >= lo_pos && j < i;
    __syncwarp();
    const uint32_t w = act ? H[j] : (uint32_t)lane;
    const bool dupl = w != (uint32_t)lane;
    const unsigned flags = __ballot_sync(FULL, inrange) | __ballot_sync(FULL, dupl);
    if (flags == 0) {  // direct path: independent swaps
        if (act) {
            z[i] = vj;
            z[j] = vi;
        }
        __syncwarp();
        return;
    }
    // round 2: the losers of round 1 announce themselves; the round-1 survivor learns its
    // partner.  A loser that is overwritten again means three or more lanes share j.
    unsigned same = 1u << lane;
    if (__any_sync(FULL, dupl)) {
        __syncwarp();
        if (dupl) H[j] = (uint8_t)lane;
        __syncwarp();
        const uint32_t h2 = act ? H[j] : (uint32_t)lane;
        const uint32_t partner = dupl ? w : h2;
        const bool triple = dupl && h2 != (uint32_t)lane;
        if (__any_sync(FULL, triple)) {  // rare: radix ballot over the bits of j
            same = __ballot_sync(FULL, act);
#pragma unroll 1
            for (int q = 0; q < jbits; ++q) {
                const unsigned bq = __ballot_sync(FULL, (j >> q) & 1u);
                same &= ((j >> q) & 1u) ? bq : ~bq;
            }
            if (!act) same = 1u << lane;
        } else {
            same |= (1u << partner);
        }
    }
    const unsigned below = (1u << lane) - 1u;
    const unsigned tm = same & below;
    const unsigned later = same & ~((2u << lane) - 1u);
    // Pred(l): the last earlier lane whose target is i_l (unique writer: the last toucher of j)
    if (inrange && later == 0) P[top - j] = (int8_t)lane;
    __syncwarp();
    int p = P[lane];
    p = p >= 0 ? p : lane;
#pragma unroll 1
    for (int it = 0; it < 5; ++it) {  // pointer jumping to the root of the Pred chain
        const int pp = __shfl_sync(FULL, p, p);
        if (!__any_sync(FULL, pp != p)) break;
        p = pp;
    }
    const T A = shfl_t(vi, p);
    const T At = shfl_t(A, tm ? 31 - __clz(tm) : lane);
    const T B = tm ? At : vj;
    if (act) {
        z[i] = B;
        if (later == 0 && j < lo_pos) z[j] = A;
    }
    __syncwarp();
}

// CM (ChaCha mode): 0 = PCG64/Lehmer only, 1 = ChaCha only, 2 = decided per array from the
// stream state's tag (stream calls, where only the device knows the generator).
template <typename T, bool SEGMENTED, bool CHA>
__device__ __forceinline__ void shuffle_mid_body(T *__restrict__ data, int64_t num_arrays, const DevPlan &plan,
                                                 uint32_t zbytes, uint64_t run_seed, int64_t base,
                                                 uint32_t *__restrict__ words32, uint64_t *state_io,
                                                 uint64_t *words64, uint64_t *rk_first, int use_tma, int gen,
                                                 unsigned char *smem_raw, DevSeg *segs, uint16_t *ring,
                                                 int8_t *predslot, uint64_t &bar, uint64_t *chawin) {
    const int lane = threadIdx.x & 31;
    T *z = reinterpret_cast<T *>(smem_raw);
    uint8_t *H = smem_raw + zbytes;
    for (uint32_t q = lane; q < plan.nseg; q += 32) segs[q] = plan.segs[q];
    if (use_tma && lane == 0) mbar_init(&bar, 1);
    __syncwarp();
    const uint32_t n = plan.n;
    const uint32_t bytes = n * (uint32_t)sizeof(T);
    const uint32_t lim = plan.lo > 1 ? plan.lo : 1;
    const int jbits = n > 1 ? 32 - __clz(n - 1) : 1;
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
        GenState gs;
        gen_init<CHA>(gs, s0, inc, n, lane);
        uint64_t *rkf = SEGMENTED ? nullptr : rk_first;
        // the first targets are generated while the payload streams in
        uint16_t *ringp = ring;
        auto sink = [ringp](uint32_t pos, uint32_t v) { ringp[pos & (RING - 1)] = (uint16_t)v; };
        if (plan.nbatches) gen_step<CHA>(gs, plan, segs, sink, lane, rkf, chawin, ck);
        if (use_tma) {
            mbar_wait(&bar, parity);
            parity ^= 1u;
        }
        __syncwarp();
        for (int64_t top = (int64_t)n - 1; top >= (int64_t)lim; top -= 32) {
            const uint32_t need = top >= (int64_t)lim + 31 ? (uint32_t)top - 31 : lim;
            while (gs.frontier > need && gs.B0 < plan.nbatches)
                gen_step<CHA>(gs, plan, segs, sink, lane, rkf, chawin, ck);
            apply_group<T>(z, ring, H, predslot, (uint32_t)top, lim, jbits, lane);
        }
        // finish the word accounting (a trailing rejection can follow the last position)
        while (gs.B0 < plan.nbatches) gen_step<CHA>(gs, plan, segs, sink, lane, rkf, chawin, ck);
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

template <typename T, bool SEGMENTED, int CM>
__global__ void __launch_bounds__(32) shuffle_mid_kernel(T *__restrict__ data, int64_t num_arrays, DevPlan plan,
                                                         uint32_t zbytes, uint64_t run_seed, int64_t base,
                                                         uint32_t *__restrict__ words32, uint64_t *state_io,
                                                         uint64_t *words64, uint64_t *rk_first, int use_tma, int gen) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ DevSeg segs[MAX_SEGS];
    __shared__ __align__(16) uint16_t ring[RING];
    __shared__ int8_t predslot[32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(16) uint64_t chawin[CM ? 256 : 2];
    bool cha = CM == 1;
    if constexpr (CM == 2) cha = is_posgen(mk128(state_io[2], state_io[3]));
    if (CM != 0 && cha)
        shuffle_mid_body<T, SEGMENTED, CM != 0>(data, num_arrays, plan, zbytes, run_seed, base, words32, state_io,
                                                words64, rk_first, use_tma, gen, smem_raw, segs, ring, predslot,
                                                bar, chawin);
    else if (CM != 1)
        shuffle_mid_body<T, SEGMENTED, false>(data, num_arrays, plan, zbytes, run_seed, base, words32, state_io,
                                              words64, rk_first, use_tma, gen, smem_raw, segs, ring, predslot, bar,
                                              chawin);
}


// -------------------------------------------------------------------------------------
// one CTA (W warps) per array: groups of G = 32*W steps
// -------------------------------------------------------------------------------------
// Same resolution as apply_group, done across the CTA through shared memory and barriers:
// the serial chain per array is n/G groups instead of n/32, and W warps share the target
// generation.  Groups with three or more lanes on one target, and the bottom of the array
// (where such groups are common), fall back to warp groups run by warp 0.
#ifndef BR_CRING
#define BR_CRING 2048
#endif
static constexpr uint32_t CRING = BR_CRING;

template <int W>
struct CtaGen {
    u128 s, inc, AJ, CJ;
    u128 W0;  // ChaCha: origin of the CTA's keystream window
    uint32_t B0, D, seg, frontier, parity;
};

// -------------------------------------------------------------------------------------
// arrays in global memory: one CTA (W warps) per array, groups of G = 32*W steps
// -------------------------------------------------------------------------------------
// Targets are generated in-CTA into a u32 ring (no global target buffer).  Repeated
// targets are found exactly with one ballot per bit of j in every warp; lane L combines the
// W*jbits masks through shared memory, which yields T(L) and "later" for any multiplicity.
static constexpr uint32_t LRING = 4096;  // u32 target ring of the large kernel (up to 16 warps)
// ring of the large kernel for W warps: one generation step (32W batches of up to k dice) and
// one group ahead of the group being applied
constexpr uint32_t large_ring(int W) { return W > 16 ? 8192u : LRING; }
#ifndef BR_LARGE_HB
#define BR_LARGE_HB 11
#endif
static constexpr int HBITS = BR_LARGE_HB;  // 2048-slot lane-chain hash per group

template <typename T, int W, typename RT = uint32_t, uint32_t RS = LRING, int HB = HBITS>
struct LargeShared {
    static constexpr uint32_t RSIZE = RS;
    using RType = RT;
    DevSeg segs[MAX_SEGS];
    RT ring[RS];
    uint32_t ht[1 << HB];  // (group tag << 16) | (lane + 1) of the last lane hashed here
    int16_t nxt[32 * W];      // previous lane in the same slot (-1: none)
    uint32_t jv[32 * W];
    int16_t P[32 * W];
    T VI[32 * W];
    T AV[32 * W];
    uint32_t fmin;
    uint32_t frontier[2];
};

// FG: the group is full (top >= lim + G - 1), every thread has a step
template <bool FG = false, typename T, int W, typename RT, uint32_t RS, int HB>
__device__ __forceinline__ void apply_group_cta_global(T *z, LargeShared<T, W, RT, RS, HB> &sh, uint32_t tag,
                                                       uint32_t top, uint32_t lim, int L) {
    constexpr int G = 32 * W;
    const bool act = FG || top >= lim + (uint32_t)L;  // 32-bit: lim + L < 2^32 for n < 2^32
    const uint32_t i = top - (uint32_t)L;
    const uint32_t j = act ? (uint32_t)sh.ring[i & (RS - 1)] : 0;
    const T vi = act ? z[i] : T(0);
    const T vj = act ? z[j] : T(0);
    const uint32_t lo_pos = (FG || top >= lim + (G - 1)) ? top - (G - 1) : lim;
    const bool inrange = act && j >= lo_pos && j < i;
    // lanes with equal targets meet in a hash slot; each slot keeps a chain of its lanes
    const uint32_t h = (j * 2654435761u) >> (32 - HB);
    int16_t link = -1;
    if (act) {
        const uint32_t old = atomicExch(&sh.ht[h], (tag << 16) | (uint32_t)(L + 1));
        if ((old >> 16) == tag) link = (int16_t)((old & 0xFFFFu) - 1);
    }
    sh.nxt[L] = link;
    sh.jv[L] = j;
    sh.P[L] = -1;
    sh.VI[L] = vi;
    __syncthreads();
    int tl = -1;
    bool later = false;
    if (act) {
        const uint32_t head = sh.ht[h];
        for (int t = (int)(head & 0xFFFFu) - 1; t >= 0; t = sh.nxt[t]) {
            if (t != L && sh.jv[t] == j) {
                if (t < L) tl = t > tl ? t : tl;
                else later = true;
            }
        }
    }
    if (inrange && !later) sh.P[top - j] = (int16_t)L;
    __syncthreads();
    int p = sh.P[L];
    p = p >= 0 ? p : L;
    for (;;) {
        const int pp = sh.P[p];
        const int np = pp >= 0 ? pp : p;
        if (!__syncthreads_or(np != p)) break;
        p = np;
    }
    const T A = sh.VI[p];
    sh.AV[L] = A;
    __syncthreads();
    const T B = tl >= 0 ? sh.AV[tl] : vj;
    if (act) {
        z[i] = B;
        if (!later && j < lo_pos) z[j] = A;
    }
    __syncthreads();
}

// One CTA generation step into the target ring of any shared layout Sh (segs, ring[RSIZE],
// frontier[2], fmin).
template <bool CHA, int W, typename Sh>
__device__ __forceinline__ void large_gen_step(CtaGen<W> &g, const DevPlan &plan, Sh &sh, int L, uint64_t *rk_first,
                                               uint64_t *chawin, const ChaKey &ck) {
    constexpr uint32_t RS = Sh::RSIZE;
    using RT = typename Sh::RType;
    const bool lh = is_lehmer(g.inc);
    constexpr int G = 32 * W;
    const uint32_t nb = plan.nbatches;
    const uint32_t b = g.B0 + L;
    bool fail = false;
    uint32_t low = 0xFFFFFFFFu;
    uint64_t rc = 0;
    if constexpr (CHA) rc = cha_cta_word<G>(chawin, ck, g.W0, cha_prev(g.s), L);  // CTA-collective
    if (b < nb) {
        uint32_t sg = g.seg;
        while (sg + 1 < plan.nseg && sh.segs[sg + 1].first_batch <= b) ++sg;
        const DevSeg S = sh.segs[sg];
        const uint32_t nbb = S.start_n - (b - S.first_batch) * S.k;
        const uint64_t t = __ldg(plan.thresh + b);
        uint64_t r = CHA ? rc : gen_out(g.s, lh);
        const uint32_t pos = nbb - 1;
        if (plan.naive && S.k == 2) {
            uint32_t j1, j2;
            naive_pair(nbb, r, j1, j2);
            sh.ring[pos & (RS - 1)] = (RT)j1;
            sh.ring[(pos - 1) & (RS - 1)] = (RT)j2;
        } else {
            for (uint32_t m = 0; m < S.k; ++m) sh.ring[(pos - m) & (RS - 1)] = (RT)die(nbb - m, r);
        }
        low = nbb - S.k;
        fail = r < t;
        if (rk_first && b == 0 && g.D == 0) *rk_first = r;
    }
    const uint32_t nact = nb - g.B0 < (uint32_t)G ? nb - g.B0 : (uint32_t)G;
    const uint32_t par = g.parity;
    g.parity ^= 1u;
    if (L == (int)nact - 1) sh.frontier[par] = low;
    if (!__syncthreads_or(fail)) {
        g.frontier = sh.frontier[par];
        g.B0 += G;
        if constexpr (CHA) g.s = cha_add(g.s, G);
        else g.s = mad128(g.s, g.AJ, g.CJ);
    } else {
        if (L == 0) sh.fmin = G;
        __syncthreads();
        if (fail) atomicMin(&sh.fmin, (uint32_t)L);
        __syncthreads();
        const uint32_t f = sh.fmin;
        if (f > 0 && L == (int)f - 1) sh.frontier[par] = low;
        __syncthreads();
        if (f > 0) g.frontier = sh.frontier[par];
        g.B0 += f;
        g.D += 1;
        if constexpr (CHA) g.s = cha_add(g.s, (uint64_t)f + 1);
        else g.s = gen_jump_small(g.s, g.inc, (int)f + 1, lh);
        __syncthreads();
    }
    while (g.seg + 1 < plan.nseg && sh.segs[g.seg + 1].first_batch <= g.B0) ++g.seg;
}

// per-array generator setup shared by the CTA kernels
template <bool CHA, int W>
__device__ __forceinline__ void cta_gen_setup(CtaGen<W> &gs, u128 &s0, u128 &inc, bool &lh, ChaKey &ck, int segmented,
                                              int gen, uint64_t run_seed, int64_t a, uint64_t *state_io, uint32_t n,
                                              int L) {
    constexpr int G = 32 * W;
    if (segmented) {
        lh = gen == 1;
        const uint64_t seed = array_seed(run_seed, (uint64_t)a);
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
    gs.inc = inc;
    if constexpr (CHA) {
        gs.s = cha_add(s0, (uint64_t)L + 1);
        gs.W0 = cha_win_unset(s0);
    } else {
        gs.s = gen_jump_small(s0, inc, L + 1, lh);
        gs.AJ = gen_SA(lh, G);
        gs.CJ = mul128(g_SG[G], inc);
    }
    gs.B0 = 0;
    gs.D = 0;
    gs.seg = 0;
    gs.frontier = n;
    gs.parity = 0;
}

template <typename T, int W, bool CHA>
__device__ __forceinline__ void shuffle_cta_large_body(T *__restrict__ data, int64_t num_arrays, const DevPlan &plan,
                                                       uint64_t run_seed, int64_t base, uint32_t *__restrict__ words32,
                                                       uint64_t *state_io, uint64_t *words64, uint64_t *rk_first,
                                                       int segmented, int gen,
                                                       LargeShared<T, W, uint32_t, large_ring(W)> &sh,
                                                       uint64_t *chawin, const uint32_t *only) {
    constexpr int G = 32 * W;
    const int L = threadIdx.x;
    for (uint32_t q = L; q < plan.nseg; q += G) sh.segs[q] = plan.segs[q];
    for (uint32_t q = L; q < (1u << HBITS); q += G) sh.ht[q] = 0;
    __syncthreads();
    uint32_t tag = 0;
    const uint32_t n = plan.n;
    const uint32_t lim = plan.lo > 1 ? plan.lo : 1;
    for (int64_t a = blockIdx.x; a < num_arrays; a += gridDim.x) {
        if (only && !only[a]) continue;  // re-run of the arrays another kernel flagged
        T *z = data + a * (int64_t)n;
        u128 s0, inc;
        bool lh;
        ChaKey ck;
        CtaGen<W> gs;
        cta_gen_setup<CHA, W>(gs, s0, inc, lh, ck, segmented, gen, run_seed, base + a, state_io, n, L);
        uint64_t *rkf = segmented ? nullptr : rk_first;
        for (int64_t top = (int64_t)n - 1; top >= (int64_t)lim; top -= G) {
            const uint32_t need = top >= (int64_t)lim + (G - 1) ? (uint32_t)top - (G - 1) : lim;
            while (gs.frontier > need && gs.B0 < plan.nbatches) large_gen_step<CHA, W>(gs, plan, sh, L, rkf, chawin, ck);
            tag = (tag + 1) & 0xFFFFu;
            if (tag == 0) {  // tag wrap: clear the slots (every 65535 groups)
                for (uint32_t q = L; q < (1u << HBITS); q += G) sh.ht[q] = 0;
                tag = 1;
                __syncthreads();
            }
            apply_group_cta_global(z, sh, tag, (uint32_t)top, lim, L);
        }
        while (gs.B0 < plan.nbatches) large_gen_step<CHA, W>(gs, plan, sh, L, rkf, chawin, ck);
        const uint64_t words = (uint64_t)plan.nbatches + gs.D;
        if (L == 0) {
            if (segmented) {
                if (words32) words32[a] = (uint32_t)words;
            } else {
                const u128 sf = CHA ? cha_add(s0, words) : gen_jump(s0, inc, words, lh);
                state_io[0] = sf.hi;
                state_io[1] = sf.lo;
                if (words64) words64[0] = words;
            }
        }
        __syncthreads();
    }
}

template <typename T, int W>
constexpr size_t large_smem_bytes(bool chacha) {
    return ((sizeof(LargeShared<T, W, uint32_t, large_ring(W)>) + 15) & ~(size_t)15) +
           (chacha ? (size_t)8 * 32 * W * sizeof(uint64_t) : 0);
}

template <typename T, int W, int CM>
__global__ void __launch_bounds__(32 * W) shuffle_cta_large_kernel(T *__restrict__ data, int64_t num_arrays,
                                                                   DevPlan plan, uint64_t run_seed, int64_t base,
                                                                   uint32_t *__restrict__ words32, uint64_t *state_io,
                                                                   uint64_t *words64, uint64_t *rk_first,
                                                                   int segmented, int gen,
                                                                   const uint32_t *__restrict__ only) {
    // dynamic shared memory: the CTA's tables, then the ChaCha keystream window (8 words per
    // thread) when the launch asks for one; sizes set at launch (large_smem_bytes)
    extern __shared__ __align__(16) unsigned char large_smem[];
    auto &sh = *reinterpret_cast<LargeShared<T, W, uint32_t, large_ring(W)> *>(large_smem);
    uint64_t *chawin = reinterpret_cast<uint64_t *>(large_smem + ((sizeof(sh) + 15) & ~(size_t)15));
    bool cha = CM == 1;
    if constexpr (CM == 2) cha = is_posgen(mk128(state_io[2], state_io[3]));
    if (CM != 0 && cha)
        shuffle_cta_large_body<T, W, CM != 0>(data, num_arrays, plan, run_seed, base, words32, state_io, words64,
                                              rk_first, segmented, gen, sh, chawin, only);
    else if (CM != 1)
        shuffle_cta_large_body<T, W, false>(data, num_arrays, plan, run_seed, base, words32, state_io, words64,
                                            rk_first, segmented, gen, sh, chawin, only);
}

// Shared-memory-resident arrays with the same hashed CTA groups: payload moved by TMA bulk
// copies, targets in a u16 ring, 1024-slot lane-chain hash.
#ifndef BR_HASH_HB
#define BR_HASH_HB 10
#endif
static constexpr int HASH_HB = BR_HASH_HB;

template <typename T, int W, bool CHA>
__device__ __forceinline__ void shuffle_cta_hash_body(T *__restrict__ data, int64_t num_arrays, const DevPlan &plan,
                                                      uint64_t run_seed, int64_t base, uint32_t *__restrict__ words32,
                                                      uint64_t *state_io, uint64_t *words64, uint64_t *rk_first,
                                                      int use_tma, int segmented, int gen, unsigned char *smem_raw,
                                                      LargeShared<T, W, uint16_t, CRING, HASH_HB> &sh, uint64_t &bar,
                                                      uint64_t *chawin) {
    constexpr int G = 32 * W;
    constexpr int HB = HASH_HB;
    const int L = threadIdx.x;
    T *z = reinterpret_cast<T *>(smem_raw);
    for (uint32_t q = L; q < plan.nseg; q += G) sh.segs[q] = plan.segs[q];
    for (uint32_t q = L; q < (1u << HB); q += G) sh.ht[q] = 0;
    if (use_tma && L == 0) mbar_init(&bar, 1);
    __syncthreads();
    const uint32_t n = plan.n;
    const uint32_t bytes = n * (uint32_t)sizeof(T);
    const uint32_t lim = plan.lo > 1 ? plan.lo : 1;
    uint32_t parity = 0, tag = 0;
    for (int64_t a = blockIdx.x; a < num_arrays; a += gridDim.x) {
        T *g = data + a * (int64_t)n;
        if (use_tma) {
            if (L == 0) {
                bulk_wait_read();
                fence_proxy_async();
                mbar_arrive_expect_tx(&bar, bytes);
                bulk_load(z, g, bytes, &bar);
            }
        } else {
            for (uint32_t e = L; e < n; e += G) z[e] = g[e];
        }
        u128 s0, inc;
        bool lh;
        ChaKey ck;
        CtaGen<W> gs;
        cta_gen_setup<CHA, W>(gs, s0, inc, lh, ck, segmented, gen, run_seed, base + a, state_io, n, L);
        uint64_t *rkf = segmented ? nullptr : rk_first;
        if (plan.nbatches) large_gen_step<CHA, W>(gs, plan, sh, L, rkf, chawin, ck);  // overlaps the payload load
        if (use_tma) {
            mbar_wait(&bar, parity);
            parity ^= 1u;
        }
        __syncthreads();
        for (int64_t top = (int64_t)n - 1; top >= (int64_t)lim; top -= G) {
            const uint32_t need = top >= (int64_t)lim + (G - 1) ? (uint32_t)top - (G - 1) : lim;
            while (gs.frontier > need && gs.B0 < plan.nbatches) large_gen_step<CHA, W>(gs, plan, sh, L, rkf, chawin, ck);
            tag = (tag + 1) & 0xFFFFu;
            if (tag == 0) {
                for (uint32_t q = L; q < (1u << HB); q += G) sh.ht[q] = 0;
                tag = 1;
                __syncthreads();
            }
            if (top >= (int64_t)lim + (G - 1)) apply_group_cta_global<true>(z, sh, tag, (uint32_t)top, lim, L);
            else apply_group_cta_global<false>(z, sh, tag, (uint32_t)top, lim, L);
        }
        while (gs.B0 < plan.nbatches) large_gen_step<CHA, W>(gs, plan, sh, L, rkf, chawin, ck);
        if (use_tma) {
            if (L == 0) {
                fence_proxy_async();
                bulk_store(g, z, bytes);
            }
        } else {
            for (uint32_t e = L; e < n; e += G) g[e] = z[e];
        }
        const uint64_t words = (uint64_t)plan.nbatches + gs.D;
        if (L == 0) {
            if (segmented) {
                if (words32) words32[a] = (uint32_t)words;
            } else {
                const u128 sf = CHA ? cha_add(s0, words) : gen_jump(s0, inc, words, lh);
                state_io[0] = sf.hi;
                state_io[1] = sf.lo;
                if (words64) words64[0] = words;
            }
        }
        __syncthreads();
    }
    if (use_tma && L == 0) bulk_wait_all();
}

template <typename T, int W, int CM>
__global__ void __launch_bounds__(32 * W) shuffle_cta_hash_kernel(T *__restrict__ data, int64_t num_arrays,
                                                                  DevPlan plan, uint64_t run_seed, int64_t base,
                                                                  uint32_t *__restrict__ words32, uint64_t *state_io,
                                                                  uint64_t *words64, uint64_t *rk_first, int use_tma,
                                                                  int segmented, int gen) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ LargeShared<T, W, uint16_t, CRING, HASH_HB> sh;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(16) uint64_t chawin[CM ? 8 * 32 * W : 2];
    bool cha = CM == 1;
    if constexpr (CM == 2) cha = is_posgen(mk128(state_io[2], state_io[3]));
    if (CM != 0 && cha)
        shuffle_cta_hash_body<T, W, CM != 0>(data, num_arrays, plan, run_seed, base, words32, state_io, words64,
                                             rk_first, use_tma, segmented, gen, smem_raw, sh, bar, chawin);
    else if (CM != 1)
        shuffle_cta_hash_body<T, W, false>(data, num_arrays, plan, run_seed, base, words32, state_io, words64,
                                           rk_first, use_tma, segmented, gen, smem_raw, sh, bar, chawin);
}

// -------------------------------------------------------------------------------------
// one CTA per shared-memory-resident array, whole-array resolution (no group chain)
// -------------------------------------------------------------------------------------
// The sequential Fisher-Yates z[i] <-> z[J[i]] (i = n-1 .. lim) has a closed form.  Let
//   ns(i) = min{m > i : J[m] = J[i]}   (the next step, in index order, with i's target)
//   ft(x) = min{m > x : J[m] = x}      (the last step before x's own that targeted x)
//   F(x)  = x if ft(x) is undefined, else F(ft(x))
// Then the final value at position i >= lim is z0[F(ns(i))] if ns(i) exists, else z0[J[i]];
// below lim it is z0[F(i)].  (Position J[i] < i is only ever written by steps m with
// J[m] = J[i]; the most recent one before step i is ns(i), and the value it deposited is the
// one position ns(i) held just before its own step -- which is z0[F(ns(i))] by the same
// argument on ft.)  Checked against the sequential loop exhaustively in tests (oracle) and
// bit-exactly on the device.
//
// So one array costs: all targets (lane-parallel generation, G batches per step), one
// atomicExch per step to thread per-target lists, a list walk per position for ns and ft,
// pointer jumping on F, and one gather z0[r] per position written straight to global
// memory -- about ten barriers per array instead of five per 32*W steps.  Measured on B200
// it is slower than the hashed group kernel for many arrays (C4: 3.25 vs 2.49 ms: the
// divergent list walks and the jumping rounds cost more instructions than the barriers they
// save), but faster for ONE array, where the CTA's latency is the whole call (C1: 0.033 vs
// 0.070 ms with 512 threads); the dispatcher uses it for single-array stream calls.
static constexpr uint16_t RES_NONE = 0xFFFF;

template <bool CHA, int W>
__device__ __forceinline__ void gen_all_targets(CtaGen<W> &g, const DevPlan &plan, const DevSeg *segs,
                                                uint16_t *J, uint32_t *fmin, int L, uint64_t *rk_first,
                                                uint64_t *chawin, const ChaKey &ck) {
    constexpr int G = 32 * W;
    const bool lh = is_lehmer(g.inc);
    const uint32_t nb = plan.nbatches;
    while (g.B0 < nb) {
        const uint32_t b = g.B0 + L;
        bool fail = false;
        uint64_t rc = 0;
        if constexpr (CHA) rc = cha_cta_word<G>(chawin, ck, g.W0, cha_prev(g.s), L);  // CTA-collective
        if (b < nb) {
            uint32_t sg = g.seg;
            while (sg + 1 < plan.nseg && segs[sg + 1].first_batch <= b) ++sg;
            const DevSeg S = segs[sg];
            const uint32_t nbb = S.start_n - (b - S.first_batch) * S.k;
            const uint64_t t = __ldg(plan.thresh + b);
            uint64_t r = CHA ? rc : gen_out(g.s, lh);
            const uint32_t pos = nbb - 1;
            if (plan.naive && S.k == 2) {
                uint32_t j1, j2;
                naive_pair(nbb, r, j1, j2);
                J[pos] = (uint16_t)j1;
                J[pos - 1] = (uint16_t)j2;
            } else {
                for (uint32_t m = 0; m < S.k; ++m) J[pos - m] = (uint16_t)die(nbb - m, r);
            }
            fail = r < t;
            if (rk_first && b == 0 && g.D == 0) *rk_first = r;
        }
        // a rejected batch is re-drawn from the next word by the lane that lands on it in the
        // next step; it rewrites the same positions (barrier-separated)
        if (!__syncthreads_or(fail)) {
            g.B0 += G;
            if constexpr (CHA) g.s = cha_add(g.s, G);
            else g.s = mad128(g.s, g.AJ, g.CJ);
        } else {
            if (L == 0) *fmin = G;
            __syncthreads();
            if (fail) atomicMin(fmin, (uint32_t)L);
            __syncthreads();
            const uint32_t f = *fmin;
            g.B0 += f;
            g.D += 1;
            if constexpr (CHA) g.s = cha_add(g.s, (uint64_t)f + 1);
            else g.s = gen_jump_small(g.s, g.inc, (int)f + 1, lh);
            __syncthreads();
        }
        while (g.seg + 1 < plan.nseg && segs[g.seg + 1].first_batch <= g.B0) ++g.seg;
    }
}

// dynamic shared memory of the resolve kernel for n elements of T
template <typename T>
__host__ __device__ __forceinline__ uint32_t resolve_smem_bytes(uint32_t n) {
    const uint32_t zb = (n * (uint32_t)sizeof(T) + 15) & ~15u;
    const uint32_t h16 = (n * 2 + 15) & ~15u;
    const uint32_t h32 = (n * 4 + 15) & ~15u;
    return zb + 4 * h16 + h32;  // z0 | J | link | ns | p | head
}

template <typename T, int W, bool CHA>
__device__ __forceinline__ void shuffle_resolve_body(T *__restrict__ data, int64_t num_arrays, const DevPlan &plan,
                                                     uint64_t run_seed, int64_t base,
                                                     uint32_t *__restrict__ words32, uint64_t *state_io,
                                                     uint64_t *words64, uint64_t *rk_first, int use_tma,
                                                     int segmented, int gen, unsigned char *smem_raw, DevSeg *segs,
                                                     uint32_t *fmin, uint64_t &bar, uint64_t *chawin) {
    constexpr int G = 32 * W;
    const int L = threadIdx.x;
    const uint32_t n = plan.n;
    const uint32_t zb = (n * (uint32_t)sizeof(T) + 15) & ~15u, h16 = (n * 2 + 15) & ~15u;
    T *z0 = reinterpret_cast<T *>(smem_raw);
    uint16_t *J = reinterpret_cast<uint16_t *>(smem_raw + zb);
    uint16_t *link = reinterpret_cast<uint16_t *>(smem_raw + zb + h16);
    uint16_t *ns = reinterpret_cast<uint16_t *>(smem_raw + zb + 2 * h16);
    uint16_t *pp = reinterpret_cast<uint16_t *>(smem_raw + zb + 3 * h16);
    uint32_t *head = reinterpret_cast<uint32_t *>(smem_raw + zb + 4 * h16);
    for (uint32_t q = L; q < plan.nseg; q += G) segs[q] = plan.segs[q];
    if (use_tma && L == 0) mbar_init(&bar, 1);
    __syncthreads();
    const uint32_t bytes = n * (uint32_t)sizeof(T);
    const uint32_t lim = plan.lo > 1 ? plan.lo : 1;
    uint32_t parity = 0;
    for (int64_t a = blockIdx.x; a < num_arrays; a += gridDim.x) {
        T *g = data + a * (int64_t)n;
        if (use_tma) {
            if (L == 0) {
                fence_proxy_async();
                mbar_arrive_expect_tx(&bar, bytes);
                bulk_load(z0, g, bytes, &bar);
            }
        } else {
            for (uint32_t e = L; e < n; e += G) z0[e] = g[e];
        }
        for (uint32_t x = L; x < n; x += G) head[x] = 0;
        u128 s0, inc;
        bool lh;
        ChaKey ck;
        CtaGen<W> gs;
        cta_gen_setup<CHA, W>(gs, s0, inc, lh, ck, segmented, gen, run_seed, base + a, state_io, n, L);
        uint64_t *rkf = segmented ? nullptr : rk_first;
        gen_all_targets<CHA, W>(gs, plan, segs, J, fmin, L, rkf, chawin, ck);
        __syncthreads();
        // per-target lists of steps: head[c] = 1 + a step with target c, link[i] = 1 + the
        // step inserted before i into the same list (0 ends a list; n <= 65535)
        for (uint32_t i = lim + L; i < n; i += G) link[i] = (uint16_t)atomicExch(&head[J[i]], i + 1);
        __syncthreads();
        for (uint32_t x = L; x < n; x += G) {
            // ns(x) for a position with a step; ft(x) for every position (as F's parent)
            uint32_t best = RES_NONE;
            if (x >= lim) {
                for (uint32_t m = head[J[x]]; m != 0; m = link[m - 1])
                    if (m - 1 > x && m - 1 < best) best = m - 1;
                ns[x] = (uint16_t)best;
            }
            best = RES_NONE;
            for (uint32_t m = head[x]; m != 0; m = link[m - 1])
                if (m - 1 > x && m - 1 < best) best = m - 1;
            pp[x] = best == RES_NONE ? (uint16_t)x : (uint16_t)best;
        }
        // F by pointer jumping (in place: every value read is an ancestor, so races only
        // shorten the chains); the rounds end when no pointer moves
        for (;;) {
            __syncthreads();
            bool moved = false;
            for (uint32_t x = L; x < n; x += G) {
                const uint16_t q = pp[x], r = pp[q];
                if (r != q) {
                    pp[x] = r;
                    moved = true;
                }
            }
            if (!__syncthreads_or(moved)) break;
        }
        if (use_tma) {
            mbar_wait(&bar, parity);
            parity ^= 1u;
        }
        for (uint32_t i = L; i < n; i += G) {
            uint32_t r;
            if (i >= lim) {
                const uint16_t m = ns[i];
                r = m != RES_NONE ? pp[m] : J[i];
            } else {
                r = pp[i];
            }
            g[i] = z0[r];
        }
        const uint64_t words = (uint64_t)plan.nbatches + gs.D;
        if (L == 0) {
            if (segmented) {
                if (words32) words32[a] = (uint32_t)words;
            } else {
                const u128 sf = CHA ? cha_add(s0, words) : gen_jump(s0, inc, words, lh);
                state_io[0] = sf.hi;
                state_io[1] = sf.lo;
                if (words64) words64[0] = words;
            }
        }
        __syncthreads();  // z0 / lists are reused by the next array
    }
}

template <typename T, int W, int CM>
__global__ void __launch_bounds__(32 * W) shuffle_resolve_kernel(T *__restrict__ data, int64_t num_arrays,
                                                                 DevPlan plan, uint64_t run_seed, int64_t base,
                                                                 uint32_t *__restrict__ words32, uint64_t *state_io,
                                                                 uint64_t *words64, uint64_t *rk_first, int use_tma,
                                                                 int segmented, int gen) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ DevSeg segs[MAX_SEGS];
    __shared__ uint32_t fmin;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(16) uint64_t chawin[CM ? 8 * 32 * W : 2];
    bool cha = CM == 1;
    if constexpr (CM == 2) cha = is_posgen(mk128(state_io[2], state_io[3]));
    if (CM != 0 && cha)
        shuffle_resolve_body<T, W, CM != 0>(data, num_arrays, plan, run_seed, base, words32, state_io, words64,
                                            rk_first, use_tma, segmented, gen, smem_raw, segs, &fmin, bar, chawin);
    else if (CM != 1)
        shuffle_resolve_body<T, W, false>(data, num_arrays, plan, run_seed, base, words32, state_io, words64,
                                          rk_first, use_tma, segmented, gen, smem_raw, segs, &fmin, bar, chawin);
}

// -------------------------------------------------------------------------------------
// arrays larger than shared memory: targets into a global buffer, then warp-group apply
// on the array in global memory
// -------------------------------------------------------------------------------------
template <bool SEGMENTED, bool CHA>
__device__ __forceinline__ void shuffle_large_gen_body(int64_t num_arrays, const DevPlan &plan, uint64_t run_seed,
                                                       int64_t base, uint32_t *__restrict__ J,
                                                       uint32_t *__restrict__ words32, uint64_t *state_io,
                                                       uint64_t *words64, uint64_t *rk_first, int gen, DevSeg *segs,
                                                       uint64_t *chawin) {
    const int lane = threadIdx.x & 31;
    const uint32_t n = plan.n;
    for (int64_t a = blockIdx.x; a < num_arrays; a += gridDim.x) {
        uint32_t *Ja = J + a * (int64_t)n;
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
        GenState gs;
        gen_init<CHA>(gs, s0, inc, n, lane);
        auto sink = [Ja](uint32_t pos, uint32_t v) { Ja[pos] = v; };
        uint64_t *rkf = SEGMENTED ? nullptr : rk_first;
        while (gs.B0 < plan.nbatches) gen_step<CHA>(gs, plan, segs, sink, lane, rkf, chawin, ck);
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
}

template <bool SEGMENTED, int CM>
__global__ void __launch_bounds__(32) shuffle_large_gen_kernel(int64_t num_arrays, DevPlan plan, uint64_t run_seed,
                                                               int64_t base, uint32_t *__restrict__ J,
                                                               uint32_t *__restrict__ words32, uint64_t *state_io,
                                                               uint64_t *words64, uint64_t *rk_first, int gen) {
    __shared__ DevSeg segs[MAX_SEGS];
    __shared__ __align__(16) uint64_t chawin[CM ? 256 : 2];
    const int lane = threadIdx.x & 31;
    for (uint32_t q = lane; q < plan.nseg; q += 32) segs[q] = plan.segs[q];
    __syncwarp();
    bool cha = CM == 1;
    if constexpr (CM == 2) cha = is_posgen(mk128(state_io[2], state_io[3]));
    if (CM != 0 && cha)
        shuffle_large_gen_body<SEGMENTED, CM != 0>(num_arrays, plan, run_seed, base, J, words32, state_io, words64,
                                                   rk_first, gen, segs, chawin);
    else if (CM != 1)
        shuffle_large_gen_body<SEGMENTED, false>(num_arrays, plan, run_seed, base, J, words32, state_io, words64,
                                                 rk_first, gen, segs, chawin);
}

// Same group resolution as apply_group, on global memory (no lane-id table: repeated
// targets are found with __match_any_sync).
template <typename T>
__device__ __forceinline__ void apply_group_global(T *z, const uint32_t *J, uint32_t top, uint32_t lim, int lane) {
    const int64_t i64 = (int64_t)top - lane;
    const bool act = i64 >= (int64_t)lim;
    const uint32_t i = act ? (uint32_t)i64 : 0;
    const uint32_t j = act ? __ldg(J + i) : (0xFFFFFFE0u | (uint32_t)lane);
    const T vi = act ? z[i] : T(0);
    const T vj = act ? z[j] : T(0);
    const uint32_t lo_pos = top >= lim + 31 ? top - 31 : lim;
    const uint32_t dm = top - j;
    const bool dv = act && dm < 32;
    unsigned pm = __ballot_sync(FULL, dv);
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const unsigned bq = __ballot_sync(FULL, dv && ((dm >> q) & 1));
        pm &= ((lane >> q) & 1) ? bq : ~bq;
    }
    const unsigned below = (1u << lane) - 1u;
    pm &= below;
    int p = pm ? 31 - __clz(pm) : lane;
#pragma unroll 1
    for (int it = 0; it < 5; ++it) {
        const int pp = __shfl_sync(FULL, p, p);
        if (!__any_sync(FULL, pp != p)) break;
        p = pp;
    }
    const T A = shfl_t(vi, p);
    const unsigned same = __match_any_sync(FULL, j);
    const unsigned tm = same & below;
    const T At = shfl_t(A, tm ? 31 - __clz(tm) : lane);
    const T B = tm ? At : vj;
    const unsigned later = same & ~((2u << lane) - 1u);
    if (act) {
        z[i] = B;
        if (later == 0 && j < lo_pos) z[j] = A;
    }
    __syncwarp();
}

template <typename T>
__global__ void __launch_bounds__(32) shuffle_large_apply_kernel(T *__restrict__ data, int64_t num_arrays,
                                                                 uint32_t n, uint32_t lim,
                                                                 const uint32_t *__restrict__ J) {
    const int lane = threadIdx.x & 31;
    for (int64_t a = blockIdx.x; a < num_arrays; a += gridDim.x) {
        T *z = data + a * (int64_t)n;
        const uint32_t *Ja = J + a * (int64_t)n;
        for (int64_t top = (int64_t)n - 1; top >= (int64_t)lim; top -= 32)
            apply_group_global<T>(z, Ja, (uint32_t)top, lim, lane);
    }
}

}  // namespace br

namespace br {
// digit_pass over many words (batched.py:69-82)
__global__ void digit_pass_kernel(const uint64_t *__restrict__ words, const uint32_t *__restrict__ bounds, int k,
                                  int64_t count, uint32_t *__restrict__ digits, uint64_t *__restrict__ rk) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t r = words[i];
        for (int m = 0; m < k; ++m) digits[i * k + m] = die(bounds[i * k + m], r);
        if (rk) rk[i] = r;
    }
}
}  // namespace br
