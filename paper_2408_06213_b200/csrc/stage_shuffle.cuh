// stage_shuffle.cuh -- many arrays too large for shared memory (C5: 256 x u64[2^20]):
// Fisher-Yates as a pipeline of shared-memory stages, one CTA per array, every random access
// in shared memory and every global access a stream.
//
// The array is cut into blocks of SP_B = 4096 positions.  Steps run from the top
// (shuffle.py:100-134: step s swaps z[s] and z[J[s]], J[s] <= s, s = n-1 down to 1), so every
// step of block sg happens after every step of the blocks above it.  Stage sg (NB-1 down to 0)
// holds block sg (its original values, mbox) in shared memory and
//   A. starts the TMA load of the block and prefetches its tile table;
//   B. generates the targets of its own steps (CTA-wide windows of striped batches with the
//      rejection realignment of shuffle.py:121-128: a rejected batch shifts every later batch
//      by one word, exact for any number of rejections);
//   C. resolves its own steps in closed form on indices only (DESIGN.md section 2.4 inside the
//      block: FT(x) = the first later in-block step targeting x, NS(s) = the next in-block step
//      after s with s's target, F = the end of the FT chain).  Afterwards every position
//      knows which shared-memory slot holds its value: Val(s) = mbox[F(s)] for a step leaving
//      the block, mbox[F(NS(s))] or mbox[J(s)] for an in-block output;
//   D. applies, in time order, the steps of higher blocks that target it ("records": target
//      offset x, step position s, deposited value).  The records of one target x form an
//      exchange chain: the earliest returns the block's value at x, each later one the value
//      deposited by the one before, and x keeps the last deposit.  A record's return value is
//      the final output of its step; it overwrites the record's value slot, which sits in the
//      SOURCE block's area (so the results of one source tile are contiguous);
//   E. writes its own records grouped by target block (one tile per lower block, through a
//      shared-memory staging area, coalesced), its in-block outputs after them, the tile table
//      entries and the slot map (position -> slot in the block's area).
// After stage 0 every slot holds a final value; shuffle_stage_gather_kernel writes
// out[p] = area[slot[p]] block by block through shared memory.  The payload itself is only
// read (block by block, stage A), so an array whose tiles would overflow a chunk (impossible
// for generated words in practice, but not excluded) is flagged and re-shuffled from its
// untouched payload by the CTA-group kernel.
//
// Record key: x | s << 12 (s < 2^20, so n <= 2^20 = 256 blocks); the source block is s >> 12.
// Exactness: stage sg sees its block exactly as the sequential loop does after all higher
// steps (their deposits in time order: tiles in source order, s inside a tile); its own
// steps are the sequential loop's (closed form, exhaustively checked in
// tests/test_resolution.py, bit-exactly against the oracle on the device in tests/test_stage.py).
#pragma once
#include "shuffle.cuh"
#include <type_traits>

namespace br {

#ifdef SP_CHECK
__device__ unsigned int g_sp_dbg[8];
__device__ int g_sp_stop = -1;  // debug: last stage to run (stages below it are skipped)
__device__ int g_sp_phase = 99;  // debug: phases to run in the last stage (1 = A-B, 2 = +C, 3 = +D)
// records the first failed check (line and three values); the guarded access is skipped
#define SP_OK(c, a0, a1, a2)                                                                   \
    ((c) ? true : (atomicCAS(&g_sp_dbg[0], 0u, (unsigned)__LINE__) == 0u                      \
                       ? (g_sp_dbg[1] = (unsigned)(a0), g_sp_dbg[2] = (unsigned)(a1),          \
                          g_sp_dbg[3] = (unsigned)(a2), g_sp_dbg[4] = blockIdx.x, false)       \
                       : false))
#else
#define SP_OK(c, a0, a1, a2) true
#endif
#define SP_ASSERT(c, ...)
#ifdef SP_PROF  // per-phase clock64 totals of CTA 0, printed at the end (profiling build)
#define SP_TICK(k)                        \
    if (L == 0) {                         \
        const long long t_ = clock64();   \
        sp_acc[k] += t_ - sp_t;           \
        sp_t = t_;                        \
    }
#else
#define SP_TICK(k)
#endif

static constexpr int SP_LOG_B = 12;
static constexpr uint32_t SP_B = 1u << SP_LOG_B;   // positions per block (one stage)
#ifndef SP_T_N
#define SP_T_N 512  // 1024 (one CTA per SM): 148 arrays 4.92 ms against 5.65, but 256 arrays take two waves, 9.63 ms against 7.55
#endif
static constexpr int SP_T = SP_T_N;                 // threads per CTA (512: two CTAs per SM)
static constexpr int SP_W = SP_T / 32;
static constexpr int SP_PER = SP_B / SP_T;          // positions per thread
static constexpr uint32_t SP_MAXNB = 256;           // blocks per array (n <= 2^20)
#ifndef SP_GJ_N
#define SP_GJ_N 1  // 512-batch windows: a rejection re-runs at most 512 (C5: 7.66 ms against 8.09 with 4; 4 slots with 512-batch windows where rejections are frequent: 8.23, register spills)
#endif
static constexpr int SP_GJ = SP_GJ_N;                     // generator slots per thread
static constexpr uint32_t SP_G = SP_GJ * SP_T;      // batches per generation window
static constexpr uint32_t SP_RING = SP_B + 8;       // targets by position - blo + 8 (8 below: the straddling batch)
static constexpr uint32_t SP_NONE = 0xFFFFFFFFu;
static constexpr uint16_t SP_NONE16 = 0xFFFF;
static constexpr uint32_t SP_JNONE = 0xFFFFFu;      // ring: no step at this position
static constexpr uint32_t SP_TGT = 0x80000000u;     // ring flag (C): the position is an in-block step's target

// inbox records per chunk: key, value and bucket entry per record in the 48 KB union
template <typename T>
__host__ __device__ constexpr uint32_t sp_cap() {
    return sizeof(T) == 8 ? 3072u : 4096u;
}

template <typename T>
struct SpShared {
    T mbox[SP_B];            // the block: original values, then after the higher blocks' deposits
    uint32_t ring[SP_RING];  // J by position (B, C), then src << 20 | J (E)
    uint32_t xcnt[SP_B / 2]; // D: records per target offset (two u16 per word), then bucket starts
    union {
        struct {
            uint32_t ft[SP_B];    // first later in-block step targeting x (atomicMin)
            uint32_t head[SP_B];  // per-target lists of in-block steps
            uint16_t link[SP_B];
            uint16_t F[SP_B];     // the end of the FT chain
        } loc;
        struct {
            uint32_t key[sp_cap<T>()];
            T val[sp_cap<T>()];
            uint32_t bkt[sp_cap<T>()];  // records bucketed by target offset: s << 12 | chunk index
        } rec;
        struct {
            uint32_t key[SP_B];
            T val[SP_B];
        } out;
    } u;
    u128 inc, AG, CG, M;  // generator constants of the array (the same for every thread)
    DevSeg segs[MAX_SEGS];
    uint64_t ub[MAX_SEGS];  // ff(start_n, k) of each segment (0: 2^64)
    uint32_t excl[SP_MAXNB + 1];  // inbox: exclusive prefix of the tile counts (tile t = source NB-1-t)
    uint32_t toff[SP_MAXNB];      // per source block: global record index minus inbox index
    uint32_t cnt[SP_MAXNB + 1];   // per target block: this stage's records, then their exclusive prefix
    uint32_t wsum[SP_W + 1];
    uint32_t carry[8];            // targets of the straddling batch for the next stage
    uint64_t bar;
    uint32_t fmin, nint, bad;
};

// exclusive scan of a[0..len) in place (len <= 2 * SP_T); every thread gets the total
__device__ __forceinline__ uint32_t sp_scan(uint32_t *a, uint32_t len, uint32_t *wsum, int L) {
    const uint32_t i0 = 2 * L, i1 = 2 * L + 1;
    const uint32_t v0 = i0 < len ? a[i0] : 0, v1 = i1 < len ? a[i1] : 0;
    const uint32_t loc = v0 + v1;
    uint32_t inc = loc;
    const int lane = L & 31, w = L >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint32_t x = lane < SP_W ? wsum[lane] : 0;
        uint32_t y = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, y, d);
            if (lane >= d) y += o;
        }
        if (lane < SP_W) wsum[lane] = y - x;  // exclusive warp offsets
        if (lane == SP_W - 1) wsum[SP_W] = y;  // grand total
    }
    __syncthreads();
    const uint32_t ex = wsum[w] + inc - loc;
    const uint32_t total = wsum[SP_W];
    if (i0 < len) a[i0] = ex;
    if (i1 < len) a[i1] = ex + v0;
    __syncthreads();
    return total;
}

// exclusive scan of a[0..len) in place by one warp (len <= 256); returns the total
__device__ __forceinline__ uint32_t sp_scan_w(uint32_t *a, uint32_t len, int lane) {
    uint32_t v[8], tot = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t i = (uint32_t)lane * 8 + q;
        v[q] = i < len ? a[i] : 0;
        tot += v[q];
    }
    uint32_t inc = tot;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= d) inc += o;
    }
    uint32_t ex = inc - tot;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t i = (uint32_t)lane * 8 + q;
        if (i < len) a[i] = ex;
        ex += v[q];
    }
    return __shfl_sync(0xFFFFFFFFu, inc, 31);
}

// exclusive scan, in place, of the SP_B u16 counters packed two per word in xc (8 per thread)
__device__ __forceinline__ void sp_scan_x(uint32_t *xc, uint32_t *wsum, int L) {
    constexpr int NWD = (int)(SP_B / SP_T / 2);  // words (two counters each) per thread
    static_assert(NWD == 4 || NWD == 2, "eight or four counters per thread");
    uint32_t wv[NWD];
    if constexpr (NWD == 4) {
        const uint4 w = reinterpret_cast<const uint4 *>(xc)[L];
        wv[0] = w.x, wv[1] = w.y, wv[2] = w.z, wv[3] = w.w;
    } else {
        const uint2 w = reinterpret_cast<const uint2 *>(xc)[L];
        wv[0] = w.x, wv[1] = w.y;
    }
    uint32_t tot = 0;
#pragma unroll
    for (int q = 0; q < NWD; ++q) tot += (wv[q] & 0xFFFFu) + (wv[q] >> 16);
    uint32_t inc = tot;
    const int lane = L & 31, wp = L >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) wsum[wp] = inc;
    __syncthreads();
    if (wp == 0) {
        const uint32_t x = lane < SP_W ? wsum[lane] : 0;
        uint32_t y = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, y, d);
            if (lane >= d) y += o;
        }
        if (lane < SP_W) wsum[lane] = y - x;
    }
    __syncthreads();
    uint32_t run = wsum[wp] + inc - tot;
    uint32_t ov[NWD];
#pragma unroll
    for (int q = 0; q < NWD; ++q) {
        const uint32_t lo = run;
        run += wv[q] & 0xFFFFu;
        ov[q] = lo | (run << 16);
        run += wv[q] >> 16;
    }
    if constexpr (NWD == 4) reinterpret_cast<uint4 *>(xc)[L] = make_uint4(ov[0], ov[1], ov[2], ov[3]);
    else reinterpret_cast<uint2 *>(xc)[L] = make_uint2(ov[0], ov[1]);
    __syncthreads();
}


__device__ __forceinline__ void sp_cp4(void *s, const void *g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void sp_cp8(void *s, const void *g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void sp_cp_wait() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// the end of the FT chain from e (C): FT values are later in-block steps, so the walk ends
__device__ __forceinline__ uint32_t sp_chase(const uint32_t *ft, uint32_t e) {
    for (uint32_t f = ft[e]; f != SP_NONE; f = ft[e]) e = f;
    return e;
}

// ---- target generation: striped slots.  Slot (thread L, j) owns the batches b == L + SP_T*j
// (mod SP_G) and holds the generator state whose output is word b + D of its next pending
// batch b.  A window [B0, wend) has at most one batch per slot; committed slots move SP_G
// batches on (one precomputed affine jump), the others keep their state.  A rejected batch f
// shifts every batch >= f by one word: pending slots step once more.
struct SpGen {
    u128 s[SP_GJ];
    uint32_t b[SP_GJ];  // pending batch of each slot
    uint32_t B0, D;
    uint8_t seg[SP_GJ];
};

__device__ __forceinline__ void sp_jump(u128 &s, u128 inc, uint32_t d, bool lh) {
    while (d > (uint32_t)JUMP_SMALL) {
        s = gen_jump_small(s, inc, JUMP_SMALL, lh);
        d -= JUMP_SMALL;
    }
    if (d) s = gen_jump_small(s, inc, (int)d, lh);
}

template <typename T>
__device__ __forceinline__ void sp_gen_init(SpGen &g, SpShared<T> &sh, uint64_t seed, bool lh, int L) {
    u128 s0, inc;
    gen_seed(seed, s0, inc, lh);
    if (L == 0) {
        sh.inc = inc;
        sh.M = gen_mult(lh);
        u128 A, C;
        gen_affine(SP_G, inc, lh, A, C);
        sh.AG = A;
        sh.CG = C;
    }
    const u128 s1 = gen_jump_small(s0, inc, L + 1, lh);  // output = word L
#pragma unroll
    for (int j = 0; j < SP_GJ; ++j) {
        u128 x = s1;
        sp_jump(x, inc, (uint32_t)(SP_T * j), lh);
        g.s[j] = x;
        g.b[j] = (uint32_t)L + (uint32_t)(SP_T * j);
        g.seg[j] = 0;
    }
    g.B0 = 0;
    g.D = 0;
}

// batch containing position p (plan.lo <= p < n)
__device__ __forceinline__ uint32_t sp_batch_of(const DevSeg *segs, uint32_t nseg, uint32_t p) {
    for (uint32_t q = 0; q < nseg; ++q) {
        const DevSeg S = segs[q];
        if (p >= S.start_n - S.count * S.k) return S.first_batch + (S.start_n - 1 - p) / S.k;
    }
    return 0;
}

// generate every batch up to and including b_need; targets into ring[pos - blo + 8]
template <typename T>
__device__ __forceinline__ void sp_gen_block(SpGen &g, const DevPlan &plan, SpShared<T> &sh, int L, uint32_t b_need,
                                             uint32_t blo, bool lh) {
    while (g.B0 <= b_need) {
        const uint32_t wend = min(g.B0 + SP_G, b_need + 1);  // window [B0, wend)
        uint32_t myfail = SP_NONE;
#pragma unroll
        for (int j = 0; j < SP_GJ; ++j) {
            const uint32_t b = g.b[j];
            if (b < wend) {
                uint32_t q = g.seg[j];
                while (q + 1 < plan.nseg && sh.segs[q + 1].first_batch <= b) ++q;
                g.seg[j] = (uint8_t)q;
                const DevSeg S = sh.segs[q];
                const uint32_t nbb = S.start_n - (b - S.first_batch) * S.k;
                uint64_t r = gen_out(g.s[j], lh);
                uint32_t *rg = sh.ring + (nbb - 1 - blo + 8);
                if (plan.naive && S.k == 2) {
                    uint32_t j1, j2;
                    naive_pair(nbb, r, j1, j2);
                    rg[0] = j1;
                    rg[-1] = j2;
                } else {
                    auto dice = [&](auto K) {
#pragma unroll
                        for (int m = 0; m < decltype(K)::value; ++m) rg[-m] = die(nbb - m, r);
                    };
                    switch (S.k) {
                        case 1: dice(std::integral_constant<int, 1>{}); break;
                        case 2: dice(std::integral_constant<int, 2>{}); break;
                        case 3: dice(std::integral_constant<int, 3>{}); break;
                        case 4: dice(std::integral_constant<int, 4>{}); break;
                        case 5: dice(std::integral_constant<int, 5>{}); break;
                        case 6: dice(std::integral_constant<int, 6>{}); break;
                        case 7: dice(std::integral_constant<int, 7>{}); break;
                        default: dice(std::integral_constant<int, 8>{}); break;
                    }
                }
                // the exact threshold (2^64 mod ff(n_b, k) < ff(n_b, k) <= the segment's first
                // product) is read only below that bound: the reference's carried bound u
                const uint64_t ub = sh.ub[q];
                if ((ub == 0 || r < ub) && r < __ldg(plan.thresh + b) && b < myfail) myfail = b;
            }
        }
        if (!__syncthreads_or(myfail != SP_NONE)) {
            const u128 AG = sh.AG, CG = sh.CG;
#pragma unroll
            for (int j = 0; j < SP_GJ; ++j)
                if (g.b[j] < wend) {
                    g.b[j] += SP_G;
                    g.s[j] = mad128_wide(g.s[j], AG, CG);
                }
            g.B0 = wend;
        } else {
            if (L == 0) sh.fmin = SP_NONE;
            __syncthreads();
            if (myfail != SP_NONE) atomicMin(&sh.fmin, myfail);
            __syncthreads();
            const uint32_t f = sh.fmin;  // the first rejected batch: it and everything after take one word more
            const u128 AG = sh.AG, CG = sh.CG, M = sh.M, inc = sh.inc;
#pragma unroll
            for (int j = 0; j < SP_GJ; ++j) {
                if (g.b[j] < f) {
                    g.b[j] += SP_G;
                    g.s[j] = mad128_wide(g.s[j], AG, CG);
                }
                g.s[j] = mad128_wide(g.s[j], M, inc);
            }
            g.B0 = f;
            g.D += 1;
            __syncthreads();
        }
    }
}


// scratch: per CTA the records' keys and the tile table (reused array after array); per
// array the value areas, the slot map and a flag
__host__ __device__ constexpr size_t sp_cta_bytes(uint32_t n) {
    const size_t nb = (n + SP_B - 1) / SP_B;
    return (((size_t)n * 4 + 255) & ~(size_t)255) + ((nb * nb * 4 + 255) & ~(size_t)255);
}

template <typename T>
__device__ __forceinline__ void shuffle_stage_body(const T *__restrict__ data, int64_t num_arrays, const DevPlan &plan,
                                                   uint64_t run_seed, int64_t base, uint32_t *__restrict__ words32,
                                                   int gen, SpShared<T> &sh, unsigned char *__restrict__ cta_scratch,
                                                   size_t cta_bytes, T *__restrict__ val_all,
                                                   uint16_t *__restrict__ slot_all, uint32_t vstride,
                                                   uint32_t *__restrict__ flags, int use_tma) {
    const int L = threadIdx.x;
    const int lane = L & 31, wid = L >> 5;
    const uint32_t n = plan.n;
    const uint32_t NB = (n + SP_B - 1) / SP_B;
    const uint32_t lo = plan.lo;
    const bool lh = gen == 1;
    uint32_t *keyg = reinterpret_cast<uint32_t *>(cta_scratch + (size_t)blockIdx.x * cta_bytes);
    uint32_t *desc = keyg + (((size_t)n * 4 + 255) & ~(size_t)255) / 4;
    uint16_t *src16 = reinterpret_cast<uint16_t *>(sh.xcnt);  // C -> E (D is done): each position's source slot

    for (uint32_t q = L; q < plan.nseg; q += SP_T) {
        const DevSeg S = plan.segs[q];
        sh.segs[q] = S;
        unsigned __int128 f = 1;
        for (uint32_t m = 0; m < S.k; ++m) f *= (uint64_t)(S.start_n - m);
        sh.ub[q] = f >> 64 ? 0ull : (uint64_t)f;  // (plans hold products <= 2^64)
    }
    for (uint32_t x = L; x < SP_B / 2; x += SP_T) sh.xcnt[x] = 0;
    for (uint32_t x = L; x <= SP_MAXNB; x += SP_T) sh.cnt[x] = 0;
    if (L == 0) {
        sh.nint = 0;
        sh.bad = 0;
        mbar_init(&sh.bar, 1);
    }
    __syncthreads();
    uint32_t parity = 0;
#ifdef SP_PROF
    long long sp_acc[10] = {0}, sp_t = clock64();
#endif
    for (int64_t a = blockIdx.x; a < num_arrays; a += gridDim.x) {
        const T *z = data + a * (int64_t)n;
        T *valg = val_all + a * (int64_t)vstride;
        uint16_t *slotg = slot_all + a * (int64_t)vstride;
        SpGen g;
        sp_gen_init<T>(g, sh, array_seed(run_seed, (uint64_t)(base + a)), lh, L);
        __syncthreads();
        uint32_t dreg = 0;  // this stage's tile-table row entry (tile L), loaded at the end of the stage above
        for (int sg = (int)NB - 1; sg >= 0; --sg) {
            const uint32_t blo = (uint32_t)sg * SP_B;
            const uint32_t bn = min(SP_B, n - blo);
            const uint32_t slo = max(blo, lo);  // positions below slo have no step
            const uint32_t ntile = NB - 1 - (uint32_t)sg;
            // ---- A. the block streams in; tile table entries of this block (all written by now)
            if (use_tma) {
                if (L == 0) {
                    fence_proxy_async();  // earlier generic accesses to mbox come first
                    mbar_arrive_expect_tx(&sh.bar, bn * (uint32_t)sizeof(T));
                    bulk_load(sh.mbox, z + blo, bn * (uint32_t)sizeof(T), &sh.bar);
                }
            } else {
                for (uint32_t x = L; x < bn; x += SP_T) sh.mbox[x] = z[blo + x];
            }
            if (L < 8) sh.ring[SP_B + L] = sh.carry[L];
            if (blo + (uint32_t)L < slo) sh.ring[L + 8] = SP_JNONE;  // no step (block 0 below plan.lo)
            // ---- D setup: the inbox tiles' prefix and chunks (warp 0), then chunk 0's records
            // are requested before the generation step so that they land behind it
            if ((uint32_t)L < ntile) {
                sh.excl[L] = dreg & 0xFFFFu;
                sh.toff[NB - 1 - (uint32_t)L] = dreg >> 16;
            }
            __syncthreads();
            if (wid == 0) {
                const uint32_t R = sp_scan_w(sh.excl, ntile, lane);
                for (uint32_t t = lane; t < ntile; t += 32) {  // global record index minus inbox index
                    const uint32_t src = NB - 1 - t;
                    sh.toff[src] = src * SP_B + sh.toff[src] - sh.excl[t];
                }
                if (lane == 0) sh.excl[ntile] = R;
            }
            __syncthreads();
            // chunks: the longest run of whole tiles from ta within sp_cap records (a tile larger
            // than a chunk marks the array for the fallback kernel)
            auto chunk_end = [&](uint32_t ta) {
                const uint32_t lim = sh.excl[ta] + sp_cap<T>();
                uint32_t l = ta, h = ntile;
                while (l < h) {
                    const uint32_t m = (l + h + 1) >> 1;
                    if (sh.excl[m] <= lim) l = m;
                    else h = m - 1;
                }
                return l;
            };
            auto issue_chunk = [&](uint32_t ta, uint32_t tb) {
                const uint32_t cbase = sh.excl[ta];
                for (uint32_t t = ta + (uint32_t)wid; t < tb; t += SP_W) {
                    const uint32_t src = NB - 1 - t;
                    const uint32_t c0 = sh.excl[t], cn = sh.excl[t + 1] - c0;
                    const uint32_t g0 = sh.toff[src] + c0;
                    for (uint32_t q = lane; q < cn; q += 32) {
                        sp_cp4(&sh.u.rec.key[c0 - cbase + q], keyg + g0 + q);
                        if (sizeof(T) == 8) sp_cp8(&sh.u.rec.val[c0 - cbase + q], valg + g0 + q);
                        else sp_cp4(&sh.u.rec.val[c0 - cbase + q], valg + g0 + q);
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            const uint32_t tb0 = ntile ? chunk_end(0) : 0;
            if (tb0) issue_chunk(0, tb0);
            // ---- B. targets of this block's steps
            if (slo < blo + bn) sp_gen_block<T>(g, plan, sh, L, sp_batch_of(sh.segs, plan.nseg, slo), blo, lh);
            __syncthreads();
            SP_TICK(0)
            if (L < 8) sh.carry[L] = sh.ring[L];
            if (use_tma) {
                mbar_wait(&sh.bar, parity);
                parity ^= 1u;
            }
            SP_TICK(1)
            uint32_t ta = 0;
            for (uint32_t ch = 0; ta < ntile; ++ch) {
                const uint32_t tb = ch == 0 ? tb0 : chunk_end(ta);
                if (tb == ta) {  // one tile alone exceeds a chunk
                    if (L == 0) sh.bad = 1;
                    break;
                }
                const uint32_t cbase = sh.excl[ta];
                const uint32_t ccount = sh.excl[tb] - cbase;
                if (ch > 0) issue_chunk(ta, tb);
                asm volatile("cp.async.wait_group 0;" ::: "memory");
                __syncthreads();
                SP_TICK(2)
                // records bucketed by target offset x (counting sort), then each record finds its
                // predecessor at x (the least later-in-order step s' > s) by scanning its bucket
                constexpr uint32_t RPT = (sp_cap<T>() + SP_T - 1) / SP_T;
                uint32_t arr[(RPT + 1) / 2];  // arrival index of each record within its bucket
#pragma unroll
                for (uint32_t j = 0; j < RPT; ++j) {
                    if (j * SP_T >= ccount) break;  // (uniform: the chunk's records end)
                    const uint32_t r = (uint32_t)L + j * SP_T;
                    uint32_t av = 0;
                    if (r < ccount) {
                        const uint32_t x = sh.u.rec.key[r] & (SP_B - 1), hs = (x & 1) * 16;
                        av = (atomicAdd(&sh.xcnt[x >> 1], 1u << hs) >> hs) & 0xFFFFu;
                    }
                    if (j & 1) arr[j / 2] |= av << 16;
                    else arr[j / 2] = av;
                }
                __syncthreads();
                sp_scan_x(sh.xcnt, sh.wsum, L);
                SP_TICK(3)
#pragma unroll
                for (uint32_t j = 0; j < RPT; ++j) {
                    if (j * SP_T >= ccount) break;  // (uniform: the chunk's records end)
                    const uint32_t r = (uint32_t)L + j * SP_T;
                    if (r < ccount) {
                        const uint32_t K = sh.u.rec.key[r];
                        const uint32_t x = K & (SP_B - 1);
                        const uint32_t st = (sh.xcnt[x >> 1] >> ((x & 1) * 16)) & 0xFFFFu;
                        sh.u.rec.bkt[st + ((arr[j / 2] >> (16 * (j & 1))) & 0xFFFFu)] = (K & ~(SP_B - 1)) | r;
                    }
                }
                __syncthreads();
                SP_TICK(4)
                uint32_t lastm = 0;
#pragma unroll
                for (uint32_t j = 0; j < RPT; ++j) {
                    if (j * SP_T >= ccount) break;  // (uniform: the chunk's records end)
                    const uint32_t r = (uint32_t)L + j * SP_T;
                    if (r < ccount) {
                        const uint32_t K = sh.u.rec.key[r];
                        const uint32_t s = K >> SP_LOG_B, x = K & (SP_B - 1);
                        const uint32_t sw = sh.xcnt[x >> 1];
                        const uint32_t st = (sw >> ((x & 1) * 16)) & 0xFFFFu;
                        const uint32_t en = (x & 1) ? (x == SP_B - 1 ? ccount : sh.xcnt[(x >> 1) + 1] & 0xFFFFu) : sw >> 16;
                        const uint32_t hiK = K | (SP_B - 1), loK = K & ~(SP_B - 1);
                        uint32_t best = SP_NONE;
                        bool last = true;
                        for (uint32_t q = st; q < en; ++q) {
                            const uint32_t e = sh.u.rec.bkt[q];
                            if (e > hiK && e < best) best = e;
                            last &= !(e < loK);
                        }
                        const T res = best != SP_NONE ? sh.u.rec.val[best & (SP_B - 1)] : sh.mbox[x];
                        const uint32_t gi = sh.toff[s >> SP_LOG_B] + cbase + r;  // (u32: toff may wrap)
                        if (SP_OK(s < n && (s >> SP_LOG_B) > (uint32_t)sg && gi < n, sg, r, K)) __stcg(valg + gi, res);
                        if (last) lastm |= 1u << j;
                    }
                }
                __syncthreads();
#pragma unroll
                for (uint32_t j = 0; j < RPT; ++j) {
                    if (j * SP_T >= ccount) break;  // (uniform: the chunk's records end)
                    const uint32_t r = (uint32_t)L + j * SP_T;
                    if ((lastm >> j) & 1) sh.mbox[sh.u.rec.key[r] & (SP_B - 1)] = sh.u.rec.val[r];
                }
                if ((uint32_t)L < SP_B / 8) reinterpret_cast<uint4 *>(sh.xcnt)[L] = make_uint4(0, 0, 0, 0);
                __syncthreads();
                SP_TICK(5)
                ta = tb;
            }
            // ---- C. this block's own steps in closed form (indices only).  Steps with an
            // in-block target are rare above block 0 (about 2048/sg of the block's 4096), so only
            // the entries they touch are initialised: FT minima and lists at their targets and at
            // themselves, and a flag on every targeted position (ring bit 31).  A position that no
            // in-block step targets, and that has none itself, is its own source.
            // (the same pass ranks E's outputs: records by target block, in-block outputs in order)
            uint32_t nin = 0;
            uint32_t rk[SP_PER / 2];
#pragma unroll
            for (int q = 0; q < SP_PER; ++q) {
                const uint32_t i = (uint32_t)L + (uint32_t)q * SP_T;
                uint32_t rank = 0;
                bool inb = true;
                if (i < bn) {
                    const uint32_t J = sh.ring[i + 8] & ~SP_TGT;
                    if (J < blo) {
                        rank = atomicAdd(&sh.cnt[J >> SP_LOG_B], 1u);
                        inb = false;
                    } else if (J != SP_JNONE) {
                        const uint32_t y = J - blo;
                        sh.u.loc.ft[y] = SP_NONE;
                        sh.u.loc.head[y] = SP_NONE;
                        sh.u.loc.ft[i] = SP_NONE;
                        atomicOr(&sh.ring[y + 8], SP_TGT);
                        ++nin;
                    }
                }
                const unsigned m = __ballot_sync(0xFFFFFFFFu, i < bn && inb);
                uint32_t b0 = 0;
                if (lane == 0 && m) b0 = atomicAdd(&sh.nint, (uint32_t)__popc(m));
                b0 = __shfl_sync(0xFFFFFFFFu, b0, 0);
                if (i < bn && inb) rank = b0 + __popc(m & ((1u << lane) - 1));
                if (q & 1) rk[q / 2] |= rank << 16;
                else rk[q / 2] = rank;
            }
            SP_TICK(6)
            const bool inblk = __syncthreads_or(nin) != 0;
            if (inblk) {
#pragma unroll
                for (int q = 0; q < SP_PER; ++q) {
                    const uint32_t i = (uint32_t)L + (uint32_t)q * SP_T;
                    if (i < bn) {
                        const uint32_t J = sh.ring[i + 8] & ~SP_TGT;
                        if (J >= blo && J != SP_JNONE) {
                            const uint32_t y = J - blo;
                            if (i > y) atomicMin(&sh.u.loc.ft[y], i);
                            sh.u.loc.link[i] = (uint16_t)atomicExch(&sh.u.loc.head[y], i);
                        }
                    }
                }
                __syncthreads();
#pragma unroll
                for (int q = 0; q < SP_PER; ++q) {
                    const uint32_t i = (uint32_t)L + (uint32_t)q * SP_T;
                    if (i < bn) {
                        const uint32_t w = sh.ring[i + 8];
                        const uint32_t J = w & ~SP_TGT;
                        uint32_t src = i;
                        if (J >= blo && J != SP_JNONE) {  // in-block output: the next step with i's target
                            uint32_t ns = SP_NONE;
                            for (uint32_t m = sh.u.loc.head[J - blo]; m != SP_NONE && m != SP_NONE16; m = sh.u.loc.link[m])
                                if (m > i && m < ns) ns = m;
                            if (ns != SP_NONE) src = sp_chase(sh.u.loc.ft, ns);
                            else src = J - blo;
                        } else if (w & SP_TGT) {  // the value leaving position i (or its final value)
                            src = sp_chase(sh.u.loc.ft, i);
                        }
                        src16[i] = (uint16_t)src;
                    }
                }
            }
            __syncthreads();
            SP_TICK(7)
            // ---- E. this block's records (by target block), in-block outputs, slot map
            if (wid == 0) {
                const uint32_t tot = sp_scan_w(sh.cnt, (uint32_t)sg, lane);
                if (lane == 0) sh.cnt[sg] = tot;
            }
            __syncthreads();
            const uint32_t nrec = sh.cnt[sg];
#pragma unroll
            for (int q = 0; q < SP_PER; ++q) {
                const uint32_t i = (uint32_t)L + (uint32_t)q * SP_T;
                if (i < bn) {
                    const uint32_t J = sh.ring[i + 8] & ~SP_TGT;
                    const uint32_t src = inblk ? src16[i] : i;
                    const uint32_t rank = (rk[q / 2] >> (16 * (q & 1))) & 0xFFFFu;
                    uint32_t slot;
                    if (J < blo) {
                        slot = sh.cnt[J >> SP_LOG_B] + rank;
                        sh.u.out.key[slot] = (J & (SP_B - 1)) | ((blo + i) << SP_LOG_B);
                    } else {
                        slot = nrec + rank;
                    }
                    sh.u.out.val[slot] = sh.mbox[src];
                    slotg[blo + i] = (uint16_t)slot;
                }
            }
            for (uint32_t tb = L; tb < (uint32_t)sg; tb += SP_T)
                __stcg(desc + (size_t)tb * NB + sg, (sh.cnt[tb] << 16) | (sh.cnt[tb + 1] - sh.cnt[tb]));
            __syncthreads();
            // staged area out, 16-byte stores
            {
                const uint32_t vb = bn * (uint32_t)sizeof(T);
                const uint32_t v16 = vb / 16;
                const uint4 *sv = reinterpret_cast<const uint4 *>(sh.u.out.val);
                uint4 *gv = reinterpret_cast<uint4 *>(valg + blo);
                for (uint32_t q = L; q < v16; q += SP_T) __stcg(gv + q, sv[q]);
                for (uint32_t x = v16 * 16 / (uint32_t)sizeof(T) + L; x < bn; x += SP_T) valg[blo + x] = sh.u.out.val[x];
                const uint32_t k16 = (nrec + 3) / 4;
                const uint4 *sk = reinterpret_cast<const uint4 *>(sh.u.out.key);
                uint4 *gk = reinterpret_cast<uint4 *>(keyg + blo);
                for (uint32_t q = L; q < k16; q += SP_T) __stcg(gk + q, sk[q]);
            }
            for (uint32_t tb = L; tb <= (uint32_t)sg; tb += SP_T) sh.cnt[tb] = 0;
            if (L == 0) sh.nint = 0;
            if ((uint32_t)L < SP_B / 8) reinterpret_cast<uint4 *>(sh.xcnt)[L] = make_uint4(0, 0, 0, 0);  // src16 -> the next stage's counters
            __syncthreads();
            // the next stage's tile-table row: complete now (this stage wrote the last entry)
            dreg = sg > 0 && (uint32_t)L < ntile + 1 ? __ldcg(desc + (size_t)(sg - 1) * NB + (NB - 1 - L)) : 0;
            SP_TICK(8)
        }
#ifdef SP_PROF
        if (L == 0 && blockIdx.x == 0)
            printf("SP_PROF cycles: gen %lld dsetup %lld load %lld count %lld scatter %lld resolve %lld C0 %lld C %lld E %lld\n",
                   sp_acc[0], sp_acc[1], sp_acc[2], sp_acc[3], sp_acc[4], sp_acc[5], sp_acc[6], sp_acc[7], sp_acc[8]);
#endif
        if (L == 0) {
            if (words32) words32[a] = plan.nbatches + g.D;
            if (sh.bad) flags[a] = 1;
            sh.bad = 0;
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void __launch_bounds__(SP_T, 1024 / SP_T) shuffle_stage_kernel(const T *__restrict__ data, int64_t num_arrays,
                                                                 DevPlan plan, uint64_t run_seed, int64_t base,
                                                                 uint32_t *__restrict__ words32, int gen,
                                                                 unsigned char *__restrict__ cta_scratch,
                                                                 size_t cta_bytes, T *__restrict__ val_all,
                                                                 uint16_t *__restrict__ slot_all, uint32_t vstride,
                                                                 uint32_t *__restrict__ flags, int use_tma) {
    extern __shared__ __align__(16) unsigned char sp_smem[];
    auto &sh = *reinterpret_cast<SpShared<T> *>(sp_smem);
    shuffle_stage_body<T>(data, num_arrays, plan, run_seed, base, words32, gen, sh, cta_scratch, cta_bytes, val_all,
                          slot_all, vstride, flags, use_tma);
}

// out[p] = area[slot[p]] for every block of every unflagged array, one block per iteration
// through shared memory (the slot map is a permutation of the block's slots)
static constexpr int SPG_T = 512;
template <typename T>
__global__ void __launch_bounds__(SPG_T) shuffle_stage_gather_kernel(T *__restrict__ data, int64_t num_arrays,
                                                                     uint32_t n, const T *__restrict__ val_all,
                                                                     const uint16_t *__restrict__ slot_all,
                                                                     uint32_t vstride,
                                                                     const uint32_t *__restrict__ flags) {
    __shared__ T buf[SP_B];
    const uint32_t NB = (n + SP_B - 1) / SP_B;
    const int64_t total = num_arrays * (int64_t)NB;
    for (int64_t g = blockIdx.x; g < total; g += gridDim.x) {
        const int64_t a = g / NB;
        if (flags[a]) continue;
        const uint32_t blo = (uint32_t)(g - a * NB) * SP_B;
        const uint32_t bn = min(SP_B, n - blo);
        const int64_t off = a * (int64_t)n + blo;
        const int64_t voff = a * (int64_t)vstride + blo;
        constexpr int PER = SP_B / SPG_T;
        T v[PER];
        uint16_t sl[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t x = threadIdx.x + k * SPG_T;
            if (x < bn) {
                v[k] = __ldcs(val_all + voff + x);
                sl[k] = __ldcs(slot_all + voff + x);
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t x = threadIdx.x + k * SPG_T;
            if (x < bn) buf[x] = v[k];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t x = threadIdx.x + k * SPG_T;
            if (x < bn) __stcs(data + off + x, buf[sl[k]]);
        }
        __syncthreads();
    }
}

}  // namespace br
