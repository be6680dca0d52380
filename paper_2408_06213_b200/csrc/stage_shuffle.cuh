// stage_shuffle.cuh -- many arrays too large for shared memory (C5: 256 x u64[2^20]):
// Fisher-Yates as a pipeline of shared-memory stages, one CTA per array, no random access
// to global memory.
//
// The array is cut into blocks of SP_B positions.  Steps run from the top (shuffle.py:100-134:
// step s swaps z[s] and z[J[s]], J[s] <= s, s = n-1 down to 1), so block sg's steps happen after
// every step of the blocks above it.  Stage sg (sg = NB-1 down to 0) holds block sg in shared
// memory and
//   1. applies, in time order, the steps of higher blocks that target it ("records" left by
//      those stages: target offset, the step's position, the value it deposits).  For a target
//      q the steps arrive as an exchange sequence: the first returns z0[q], each later one the
//      value of the one before, and q keeps the last deposit.  The returned value is the step's
//      final output (out[s] = the value at J[s] just before step s); it goes to the result slot
//      of the record, which sits in the SOURCE block's result area;
//   2. generates the targets of its own steps (CTA-wide, with the rejection realignment of
//      large_gen_step: word alignment is exact for any number of rejections);
//   3. runs its own steps in closed form (DESIGN.md section 2.4 restricted to the block):
//      with FT(x) the first later step targeting x inside the block and NS(s) the next such
//      step after s with s's target, the value at x before step x is Val(x) = Val(FT(x)) or the
//      block contents after (1); an in-block step outputs Val(NS(s)) or the contents of its
//      target; a step targeting a lower block leaves a record (target, s, Val(s)) for the stage
//      of that block;
//   4. writes its records grouped by target block (tiles), a tile table entry per lower block,
//      its in-block outputs into its result area and a slot map (position -> result slot).
// After stage 0 every result slot is filled; out[p] = result[slot[p]] is gathered block by
// block through shared memory by a second, fully parallel kernel (shuffle_stage_gather_kernel).
// Global traffic is streaming (blocks, records, results, slot maps); all random accesses are
// in shared memory.  The next block streams in (TMA bulk copy) while the current one is
// worked on.
//
// Exactness: stage sg sees the block exactly as the sequential loop would after all higher
// steps (their deposits in time order, records carry s); its own steps are the sequential
// loop's (closed form, checked exhaustively in tests/test_resolution.py and bit-exactly
// against the oracle on the device).
#pragma once
#include "shuffle.cuh"

namespace br {

#ifndef SP_LOG_B
#define SP_LOG_B 11
#endif
static constexpr uint32_t SP_B = 1u << SP_LOG_B;  // positions per block (one stage)
static constexpr int SP_W = SP_B / 256;           // warps per CTA (8 positions per thread)
static constexpr int SP_T = 32 * SP_W;            // threads per CTA
static constexpr uint32_t SP_C = SP_B;            // records per chunk of step 1 (a whole tile always fits)
static constexpr uint32_t SP_RING = 2 * SP_B;     // u32 target ring: a block + the straddling batch
static constexpr uint32_t SP_MAXNB = 2 * SP_T;    // blocks per array (the tile scans cover 2 per thread)
static constexpr uint32_t SP_NONE = 0xFFFFFFFFu;
static constexpr uint16_t SP_NONE16 = 0xFFFF;

template <typename T>
struct SpShared {
    static constexpr uint32_t RSIZE = SP_RING;
    using RType = uint32_t;
    DevSeg segs[MAX_SEGS];
    uint32_t ring[SP_RING];  // targets by position (large_gen_step)
    T mbuf[2][SP_B];         // the block's contents; the next block streams into the other buffer
    uint32_t head[SP_B];     // per-target chain heads (atomicExch), SP_NONE = empty
    union {
        struct {  // step 1: one chunk of records
            uint32_t key[SP_C];  // the record's step position s (larger = earlier in time)
            T val[SP_C];
            uint16_t link[SP_C];
            uint16_t q[SP_C];
        } rec;
        struct {  // step 3: the block's own steps
            uint16_t F[SP_B];  // FT pointer, then the end of the FT chain (Val(x) = mbox[F[x]])
            uint16_t link[SP_B];
        } loc;
    } u;
    uint32_t vstart[SP_MAXNB];  // tiles: exclusive prefix of counts; step 4: per-target-block prefix
    uint32_t tbase[SP_MAXNB];   // tiles: first record index; step 4: per-target-block counts
    uint32_t nd[SP_MAXNB];      // the next stage's tile table (prefetched during this stage)
    uint32_t wsum[SP_W + 1];
    uint64_t bar[2];
    uint32_t frontier[2];
    uint32_t fmin;
    uint32_t nint;
    uint32_t chunk_end;
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

// global scratch: per CTA (records and tile table, reused array after array) and per array
// (result slots and slot map, read by the gather kernel)
template <typename T>
__host__ __device__ constexpr size_t sp_cta_bytes(uint32_t n) {
    const size_t nb = (n + SP_B - 1) / SP_B;
    return (((size_t)n * 4 + 255) & ~(size_t)255) +           // record (target offset | position << 16)
           (((size_t)n * sizeof(T) + 255) & ~(size_t)255) +   // record value
           ((nb * nb * 4 + 255) & ~(size_t)255);              // tile table
}
template <typename T>
__host__ __device__ constexpr size_t sp_array_bytes(uint32_t n) {
    return (size_t)n * (sizeof(T) + 2);  // result slots + slot map
}

// ---- target generation for one block: striped lanes, no per-stage jump
// Slot (thread L, j) owns the batches b == L + SP_T*j (mod SP_G) and holds the generator state
// whose output is word b + D of its next pending batch b.  A step covers the window
// [B0, B0 + nact) (nact <= SP_G, so a slot has at most one batch in it); committed slots move
// SP_G batches on (one precomputed affine jump), the others keep their state.  A rejected batch
// f shifts every batch >= f by one word (shuffle.py:121-128): pending slots step once more.
static constexpr int SP_GJ = 5;                 // slots per thread (k = 2: a block's batches in one step)
static constexpr uint32_t SP_G = SP_GJ * SP_T;  // batches per step

struct SpGen {
    u128 s[SP_GJ];
    uint32_t b[SP_GJ];   // pending batch of each slot
    uint8_t seg[SP_GJ];  // its segment
    u128 inc, AG, CG, M;
    uint32_t B0, D;
    bool lh;
};

__device__ __forceinline__ void sp_jump(u128 &s, u128 inc, uint32_t d, bool lh) {
    while (d > (uint32_t)JUMP_SMALL) {
        s = gen_jump_small(s, inc, JUMP_SMALL, lh);
        d -= JUMP_SMALL;
    }
    if (d) s = gen_jump_small(s, inc, (int)d, lh);
}

template <typename T>
__device__ __forceinline__ void sp_gen_init(SpGen &g, uint64_t seed, bool lh, int L) {
    u128 s0, inc;
    gen_seed(seed, s0, inc, lh);
    g.inc = inc;
    g.lh = lh;
    g.M = gen_mult(lh);
    gen_affine(SP_G, inc, lh, g.AG, g.CG);
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

// generate every batch up to and including b_need into the target ring
template <typename T>
__device__ __forceinline__ void sp_gen_block(SpGen &g, const DevPlan &plan, SpShared<T> &sh, int L, uint32_t b_need) {
    constexpr uint32_t RS = SP_RING;
    while (g.B0 <= b_need) {
        const uint32_t wend = min(g.B0 + SP_G, b_need + 1);  // window [B0, wend)
        uint64_t t[SP_GJ];
#pragma unroll
        for (int j = 0; j < SP_GJ; ++j)
            if (g.b[j] < wend) t[j] = __ldg(plan.thresh + g.b[j]);
        uint32_t myfail = 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < SP_GJ; ++j) {
            const uint32_t b = g.b[j];
            if (b < wend) {
                uint32_t q = g.seg[j];
                while (q + 1 < plan.nseg && sh.segs[q + 1].first_batch <= b) ++q;
                g.seg[j] = (uint8_t)q;
                const DevSeg S = sh.segs[q];
                const uint32_t nbb = S.start_n - (b - S.first_batch) * S.k;
                uint64_t r = gen_out(g.s[j], g.lh);
                const uint32_t pos = nbb - 1;
                if (plan.naive && S.k == 2) {
                    uint32_t j1, j2;
                    naive_pair(nbb, r, j1, j2);
                    sh.ring[pos & (RS - 1)] = j1;
                    sh.ring[(pos - 1) & (RS - 1)] = j2;
                } else {
                    for (uint32_t m = 0; m < S.k; ++m) sh.ring[(pos - m) & (RS - 1)] = die(nbb - m, r);
                }
                if (r < t[j] && b < myfail) myfail = b;
            }
        }
        if (!__syncthreads_or(myfail != 0xFFFFFFFFu)) {
#pragma unroll
            for (int j = 0; j < SP_GJ; ++j)
                if (g.b[j] < wend) {
                    g.b[j] += SP_G;
                    g.s[j] = mad128(g.s[j], g.AG, g.CG);
                }
            g.B0 = wend;
        } else {
            if (L == 0) sh.fmin = 0xFFFFFFFFu;
            __syncthreads();
            if (myfail != 0xFFFFFFFFu) atomicMin(&sh.fmin, myfail);
            __syncthreads();
            const uint32_t f = sh.fmin;  // the first rejected batch: it and everything after take one word more
#pragma unroll
            for (int j = 0; j < SP_GJ; ++j) {
                if (g.b[j] < f) {
                    g.b[j] += SP_G;
                    g.s[j] = mad128(g.s[j], g.AG, g.CG);
                }
                g.s[j] = mad128(g.s[j], g.M, g.inc);
            }
            g.B0 = f;
            g.D += 1;
            __syncthreads();
        }
    }
}

template <typename T>
__device__ __forceinline__ void shuffle_stage_body(T *__restrict__ data, int64_t num_arrays, const DevPlan &plan,
                                                   uint64_t run_seed, int64_t base, uint32_t *__restrict__ words32,
                                                   int gen, SpShared<T> &sh, unsigned char *__restrict__ cta_scratch,
                                                   size_t cta_bytes, T *__restrict__ res_all,
                                                   uint16_t *__restrict__ slot_all, int use_tma) {
    constexpr int PER = SP_B / SP_T;   // positions per thread in steps 3-4
    constexpr int RPER = SP_C / SP_T;  // records per thread in step 1
    const int L = threadIdx.x;
    const uint32_t n = plan.n;
    const uint32_t NB = (n + SP_B - 1) / SP_B;
    const uint32_t lo = plan.lo;
    unsigned char *w = cta_scratch + (size_t)blockIdx.x * cta_bytes;
    uint32_t *fwdq = reinterpret_cast<uint32_t *>(w);
    w += ((size_t)n * 4 + 255) & ~(size_t)255;
    T *fwdv = reinterpret_cast<T *>(w);
    w += ((size_t)n * sizeof(T) + 255) & ~(size_t)255;
    uint32_t *desc = reinterpret_cast<uint32_t *>(w);

    for (uint32_t q = L; q < plan.nseg; q += SP_T) sh.segs[q] = plan.segs[q];
    for (uint32_t x = L; x < SP_B; x += SP_T) sh.head[x] = SP_NONE;
    if (L == 0) {
        sh.nint = 0;
        mbar_init(&sh.bar[0], 1);
        mbar_init(&sh.bar[1], 1);
    }
    __syncthreads();
    uint32_t par0 = 0, par1 = 0;
    for (int64_t a = blockIdx.x; a < num_arrays; a += gridDim.x) {
        T *z = data + a * (int64_t)n;
        T *res = res_all + a * (int64_t)n;
        uint16_t *slot = slot_all + a * (int64_t)n;
        // block sg into buffer b: one bulk copy by thread 0 (completion on bar[b]) or plain loads
        auto fetch = [&](int b, uint32_t sgf) {
            const uint32_t blo = sgf * SP_B;
            const uint32_t bn = min(SP_B, n - blo);
            if (use_tma) {
                if (L == 0) {
                    fence_proxy_async();  // earlier generic accesses to the buffer come first
                    mbar_arrive_expect_tx(&sh.bar[b], bn * (uint32_t)sizeof(T));
                    bulk_load(sh.mbuf[b], z + blo, bn * (uint32_t)sizeof(T), &sh.bar[b]);
                }
            } else {
                for (uint32_t x = L; x < bn; x += SP_T) sh.mbuf[b][x] = z[blo + x];
            }
        };
        SpGen g;
        sp_gen_init<T>(g, array_seed(run_seed, (uint64_t)(base + a)), gen == 1, L);
        int cur = 0;
        fetch(0, NB - 1);
        for (int sg = (int)NB - 1; sg >= 0; --sg) {
            const uint32_t blo = (uint32_t)sg * SP_B;
            const uint32_t bn = min(SP_B, n - blo);
            const uint32_t slo = max(blo, lo);  // positions below slo have no step
            T *mbox = sh.mbuf[cur];
            // ---- tile table of this block (prefetched by the previous stage into nd)
            const uint32_t ntile = NB - 1 - (uint32_t)sg;  // tile j comes from block NB-1-j
            for (uint32_t j = L; j < ntile; j += SP_T) {
                const uint32_t d = sh.nd[j];
                sh.vstart[j] = d & 0xFFFFu;
                sh.tbase[j] = (NB - 1 - j) * SP_B + (d >> 16);
            }
            if (use_tma) {
                if (cur == 0) {
                    mbar_wait(&sh.bar[0], par0);
                    par0 ^= 1u;
                } else {
                    mbar_wait(&sh.bar[1], par1);
                    par1 ^= 1u;
                }
            }
            __syncthreads();
            if (sg > 0) fetch(cur ^ 1, (uint32_t)sg - 1);  // the next block streams in meanwhile
            const uint32_t R = sp_scan(sh.vstart, ntile, sh.wsum, L);
            // ---- the next stage's tile table (all but this stage's own tile, written at its end)
            // and an L2 prefetch of its records
            if (sg > 0) {
                for (uint32_t j = L; j + 1 < NB - (uint32_t)sg; j += SP_T) {
                    const uint32_t sp = NB - 1 - j;
                    const uint32_t d = __ldcg(desc + (size_t)sp * NB + (uint32_t)(sg - 1));
                    sh.nd[j] = d;
                    const uint32_t cnt = d & 0xFFFFu;
                    if (cnt) {
                        const size_t first = (size_t)sp * SP_B + (d >> 16);
                        const uintptr_t q0 = (uintptr_t)(fwdq + first) & ~(uintptr_t)15;
                        const uintptr_t q1 = ((uintptr_t)(fwdq + first + cnt) + 15) & ~(uintptr_t)15;
                        const uintptr_t v0 = (uintptr_t)(fwdv + first) & ~(uintptr_t)15;
                        const uintptr_t v1 = ((uintptr_t)(fwdv + first + cnt) + 15) & ~(uintptr_t)15;
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q0), "r"((uint32_t)(q1 - q0))
                                     : "memory");
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(v0), "r"((uint32_t)(v1 - v0))
                                     : "memory");
                    }
                }
            }
            // ---- the block as the higher blocks left it: z0, then their deposits in time order.
            // Chunks of whole tiles (records of one tile are in no particular order; tiles are in
            // time order), as many as fit SP_C records; records of one chunk are ordered by key
            for (uint32_t jt = 0; jt < ntile;) {
                if (L == 0) {  // last tile je with end(je) - start(jt) <= SP_C
                    uint32_t a0 = jt, a1 = ntile - 1;
                    while (a0 < a1) {
                        const uint32_t mid = (a0 + a1 + 1) >> 1;
                        const uint32_t end = mid + 1 < ntile ? sh.vstart[mid + 1] : R;
                        if (end - sh.vstart[jt] <= SP_C) a0 = mid;
                        else a1 = mid - 1;
                    }
                    sh.chunk_end = a0 + 1;
                }
                __syncthreads();
                const uint32_t jn = sh.chunk_end;
                const uint32_t c0 = sh.vstart[jt];
                const uint32_t cn = (jn < ntile ? sh.vstart[jn] : R) - c0;
                const bool act = (uint32_t)(RPER * L) < cn;  // thread L takes records RPER*L + k
                uint32_t gi[RPER];
                bool last[RPER];
                if (act) {
                    uint32_t jj, a1 = jn - 1;
                    {
                        uint32_t a0 = jt;
                        const uint32_t rr = c0 + RPER * L;
                        while (a0 < a1) {
                            const uint32_t mid = (a0 + a1 + 1) >> 1;
                            if (sh.vstart[mid] <= rr) a0 = mid;
                            else a1 = mid - 1;
                        }
                        jj = a0;
                    }
#pragma unroll
                    for (int k = 0; k < RPER; ++k) {
                        const uint32_t r = RPER * (uint32_t)L + (uint32_t)k;
                        gi[k] = SP_NONE;
                        if (r < cn) {
                            const uint32_t rr = c0 + r;
                            while (jj + 1 < jn && sh.vstart[jj + 1] <= rr) ++jj;
                            gi[k] = sh.tbase[jj] + (rr - sh.vstart[jj]);
                        }
                    }
                    uint32_t fq[RPER];
                    T fv[RPER];
#pragma unroll
                    for (int k = 0; k < RPER; ++k)
                        if (gi[k] != SP_NONE) {
                            fq[k] = __ldcg(fwdq + gi[k]);
                            fv[k] = __ldcg(fwdv + gi[k]);
                        }
#pragma unroll
                    for (int k = 0; k < RPER; ++k)
                        if (gi[k] != SP_NONE) {
                            const uint32_t si = (uint32_t)k * SP_T + (uint32_t)L;  // conflict-free slot
                            const uint32_t q = fq[k] & 0xFFFFu;
                            // key = the step position s (the record lies in its source block's area)
                            sh.u.rec.key[si] = (gi[k] / SP_B) * SP_B + (fq[k] >> 16);
                            sh.u.rec.val[si] = fv[k];
                            sh.u.rec.q[si] = (uint16_t)q;
                            const uint32_t old = atomicExch(&sh.head[q], si);
                            sh.u.rec.link[si] = old == SP_NONE ? SP_NONE16 : (uint16_t)old;
                        }
                }
                __syncthreads();
                if (act) {
#pragma unroll
                    for (int k = 0; k < RPER; ++k) {
                        last[k] = false;
                        if (gi[k] != SP_NONE) {
                            const uint32_t si = (uint32_t)k * SP_T + (uint32_t)L;
                            const uint32_t K = sh.u.rec.key[si];
                            const uint32_t q = sh.u.rec.q[si];
                            uint32_t prev = SP_NONE, pk = SP_NONE;
                            bool lst = true;
                            for (uint32_t m = sh.head[q]; m != SP_NONE;) {
                                const uint32_t km = sh.u.rec.key[m];
                                if (km > K && km < pk) {
                                    pk = km;
                                    prev = m;
                                }
                                lst &= !(km < K);
                                const uint16_t nx = sh.u.rec.link[m];
                                m = nx == SP_NONE16 ? SP_NONE : nx;
                            }
                            __stcg(res + gi[k], prev != SP_NONE ? sh.u.rec.val[prev] : mbox[q]);
                            last[k] = lst;
                        }
                    }
                }
                __syncthreads();
                if (act) {
#pragma unroll
                    for (int k = 0; k < RPER; ++k)
                        if (gi[k] != SP_NONE) {
                            const uint32_t si = (uint32_t)k * SP_T + (uint32_t)L;
                            const uint32_t q = sh.u.rec.q[si];
                            if (last[k]) mbox[q] = sh.u.rec.val[si];
                            sh.head[q] = SP_NONE;
                        }
                }
                __syncthreads();
                jt = jn;
            }
            // ---- the targets of this block's steps
            sp_gen_block<T>(g, plan, sh, L, sp_batch_of(sh.segs, plan.nseg, slo));
            __syncthreads();
            // ---- this block's steps in closed form
            uint32_t Jr[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const uint32_t i = (uint32_t)L + (uint32_t)k * SP_T;
                const uint32_t s = blo + i;
                Jr[k] = SP_NONE;
                if (i < bn && s >= slo) {
                    const uint32_t J = sh.ring[s & (SP_RING - 1)];
                    Jr[k] = J;
                    if (J >= blo) {
                        const uint32_t old = atomicExch(&sh.head[J - blo], i);
                        sh.u.loc.link[i] = old == SP_NONE ? SP_NONE16 : (uint16_t)old;
                    }
                }
            }
            __syncthreads();
            uint16_t ns[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const uint32_t i = (uint32_t)L + (uint32_t)k * SP_T;
                ns[k] = SP_NONE16;
                if (i < bn) {
                    uint32_t ft = SP_NONE;  // first in-block step after i targeting i
                    for (uint32_t m = sh.head[i]; m != SP_NONE;) {
                        if (m > i && m < ft) ft = m;
                        const uint16_t nx = sh.u.loc.link[m];
                        m = nx == SP_NONE16 ? SP_NONE : nx;
                    }
                    sh.u.loc.F[i] = ft == SP_NONE ? SP_NONE16 : (uint16_t)ft;
                    if (Jr[k] != SP_NONE && Jr[k] >= blo) {  // next in-block step after i with i's target
                        uint32_t nx2 = SP_NONE;
                        for (uint32_t m = sh.head[Jr[k] - blo]; m != SP_NONE;) {
                            if (m > i && m < nx2) nx2 = m;
                            const uint16_t nx = sh.u.loc.link[m];
                            m = nx == SP_NONE16 ? SP_NONE : nx;
                        }
                        ns[k] = nx2 == SP_NONE ? SP_NONE16 : (uint16_t)nx2;
                    }
                }
            }
            for (uint32_t t = L; t < (uint32_t)sg; t += SP_T) sh.tbase[t] = 0;  // per-target-block counts
            __syncthreads();
            uint16_t endp[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const uint32_t i = (uint32_t)L + (uint32_t)k * SP_T;
                uint32_t e = i;
                if (i < bn)
                    for (uint16_t f = sh.u.loc.F[e]; f != SP_NONE16; f = sh.u.loc.F[e]) e = f;
                endp[k] = (uint16_t)e;
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const uint32_t i = (uint32_t)L + (uint32_t)k * SP_T;
                if (i < bn) sh.u.loc.F[i] = endp[k];
            }
            __syncthreads();
            // ---- outputs: in-block ones into the result area, records for lower blocks
            T ov[PER];
            uint32_t rk[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const uint32_t i = (uint32_t)L + (uint32_t)k * SP_T;
                rk[k] = 0;
                if (i >= bn) continue;
                const uint32_t J = Jr[k];
                if (J == SP_NONE) {  // no step at this position (below lo): its final value
                    ov[k] = mbox[sh.u.loc.F[i]];
                    rk[k] = atomicAdd(&sh.nint, 1u);
                } else if (J >= blo) {
                    ov[k] = mbox[ns[k] != SP_NONE16 ? sh.u.loc.F[ns[k]] : J - blo];
                    rk[k] = atomicAdd(&sh.nint, 1u);
                    sh.head[J - blo] = SP_NONE;
                } else {
                    ov[k] = mbox[sh.u.loc.F[i]];  // Val(s): the value leaving position s
                    rk[k] = atomicAdd(&sh.tbase[J / SP_B], 1u);
                }
            }
            __syncthreads();
            for (uint32_t t = L; t < (uint32_t)sg; t += SP_T) sh.vstart[t] = sh.tbase[t];
            __syncthreads();
            const uint32_t next = sp_scan(sh.vstart, (uint32_t)sg, sh.wsum, L);
            for (uint32_t t = L; t < (uint32_t)sg; t += SP_T)
                __stcg(desc + (size_t)sg * NB + t, (sh.vstart[t] << 16) | sh.tbase[t]);
            if (L == 0 && sg > 0) sh.nd[NB - 1 - (uint32_t)sg] = (sh.vstart[sg - 1] << 16) | sh.tbase[sg - 1];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const uint32_t i = (uint32_t)L + (uint32_t)k * SP_T;
                if (i >= bn) continue;
                const uint32_t J = Jr[k];
                uint32_t sl;
                if (J == SP_NONE || J >= blo) {
                    sl = next + rk[k];
                    __stcg(res + blo + sl, ov[k]);
                } else {
                    const uint32_t tb = J / SP_B;
                    sl = sh.vstart[tb] + rk[k];
                    __stcg(fwdq + blo + sl, (J - tb * SP_B) | (i << 16));
                    __stcg(fwdv + blo + sl, ov[k]);
                }
                __stcg(slot + blo + i, (uint16_t)sl);
            }
            if (L == 0) sh.nint = 0;
            __syncthreads();
            cur ^= 1;
        }
        if (L == 0 && words32) words32[a] = plan.nbatches + g.D;
    }
}

template <typename T>
__global__ void __launch_bounds__(SP_T, 2) shuffle_stage_kernel(T *__restrict__ data, int64_t num_arrays, DevPlan plan,
                                                             uint64_t run_seed, int64_t base,
                                                             uint32_t *__restrict__ words32, int gen,
                                                             unsigned char *__restrict__ cta_scratch, size_t cta_bytes,
                                                             T *__restrict__ res, uint16_t *__restrict__ slot,
                                                             int use_tma) {
    extern __shared__ __align__(16) unsigned char sp_smem[];
    auto &sh = *reinterpret_cast<SpShared<T> *>(sp_smem);
    shuffle_stage_body<T>(data, num_arrays, plan, run_seed, base, words32, gen, sh, cta_scratch, cta_bytes, res, slot,
                          use_tma);
}

// out[p] = result[slot[p]] for every block of every array: one block per iteration through
// shared memory (the slot map is a permutation of the block's result slots)
static constexpr int SPG_T = 512;
template <typename T>
__global__ void __launch_bounds__(SPG_T) shuffle_stage_gather_kernel(T *__restrict__ data, int64_t num_arrays,
                                                                     uint32_t n, const T *__restrict__ res,
                                                                     const uint16_t *__restrict__ slot) {
    __shared__ T buf[SP_B];
    const uint32_t NB = (n + SP_B - 1) / SP_B;
    const int64_t total = num_arrays * (int64_t)NB;
    for (int64_t g = blockIdx.x; g < total; g += gridDim.x) {
        const int64_t a = g / NB;
        const uint32_t blo = (uint32_t)(g - a * NB) * SP_B;
        const uint32_t bn = min(SP_B, n - blo);
        const int64_t off = a * (int64_t)n + blo;
        constexpr int PER = SP_B / SPG_T;
        T v[PER];
        uint16_t sl[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t x = threadIdx.x + k * SPG_T;
            if (x < bn) {
                v[k] = __ldcs(res + off + x);
                sl[k] = __ldcs(slot + off + x);
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
            if (x < bn) data[off + x] = buf[sl[k]];
        }
        __syncthreads();
    }
}

}  // namespace br
