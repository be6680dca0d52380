// roll.cuh -- bulk batched dice rolls (configs[1], "C2").
//
// Semantics: the sequential loop
//     for i in range(nb): roll_batch(src, BatchSpec(RadixBases.of(bounds[i*k:(i+1)*k])))
// of batched.py:102-123 on one PCG64 stream.  Batch i consumes word i + D_i, where D_i
// counts the extra words drawn by rejected batches before it (a rejection re-draws the
// WHOLE batch from the next word, batched.py:120-122).
//
// Parallel form (one HBM pass in the common case):
//   roll_main   every warp owns a contiguous batch range, lane l takes batches l, l+32, ...
//               (coalesced 256 B bound loads / roll stores per warp instruction) and jumps
//               its PCG64 lane state by 32 words per step; it SPECULATES D_i = 0 and marks
//               the first rejected batch (atomicMax of ~i).  P(reject) <= 2^-32 per batch
//               for bounds < 2^16, so the speculation is almost always right.
//   roll_fixup  cooperative grid, always launched: if nothing was rejected it only writes
//               the advanced state; otherwise it resolves the first rejected batch
//               (re-draw from the next word), re-runs the tail with the new shift, and
//               repeats until no rejection is left -- exact for any rejection rate.
#pragma once
#include "chacha.cuh"
#include "jump.cuh"

namespace br {

// the fixup kernel runs one 256-thread block per SM: at most this many warps (256 SMs)
constexpr int ROLL_MAX_WARPS = 2048;

struct RollWs {
    unsigned long long neg_first;  // ~(first rejected batch); 0 = none
    unsigned long long D;          // shift published by the fixup resolver
    unsigned long long extra;      // words consumed beyond one per batch (last call)
    unsigned int error;            // deferred status (BR_E_INVALID / BR_E_BOUND_OVERFLOW)
    unsigned int bar_count;
    unsigned int bar_gen;
    unsigned int main_done;  // 1: this call's main kernel rolled the stream (else the fixup does)
    unsigned int pad[2];
    unsigned long long final_hi, final_lo;  // state after nb words (no-rejection case), by the main kernel
    unsigned long long q[3];  // fixup iteration i records its first rejection in q[i % 3]; all 0 between calls
    unsigned long long prof[4];  // BR_FIXUP_PROF builds: block 0's ns in re-run / barrier / record reads, iterations
    // Per-warp resolutions of the fixup (iteration i writes rec[i % 2]): the first rejected
    // batch a warp met in its round, already re-drawn by the lane that met it
    struct Rec {
        unsigned long long extra;  // words beyond the first
        unsigned long long hi, lo;  // PCG64 / Lehmer: the state whose output is the next batch's word
        unsigned long long pad;
    } rec[2][ROLL_MAX_WARPS];
};

// Programmatic dependent launch: the main kernel lets the fixup kernel be scheduled early;
// the fixup waits for the main grid's completion (and memory) before reading anything.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

struct RollArgs {
    const uint32_t *__restrict__ bounds;
    int k;
    int64_t nb;
    uint64_t *state;  // br_pcg64 {state_hi, state_lo, inc_hi, inc_lo}, in/out
    uint32_t *__restrict__ rolls;
    uint8_t *__restrict__ words;
    uint8_t *__restrict__ flags;
    uint64_t *__restrict__ rk;
    RollWs *ws;
    int naive;  // digits by division of one draw on the product (batched.py:126-128)
};

// roll_batch_naive (batched.py:126-128): value v = hi(P*w) of one Lemire draw on the
// product P, decoded by divisions (mixed_radix.py:53-67), least significant digit first.
// Accepts exactly when the batched form does (Theorem 1: r_k == P*w mod 2^64), so only the
// digit extraction differs -- the k-1 divisions are what the baseline measures.
template <int K>
__device__ __forceinline__ void naive_digits(const uint32_t (&b)[K], uint64_t v, uint32_t (&d)[K]) {
#pragma unroll
    for (int m = K - 1; m > 0; --m) {
        const uint64_t q = v / b[m];
        d[m] = (uint32_t)(v - q * b[m]);
        v = q;
    }
    d[0] = (uint32_t)v;
}

// Evaluate one batch on word w (batched.py:102-123).  Returns 0 accept, 1 reject,
// 2 invalid bases (err set).  d[] receives the digits, r the final remainder.
template <int K>
__device__ __forceinline__ int eval_batch(const uint32_t (&b)[K], uint64_t w, uint32_t (&d)[K],
                                          uint64_t &r, uint8_t &tc, int &err, bool naive = false) {
    r = w;
    if (!naive || K == 1) {
#pragma unroll
        for (int m = 0; m < K; ++m) d[m] = die(b[m], r);
    }
    uint64_t prod;
    bool full = false;
    if constexpr (K == 1) {
        if (b[0] == 0) { err = 1; return 2; }
        prod = b[0];
    } else if constexpr (K == 2) {
        if (b[0] == 0 || b[1] == 0) { err = 1; return 2; }
        prod = (uint64_t)b[0] * b[1];
    } else {
        bool zero = false;
#pragma unroll
        for (int m = 0; m < K; ++m) zero |= (b[m] == 0);
        if (zero) { err = 1; return 2; }
        // exact product with overflow detection (mixed_radix.py:33-34)
        uint64_t lo = 1, hi = 0;
#pragma unroll
        for (int m = 0; m < K; ++m) {
            uint64_t nlo = lo * b[m];
            uint64_t nhi = hi * b[m] + mulhi64(lo, b[m]);
            lo = nlo;
            hi = nhi;
            if (hi > 1 || (hi == 1 && lo != 0)) { err = 2; return 2; }
        }
        full = (hi == 1);
        prod = lo;
    }
    if (naive && K > 1) {  // one draw on the product, digits by division (bases are non-zero here)
        naive_digits<K>(b, full ? w : mulhi64(prod, w), d);
        r = full ? 0 : prod * w;
    }
    if (full) { tc = 1; return 0; }  // product 2^64: threshold 0, always accepted
    if (r >= prod) { tc = 0; return 0; }
    tc = 1;
    uint64_t t = (0 - prod) % prod;  // 2^64 mod prod, the only remainder (batched.py:119)
    return r < t ? 1 : 0;
}

template <int K>
__device__ __forceinline__ void load_bounds(const uint32_t *__restrict__ p, uint32_t (&b)[K]) {
    if constexpr (K == 2) {
        uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
        b[0] = v.x;
        b[1] = v.y;
    } else if constexpr (K == 4) {
        uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
        b[0] = v.x;
        b[1] = v.y;
        b[2] = v.z;
        b[3] = v.w;
    } else {
#pragma unroll
        for (int m = 0; m < K; ++m) b[m] = __ldg(p + m);
    }
}

template <int K>
__device__ __forceinline__ void store_rolls(uint32_t *__restrict__ p, const uint32_t (&d)[K]) {
    if constexpr (K == 2) {
        *reinterpret_cast<uint2 *>(p) = make_uint2(d[0], d[1]);
    } else if constexpr (K == 4) {
        *reinterpret_cast<uint4 *>(p) = make_uint4(d[0], d[1], d[2], d[3]);
    } else {
#pragma unroll
        for (int m = 0; m < K; ++m) p[m] = d[m];
    }
}

__device__ __forceinline__ void set_error(RollWs *ws, int err) {
    atomicCAS(&ws->error, 0u, (unsigned)err);
}

// Speculative pass over batches [begin, end): batch i uses word i (no earlier rejection);
// warp w owns one contiguous range.
template <int K, int U>
__device__ __forceinline__ void roll_range(const RollArgs &a, u128 s0, u128 inc, int64_t begin, int64_t end) {
    const bool lh = is_lehmer(inc);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t total = end - begin;
    if (total <= 0) return;
    const int64_t per = (((total + nwarps - 1) / nwarps) + 31) & ~(int64_t)31;
    const int64_t wb = begin + warp * per;
    const int64_t we = min(wb + per, end);
    if (wb >= we) return;
    // lane state: word index wb + lane  ->  state index (word index + 1)
    u128 s = gen_jump(s0, inc, (uint64_t)wb, lh);
    s = gen_jump_small(s, inc, lane + 1, lh);
    const u128 A32 = gen_SA(lh, 32);
    const u128 C32 = mul128(g_SG[32], inc);
    int err = 0;
    // software pipeline: the bounds of the next U*32 batches are in flight while the
    // current ones are rolled
    uint32_t cur[U][K], nxt[U][K];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t b = wb + 32 * u + lane;
        if (b < we) load_bounds<K>(a.bounds + b * K, cur[u]);
    }
    for (int64_t b0 = wb; b0 < we; b0 += 32 * U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t b = b0 + 32 * (U + u) + lane;
            if (b < we) load_bounds<K>(a.bounds + b * K, nxt[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t b = b0 + 32 * u + lane;
            if (b < we) {
                const uint64_t w = gen_out(s, lh);
                uint32_t d[K];
                uint64_t r;
                uint8_t tc = 0;
                int st = eval_batch<K>(cur[u], w, d, r, tc, err, a.naive != 0);
                store_rolls<K>(a.rolls + b * K, d);
                a.words[b] = 1;
                if (a.flags) a.flags[b] = tc;
                if (a.rk) a.rk[b] = r;
                if (st == 1) atomicMax(&a.ws->neg_first, ~(unsigned long long)b);
            }
            s = K >= 3 ? mad128_wide(s, A32, C32) : mad128(s, A32, C32);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int m = 0; m < K; ++m) cur[u][m] = nxt[u][m];
    }
    if (err) set_error(a.ws, err);
}

// state after nb words, for the fixup kernel's no-rejection case (one lane of the grid)
__device__ __forceinline__ void publish_final(const RollArgs &a, u128 s0, u128 inc) {
    const bool lh = is_lehmer(inc);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const u128 sf = gen_jump(s0, inc, (uint64_t)a.nb, lh);
        a.ws->final_hi = sf.hi;
        a.ws->final_lo = sf.lo;
    }
}

// ---- ChaCha streams.  Only the device state says which generator a stream is (tag in
// inc_lo, key after the head), so every roll kernel checks it and branches here.  Warp w
// owns a contiguous batch range; lane l of a sub-step takes batch b0 + l, whose word
// (position s0 + b) comes from the warp's 256-word keystream window.
template <int K>
__device__ __forceinline__ void roll_range_cha(const RollArgs &a, u128 s0, int64_t begin, int64_t end,
                                               uint64_t *win) {
    const ChaKey ck = cha_key_of_state(a.state);
    const uint32_t lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t total = end - begin;
    if (total <= 0) return;
    const int64_t per = (((total + nwarps - 1) / nwarps) + 31) & ~(int64_t)31;
    const int64_t wb = begin + warp * per;
    const int64_t we = min(wb + per, end);
    if (wb >= we) return;  // warp-uniform
    u128 W0 = cha_win_unset(cha_add(s0, (uint64_t)wb));
    int err = 0;
    // windows of U sub-steps: the bounds of all U are requested before the keystream block
    // computation, which then hides their latency
    constexpr int U = K <= 2 ? 8 : 4;
    for (int64_t c0 = wb; c0 < we; c0 += 32 * U) {
        uint32_t bb[U][K];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t b = c0 + 32 * u + lane;
            if (b < we) load_bounds<K>(a.bounds + b * K, bb[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t b = c0 + 32 * u + lane;
            if (c0 + 32 * u >= we) break;  // warp-uniform
            const uint64_t w = cha_warp_word(win, ck, W0, cha_add(s0, (uint64_t)b), lane);
            if (b < we) {
                uint32_t d[K];
                uint64_t r;
                uint8_t tc = 0;
                const int st = eval_batch<K>(bb[u], w, d, r, tc, err, a.naive != 0);
                store_rolls<K>(a.rolls + b * K, d);
                a.words[b] = 1;
                if (a.flags) a.flags[b] = tc;
                if (a.rk) a.rk[b] = r;
                if (st == 1) atomicMax(&a.ws->neg_first, ~(unsigned long long)b);
            }
        }
    }
    if (err) set_error(a.ws, err);
}

// speculative main pass of a ChaCha stream: run by the (cooperative) fixup kernel itself,
// so the PCG64 main kernels only carry a one-compare early exit
template <int K>
__device__ __forceinline__ void roll_cha_main(const RollArgs &a, uint64_t *win) {
    const u128 s0 = mk128(a.state[0], a.state[1]);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const u128 sf = cha_add(s0, (uint64_t)a.nb);
        a.ws->final_hi = sf.hi;
        a.ws->final_lo = sf.lo;
    }
    roll_range_cha<K>(a, s0, 0, a.nb, win);
}

// ChaCha keystreams and replayed word sequences take the position-addressed roll path
__device__ __forceinline__ bool roll_is_chacha(const RollArgs &a) {
    return a.state[3] == CHACHA_TAG || a.state[3] == WORDS_TAG;
}

// Which main kernel runs is the host's guess (the generator of a state buffer is known where
// it was uploaded); the device has the final word: a main kernel that does not match the
// stream's tag exits and records main_done = 0, and the fixup kernel then rolls the stream
// itself.  One writer (block 0, thread 0), read by the fixup after griddepcontrol.wait.
__device__ __forceinline__ void mark_main(const RollArgs &a, unsigned done) {
    if (blockIdx.x == 0 && threadIdx.x == 0) a.ws->main_done = done;
}

// ChaCha main pass at full occupancy (launched when the host knows the stream is ChaCha).
// Each thread owns whole keystream blocks: block m (positions 8m..8m+7) is computed once in
// registers and rolls the batches whose words it holds (batch b uses position s0 + b), so
// no word goes through shared memory.  Bounds and rolls move 8 bytes per batch with lanes
// 64 bytes apart; consecutive batches of a lane reuse the same sectors (L1 for loads, L2
// write combining for stores).
template <int K>
__global__ void __launch_bounds__(256) roll_cha_kernel(RollArgs a) {
    pdl_launch_dependents();
    if (!roll_is_chacha(a)) {
        mark_main(a, 0);
        return;
    }
    mark_main(a, 1);
    const u128 s0 = mk128(a.state[0], a.state[1]);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const u128 sf = cha_add(s0, (uint64_t)a.nb);
        a.ws->final_hi = sf.hi;
        a.ws->final_lo = sf.lo;
    }
    const ChaKey ck = cha_key_of_state(a.state);
    const uint32_t q0 = (uint32_t)(s0.lo & 7);          // word of the first block that is batch 0
    const uint64_t blk0 = cha_block_of(s0);
    const int64_t nblk = ((int64_t)q0 + a.nb + 7) >> 3;
    int err = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nblk; t += (int64_t)gridDim.x * blockDim.x) {
        uint32_t kb[16];
        cha_block_any(ck, blk0 + (uint64_t)t, kb);
        const int64_t b0 = t * 8 - q0;  // batch of word 0 of this block
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int64_t b = b0 + q;
            if (b < 0 || b >= a.nb) continue;
            const uint64_t w = ((uint64_t)kb[2 * q + 1] << 32) | kb[2 * q];
            uint32_t bb[K], d[K];
            load_bounds<K>(a.bounds + b * K, bb);
            uint64_t r;
            uint8_t tc = 0;
            const int st = eval_batch<K>(bb, w, d, r, tc, err, a.naive != 0);
            store_rolls<K>(a.rolls + b * K, d);
            a.words[b] = 1;
            if (a.flags) a.flags[b] = tc;
            if (a.rk) a.rk[b] = r;
            if (st == 1) atomicMax(&a.ws->neg_first, ~(unsigned long long)b);
        }
    }
    if (err) set_error(a.ws, err);
}

template <int K>
__global__ void __launch_bounds__(256) roll_main_kernel(RollArgs a) {
    pdl_launch_dependents();
    if (roll_is_chacha(a)) {  // the fixup kernel rolls ChaCha streams met here
        mark_main(a, 0);
        return;
    }
    mark_main(a, 1);
    const u128 s0 = mk128(a.state[0], a.state[1]);
    const u128 inc = mk128(a.state[2], a.state[3]);
    publish_final(a, s0, inc);
    roll_range<K, 4>(a, s0, inc, 0, a.nb);
}


// Rare path of the fast kernel, out of line: zero bounds, and batches whose final
// remainder fell below the product (threshold needed; P < 2^-32 per batch for C2).
__device__ __noinline__ void roll_slow(RollWs *ws, uint8_t *flags, int64_t b, uint64_t r, uint64_t prod) {
    if (prod == 0) {
        set_error(ws, 1);  // a zero bound (mixed_radix.py:31-32: bases must be positive)
        return;
    }
    if (flags) flags[b] = 1;
    const uint64_t t = (0 - prod) % prod;
    if (r < t) atomicMax(&ws->neg_first, ~(unsigned long long)b);
}

// Main kernel for k <= 2 (the C2 shape): every lane moves 16 bytes of bounds per load
// (VB = 4/K batches), four loads in flight, and rolls 16 bytes / words VB bytes per store.
// Lane l of sub-step u owns batches base + 32*VB*u + VB*l + v (v < VB); its words come
// from VB consecutive PCG steps, the lane state then jumps 32*VB words.
#ifndef ROLL_U
#define ROLL_U 8
#endif
#ifndef ROLL_MINB
#define ROLL_MINB 2
#endif
#ifndef ROLL_LB
#define ROLL_LB 16
#endif

// LB bytes of consecutive u32 per lane.  32-byte lanes use Blackwell's 256-bit
// LDG/STG (LDG.E.NA.EFL2.256) with L1 no-allocate / L2 evict-first: bounds are read once and
// rolls written once, so neither should displace anything in L2.
template <int LB>
struct Vec {
    uint32_t v[LB / 4];
};

template <int LB>
__device__ __forceinline__ Vec<LB> ld_vec(const uint32_t *p) {
    Vec<LB> r;
    if constexpr (LB == 32) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                       "=r"(r.v[6]), "=r"(r.v[7])
                     : "l"(p));
    } else {
        const uint4 x = __ldg(reinterpret_cast<const uint4 *>(p));
        r.v[0] = x.x;
        r.v[1] = x.y;
        r.v[2] = x.z;
        r.v[3] = x.w;
    }
    return r;
}

template <int LB>
__device__ __forceinline__ void st_vec(uint32_t *p, const Vec<LB> &r) {
    if constexpr (LB == 32) {
        asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                     "r"(r.v[0]), "r"(r.v[1]), "r"(r.v[2]), "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]), "r"(r.v[6]),
                     "r"(r.v[7])
                     : "memory");
    } else {
        *reinterpret_cast<uint4 *>(p) = make_uint4(r.v[0], r.v[1], r.v[2], r.v[3]);
    }
}

// Main kernel for k <= 2 (the C2 shape): every lane moves LB bytes of bounds per load
// (VB = LB/(4K) batches), U loads in flight, and rolls LB bytes / words VB bytes per store.
// Lane l of sub-step u owns batches base + 32*VB*u + VB*l + v (v < VB); its words come
// from VB consecutive generator steps, the lane state then jumps 32*VB words.  The
// generator kind (PCG64 or Lehmer: inc == 0) is a template of the loop, chosen once.  The
// rare path (r_k below the product: threshold needed; or a zero bound) is flagged per batch
// and handled after the sub-step by re-deriving its words (fast_recheck).
template <int K, bool NAIVE, bool LH, int VB, int LB>
__device__ __noinline__ void fast_recheck(RollWs *ws, uint8_t *flags, u128 st, u128 inc, Vec<LB> bv, int64_t b0,
                                          unsigned bad) {
    const uint32_t *bb = bv.v;
    const u128 M = gen_mult(LH);
    for (int v = 0; v < VB; ++v) {
        if ((bad >> v) & 1u) {
            uint64_t r = gen_out(st, LH);
            uint64_t prod;
            if constexpr (K == 2 && NAIVE) {
                prod = (uint64_t)bb[2 * v] * bb[2 * v + 1];
                r = prod * r;
            } else if constexpr (K == 2) {
                die(bb[2 * v], r);
                die(bb[2 * v + 1], r);
                prod = (uint64_t)bb[2 * v] * bb[2 * v + 1];
            } else {
                die(bb[v], r);
                prod = bb[v];
            }
            roll_slow(ws, flags, b0 + v, r, prod);
        }
        st = mad128(st, M, inc);
    }
}

template <int K, bool FLAGS, bool RK, bool NAIVE, bool LH>
__device__ __forceinline__ void roll_fast_body(const RollArgs &a, u128 s0, u128 inc) {
    constexpr int LB = ROLL_LB;
    constexpr int VB = LB / (4 * K);
    static_assert(32 * VB <= JUMP_SMALL, "jump table covers the lane offsets");
    constexpr int U = ROLL_U;
    constexpr int64_t CH = 32 * VB * U;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nchunks = a.nb / CH;
    const int64_t cpw = (nchunks + nwarps - 1) / nwarps;
    const int64_t c0 = warp * cpw, c1 = min(c0 + cpw, nchunks);
    const u128 M = gen_mult(LH);
    if (c0 < c1) {
        const int64_t wb = c0 * CH;
        u128 s = gen_jump(s0, inc, (uint64_t)wb, LH);
        s = gen_jump_small(s, inc, VB * lane + 1, LH);
        const u128 AJ = gen_SA(LH, 32 * VB);
        const u128 CJ = mul128(g_SG[32 * VB], inc);
        const uint32_t *bp = a.bounds + (wb + VB * lane) * K;
        uint32_t *rp = a.rolls + (wb + VB * lane) * K;
        uint8_t *wp = a.words + wb + VB * lane;
        constexpr int STEP = 32 * VB * K;  // u32 per sub-step
        Vec<LB> cur[U], nxt[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cur[u] = ld_vec<LB>(bp + STEP * u);
        for (int64_t c = c0; c < c1; ++c) {
            if (c + 1 < c1) {
#pragma unroll
                for (int u = 0; u < U; ++u) nxt[u] = ld_vec<LB>(bp + STEP * (U + u));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                Vec<LB> dd;
                u128 st = s;
                const int64_t b0 = wb + (c - c0) * CH + 32 * VB * u + VB * lane;
                unsigned bad = 0;
#pragma unroll
                for (int v = 0; v < VB; ++v) {
                    uint64_t r = gen_out(st, LH);
                    uint64_t prod;
                    if constexpr (K == 2 && NAIVE) {  // roll_batch_naive: one division by b1
                        const uint32_t b1 = cur[u].v[2 * v + 1];
                        prod = (uint64_t)cur[u].v[2 * v] * b1;
                        const uint64_t val = mulhi64(prod, r);
                        r = prod * r;
                        const uint64_t q = b1 ? val / b1 : 0;
                        dd.v[2 * v] = (uint32_t)q;
                        dd.v[2 * v + 1] = (uint32_t)(val - q * b1);
                    } else if constexpr (K == 2) {
                        dd.v[2 * v] = die(cur[u].v[2 * v], r);
                        dd.v[2 * v + 1] = die(cur[u].v[2 * v + 1], r);
                        prod = (uint64_t)cur[u].v[2 * v] * cur[u].v[2 * v + 1];
                    } else {
                        dd.v[v] = die(cur[u].v[v], r);
                        prod = cur[u].v[v];
                    }
                    if constexpr (FLAGS) a.flags[b0 + v] = r < prod;
                    if constexpr (RK) a.rk[b0 + v] = r;
                    bad |= (unsigned)(r < prod || prod == 0) << v;
                    if (v + 1 < VB) st = mad128_wide(st, M, inc);
                }
                if (__builtin_expect(bad != 0, 0)) fast_recheck<K, NAIVE, LH, VB, LB>(a.ws, a.flags, s, inc, cur[u], b0, bad);
                st_vec<LB>(rp + STEP * u, dd);
                if constexpr (VB == 2)
                    *reinterpret_cast<uint16_t *>(wp + 32 * VB * u) = 0x0101;
                else if constexpr (VB == 4)
                    *reinterpret_cast<uint32_t *>(wp + 32 * VB * u) = 0x01010101u;
                else
                    *reinterpret_cast<uint2 *>(wp + 32 * VB * u) = make_uint2(0x01010101u, 0x01010101u);
                s = mad128_wide(s, AJ, CJ);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) cur[u] = nxt[u];
            bp += STEP * U;
            rp += STEP * U;
            wp += CH;
        }
    }
    // the last partial chunk (< CH batches) with the generic per-batch path
    if (nchunks * CH < a.nb) roll_range<K, 1>(a, s0, inc, nchunks * CH, a.nb);
}

// k = 2 (C2): one loop with the generator kind as a runtime value and the rare-path test
// inline; the templated form below spills at this shape (measured 12% slower on C2)
template <int K, bool FLAGS, bool RK, bool NAIVE>
__device__ __forceinline__ void roll_fast_body_rt(const RollArgs &a) {
    constexpr int LB = ROLL_LB;
    constexpr int VB = LB / (4 * K);
    static_assert(32 * VB <= JUMP_SMALL, "jump table covers the lane offsets");
    constexpr int U = ROLL_U;
    constexpr int64_t CH = 32 * VB * U;
    const u128 s0 = mk128(a.state[0], a.state[1]);
    const u128 inc = mk128(a.state[2], a.state[3]);
    const bool lh = is_lehmer(inc);
    publish_final(a, s0, inc);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nchunks = a.nb / CH;
    const int64_t cpw = (nchunks + nwarps - 1) / nwarps;
    const int64_t c0 = warp * cpw, c1 = min(c0 + cpw, nchunks);
    const u128 M = gen_mult(lh);
    if (c0 < c1) {
        const int64_t wb = c0 * CH;
        u128 s = gen_jump(s0, inc, (uint64_t)wb, lh);
        s = gen_jump_small(s, inc, VB * lane + 1, lh);
        const u128 AJ = gen_SA(lh, 32 * VB);
        const u128 CJ = mul128(g_SG[32 * VB], inc);
        const uint32_t *bp = a.bounds + (wb + VB * lane) * K;
        uint32_t *rp = a.rolls + (wb + VB * lane) * K;
        uint8_t *wp = a.words + wb + VB * lane;
        constexpr int STEP = 32 * VB * K;  // u32 per sub-step
        Vec<LB> cur[U], nxt[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cur[u] = ld_vec<LB>(bp + STEP * u);
        for (int64_t c = c0; c < c1; ++c) {
            if (c + 1 < c1) {
#pragma unroll
                for (int u = 0; u < U; ++u) nxt[u] = ld_vec<LB>(bp + STEP * (U + u));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                Vec<LB> dd;
                u128 st = s;
                const int64_t b0 = wb + (c - c0) * CH + 32 * VB * u + VB * lane;
#pragma unroll
                for (int v = 0; v < VB; ++v) {
                    uint64_t r = gen_out(st, lh);
                    uint64_t prod;
                    if constexpr (K == 2 && NAIVE) {  // roll_batch_naive: one division by b1
                        const uint32_t b1 = cur[u].v[2 * v + 1];
                        prod = (uint64_t)cur[u].v[2 * v] * b1;
                        const uint64_t val = mulhi64(prod, r);
                        r = prod * r;
                        const uint64_t q = b1 ? val / b1 : 0;
                        dd.v[2 * v] = (uint32_t)q;
                        dd.v[2 * v + 1] = (uint32_t)(val - q * b1);
                    } else if constexpr (K == 2) {
                        dd.v[2 * v] = die(cur[u].v[2 * v], r);
                        dd.v[2 * v + 1] = die(cur[u].v[2 * v + 1], r);
                        prod = (uint64_t)cur[u].v[2 * v] * cur[u].v[2 * v + 1];
                    } else {
                        dd.v[v] = die(cur[u].v[v], r);
                        prod = cur[u].v[v];
                    }
                    if constexpr (FLAGS) a.flags[b0 + v] = r < prod;
                    if constexpr (RK) a.rk[b0 + v] = r;
                    if (__builtin_expect(r < prod || prod == 0, 0)) roll_slow(a.ws, a.flags, b0 + v, r, prod);
                    if (v + 1 < VB) st = mad128(st, M, inc);
                }
                st_vec<LB>(rp + STEP * u, dd);
                if constexpr (VB == 2)
                    *reinterpret_cast<uint16_t *>(wp + 32 * VB * u) = 0x0101;
                else if constexpr (VB == 4)
                    *reinterpret_cast<uint32_t *>(wp + 32 * VB * u) = 0x01010101u;
                else
                    *reinterpret_cast<uint2 *>(wp + 32 * VB * u) = make_uint2(0x01010101u, 0x01010101u);
                s = mad128(s, AJ, CJ);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) cur[u] = nxt[u];
            bp += STEP * U;
            rp += STEP * U;
            wp += CH;
        }
    }
    if (nchunks * CH < a.nb) roll_range<K, 1>(a, s0, inc, nchunks * CH, a.nb);
}

template <int K, bool FLAGS, bool RK, bool NAIVE = false>
__global__ void __launch_bounds__(256, ROLL_MINB) roll_fast_kernel(RollArgs a) {
    static_assert(K == 1 || K == 2, "fast path is for k <= 2");
    pdl_launch_dependents();
    if (roll_is_chacha(a)) {  // the fixup kernel rolls ChaCha streams met here
        mark_main(a, 0);
        return;
    }
    mark_main(a, 1);
    if constexpr (K == 2) {
        roll_fast_body_rt<K, FLAGS, RK, NAIVE>(a);
    } else {
        const u128 s0 = mk128(a.state[0], a.state[1]);
        const u128 inc = mk128(a.state[2], a.state[3]);
        publish_final(a, s0, inc);
        if (is_lehmer(inc)) roll_fast_body<K, FLAGS, RK, NAIVE, true>(a, s0, inc);
        else roll_fast_body<K, FLAGS, RK, NAIVE, false>(a, s0, inc);
    }
}

// Fixup re-run of batches [begin, end) at shift D (batch b uses word b + D), front first:
// round r gives each warp one chunk of CHK = 32*U consecutive batches out of the nwarps*CHK
// batches that follow begin + r*nwarps*CHK, so once a rejection is recorded in `slot`, every
// warp stops after the round it is in.  (With one contiguous range per warp, each warp would
// roll ~1/rejection-rate batches of its own range before the first rejection is known: about
// nwarps/rate batches per resolved rejection, measured 40 us each at a rate of 1e-3.)
template <bool CHA, int K>
struct FrontPlan {
    static constexpr int U = CHA ? (K <= 2 ? 8 : 4) : 4;
    static constexpr int64_t CHK = 32 * U;
    u128 AL, CL;    // word offset warp*CHK + lane (the lane's first batch of a round)
    u128 AS, CS;    // one round: nwarps*CHK words
    u128 A32, C32;  // one sub-step: 32 words
};

// once per fixup kernel (PCG64 / Lehmer streams)
template <bool CHA, int K>
__device__ __forceinline__ FrontPlan<CHA, K> front_plan(u128 inc, bool lh) {
    FrontPlan<CHA, K> p{};
    if constexpr (!CHA) {
        const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
        gen_affine((uint64_t)(warp * p.CHK + (threadIdx.x & 31)), inc, lh, p.AL, p.CL);
        gen_affine((uint64_t)(nwarps * p.CHK), inc, lh, p.AS, p.CS);
        p.A32 = gen_SA(lh, 32);
        p.C32 = mul128(g_SG[32], inc);
    }
    return p;
}

// sb: (PCG64 / Lehmer) the state whose output is word begin + D
// A warp's first rejected batch is re-drawn on the spot by the lane that met it (outputs
// written, result in the warp's record), and the warp stops: the grid-wide first rejection
// is some warp's first, so after the barrier every block finds its resolution in one record.
template <int K, bool CHA>
__device__ __forceinline__ void redraw_lane(const RollArgs &a, u128 s0, u128 inc, bool lh, u128 st, int64_t b,
                                            uint64_t D, RollWs::Rec *rec) {
    const uint64_t widx = (uint64_t)b + D + 1;
    uint32_t bb[K];
    load_bounds<K>(a.bounds + b * K, bb);  // cached: the lane just read them
    ChaKey ck;
    ChaCursor cc;
    cc.valid = false;
    if constexpr (CHA) {
        ck = cha_key_of_state(a.state);
        st = cha_add(s0, widx + 1);
    } else {
        st = mad128(st, gen_mult(lh), inc);  // st output word b + D: now word widx
    }
    uint64_t extra = 1;
    for (;;) {
        uint32_t d[K];
        uint64_t r;
        uint8_t tc;
        int err = 0;
        const uint64_t w = CHA ? cha_out_cached(ck, cc, st) : gen_out(st, lh);
        if (eval_batch<K>(bb, w, d, r, tc, err, a.naive != 0) != 1) {
            store_rolls<K>(a.rolls + b * K, d);
            a.words[b] = (uint8_t)(1 + extra > 255 ? 255 : 1 + extra);
            if (a.flags) a.flags[b] = 1;
            if (a.rk) a.rk[b] = r;
            break;
        }
        ++extra;
        st = CHA ? cha_add(st, 1) : mad128(st, gen_mult(lh), inc);
    }
    if constexpr (!CHA) st = mad128(st, gen_mult(lh), inc);
    rec->extra = extra;
    rec->hi = st.hi;
    rec->lo = st.lo;
}

template <int K, bool CHA>
__device__ __forceinline__ void roll_front(const RollArgs &a, u128 s0, u128 inc, u128 sb, const FrontPlan<CHA, K> &fp,
                                           bool lh, int64_t begin, int64_t end, uint64_t D,
                                           unsigned long long *slot, RollWs::Rec *recs, uint64_t *win) {
    constexpr int U = FrontPlan<CHA, K>::U;
    constexpr int64_t CHK = FrontPlan<CHA, K>::CHK;
    const uint32_t lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t stride = nwarps * CHK;
    int64_t c0 = begin + warp * CHK;
    if (c0 >= end) return;  // warp-uniform
    volatile unsigned long long *vslot = slot;
    u128 s, W0;
    ChaKey ck;
    if constexpr (CHA) {
        ck = cha_key_of_state(a.state);
        W0 = cha_win_unset(cha_add(s0, (uint64_t)c0 + D));
    } else {
        s = mad128(sb, fp.AL, fp.CL);  // lane state: word c0 + D + lane
    }
    int err = 0;
    uint32_t cur[U][K], nxt[U][K];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t b = c0 + 32 * u + lane;
        if (b < end) load_bounds<K>(a.bounds + b * K, cur[u]);
    }
    for (; c0 < end; c0 += stride) {
        unsigned long long nf = lane == 0 ? *vslot : 0ull;
        nf = __shfl_sync(0xFFFFFFFFu, nf, 0);
        if (nf != 0 && (int64_t)(~nf) < c0) break;  // an earlier rejection supersedes this round
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t b = c0 + stride + 32 * u + lane;
            if (b < end) load_bounds<K>(a.bounds + b * K, nxt[u]);
        }
        u128 st = s;
        bool hit = false;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t b = c0 + 32 * u + lane;
            if (c0 + 32 * u >= end) break;  // warp-uniform
            uint64_t w;
            if constexpr (CHA) w = cha_warp_word(win, ck, W0, cha_add(s0, (uint64_t)b + D), lane);
            else w = gen_out(st, lh);
            int res = 0;
            if (b < end) {
                uint32_t d[K];
                uint64_t r;
                uint8_t tc = 0;
                res = eval_batch<K>(cur[u], w, d, r, tc, err, a.naive != 0);
                store_rolls<K>(a.rolls + b * K, d);
                a.words[b] = 1;
                if (a.flags) a.flags[b] = tc;
                if (a.rk) a.rk[b] = r;
            }
            const unsigned m = __ballot_sync(0xFFFFFFFFu, res == 1);
            if (m) {
                if (lane == (uint32_t)(__ffs(m) - 1)) {
                    atomicMax(slot, ~(unsigned long long)b);
                    redraw_lane<K, CHA>(a, s0, inc, lh, st, b, D, &recs[warp]);
                }
                hit = true;
                break;
            }
            if constexpr (!CHA) st = mad128(st, fp.A32, fp.C32);
        }
        if (hit) break;
        if constexpr (!CHA) s = mad128(s, fp.AS, fp.CS);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int m = 0; m < K; ++m) cur[u][m] = nxt[u][m];
    }
    if (err) set_error(a.ws, err);
}

// Grid-wide barrier of the fixup kernel: one block per SM, co-resident once the main kernel
// it waits for has drained (capi.cu launch_roll; BR_ROLL_FIXUP=cooperative makes the launch
// guarantee it).
// Arrival is a release add on the count, departure an acquire read of the generation: the
// block's writes (ordered before thread 0 by bar.sync, carried by the release's cumulativity)
// are visible to every block that leaves.  The last arriver resets the count and bumps the
// generation with release semantics.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_barrier(RollWs *ws) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire_u32(&ws->bar_gen);
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(&ws->bar_count) : "memory");
        if (old == gridDim.x - 1) {
            ws->bar_count = 0;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&ws->bar_gen) : "memory");
        } else {
            while (ld_acquire_u32(&ws->bar_gen) == g) {
            }
        }
    }
    __syncthreads();
}

template <int K, bool CHA>
__device__ __forceinline__ void roll_fixup_body(const RollArgs &a, uint64_t *win) {
    RollWs *ws = a.ws;
    volatile RollWs *vws = ws;
    const u128 s0 = mk128(a.state[0], a.state[1]);
    const u128 inc = mk128(a.state[2], a.state[3]);
    const bool lh = is_lehmer(inc);
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    if (vws->error) {  // invalid bases: leave the source untouched (reference raises first)
        __syncthreads();
        if (leader) { ws->neg_first = 0; ws->extra = 0; }
        return;
    }
    // One grid barrier per resolved rejection.  Iteration i: every block re-draws the rejected
    // batch itself (same words, same answer; block 0 writes it), re-rolls the tail front first
    // recording the next rejection in q[i % 3], and meets the others at the barrier.  q[(i+1) % 3]
    // is cleared during iteration i: every block read it (as q[(i-2) % 3]) before barrier i-1.
    __shared__ unsigned long long sh_D;
    __shared__ u128 sh_base;
    unsigned long long nf = vws->neg_first;
    uint64_t D = 0;
    int it = 0;
    FrontPlan<CHA, K> fp;
    u128 base = s0;  // PCG64 / Lehmer: the state whose output is word cur + 1 + D
    int64_t cur = 0;
    if (nf != 0) {
        fp = front_plan<CHA, K>(inc, lh);
        cur = (int64_t)(~nf);
        if (threadIdx.x == 0) {
            // the main pass's first rejection: batch `cur` rejected word cur + D; every block
            // re-draws it itself from the next words until accepted (batched.py:120-122), block 0
            // writes it
            uint64_t widx = (uint64_t)cur + 1;
            u128 st = CHA ? cha_add(s0, widx + 1) : gen_jump(s0, inc, widx + 1, lh);
            uint32_t bb[K];
            load_bounds<K>(a.bounds + cur * K, bb);
            uint64_t extra = 1;
            ChaKey ck;
            ChaCursor cc;
            cc.valid = false;
            if constexpr (CHA) ck = cha_key_of_state(a.state);
            for (;;) {
                uint32_t d[K];
                uint64_t r;
                uint8_t tc;
                int err = 0;
                const uint64_t w = CHA ? cha_out_cached(ck, cc, st) : gen_out(st, lh);
                if (eval_batch<K>(bb, w, d, r, tc, err, a.naive != 0) != 1) {
                    if (blockIdx.x == 0) {
                        store_rolls<K>(a.rolls + cur * K, d);
                        a.words[cur] = (uint8_t)(1 + extra > 255 ? 255 : 1 + extra);
                        if (a.flags) a.flags[cur] = 1;
                        if (a.rk) a.rk[cur] = r;
                    }
                    break;
                }
                ++extra;
                st = CHA ? cha_add(st, 1) : mad128(st, gen_mult(lh), inc);
            }
            sh_D = extra;
            if constexpr (!CHA) sh_base = mad128(st, gen_mult(lh), inc);
        }
        __syncthreads();
        D = sh_D;
        base = sh_base;
    }
    // One grid barrier per resolved rejection.  Iteration i re-rolls the tail after `cur` front
    // first; the lane that meets the next rejection re-draws it (roll_front) and records it in
    // q[i % 3] and its warp's rec[i % 2].  q[(i+1) % 3] is cleared during iteration i: every
    // block read it (as q[(i-2) % 3]) before barrier i-1; rec[i % 2] is rewritten in iteration
    // i+2, after every block has read it and reached barrier i+1.
    constexpr int64_t CHK = FrontPlan<CHA, K>::CHK;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
#ifdef BR_FIXUP_PROF
    uint64_t t_front = 0, t_bar = 0, t_post = 0, t0 = 0, t1 = 0;
#define BR_PROF_T(x) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(x))
#else
#define BR_PROF_T(x)
#endif
    while (nf != 0) {
        if (leader) ws->q[(it + 1) % 3] = 0;
        BR_PROF_T(t0);
        roll_front<K, CHA>(a, s0, inc, base, fp, lh, cur + 1, a.nb, D, &ws->q[it % 3], ws->rec[it & 1], win);
        __syncthreads();
        BR_PROF_T(t1);
#ifdef BR_FIXUP_PROF
        t_front += t1 - t0;
#endif
        grid_barrier(ws);
        BR_PROF_T(t0);
#ifdef BR_FIXUP_PROF
        t_bar += t0 - t1;
#endif
        nf = vws->q[it % 3];
        if (nf != 0) {
            const int64_t nxt = (int64_t)(~nf);
            const int64_t w = ((nxt - (cur + 1)) / CHK) % nwarps;  // the warp whose round held it
            const volatile RollWs::Rec *r = &vws->rec[it & 1][w];
            D += r->extra;
            base = mk128(r->hi, r->lo);
            cur = nxt;
        }
        BR_PROF_T(t1);
#ifdef BR_FIXUP_PROF
        t_post += t1 - t0;
#endif
        ++it;
    }
#ifdef BR_FIXUP_PROF
    if (leader) {
        ws->prof[0] = t_front;
        ws->prof[1] = t_bar;
        ws->prof[2] = t_post;
        ws->prof[3] = it;
    }
#endif
#undef BR_PROF_T
    // every block has passed barrier it-1, so it read the initial neg_first and q[(it-2) % 3];
    // q[(it-1) % 3] is 0 (the loop ended on it) and q[it % 3] was cleared in iteration it-1
    if (leader && it > 0) {
        ws->neg_first = 0;
        ws->q[(it + 1) % 3] = 0;
    }
    if (leader) {
        if (D == 0) {
            a.state[0] = vws->final_hi;
            a.state[1] = vws->final_lo;
        } else {
            const u128 sf = CHA ? cha_add(s0, (uint64_t)a.nb + D) : gen_jump(s0, inc, (uint64_t)a.nb + D, lh);
            a.state[0] = sf.hi;
            a.state[1] = sf.lo;
        }
        ws->extra = D;
    }
}

template <int K>
__global__ void __launch_bounds__(256) roll_fixup_kernel(RollArgs a) {
    pdl_wait();
    __shared__ __align__(16) uint64_t win[8][256];
    const bool done = ((volatile RollWs *)a.ws)->main_done != 0;
    if (roll_is_chacha(a)) {
        uint64_t *w = win[(threadIdx.x >> 5) & 7];
        if (!done) {
            roll_cha_main<K>(a, w);
            grid_barrier(a.ws);
        }
        roll_fixup_body<K, true>(a, w);
    } else {
        if (!done) {  // the main kernel was the ChaCha one: roll the PCG64/Lehmer stream here
            const u128 s0 = mk128(a.state[0], a.state[1]), inc = mk128(a.state[2], a.state[3]);
            publish_final(a, s0, inc);
            roll_range<K, 1>(a, s0, inc, 0, a.nb);
            grid_barrier(a.ws);
        }
        roll_fixup_body<K, false>(a, nullptr);
    }
}

}  // namespace br
