// jump.cuh -- device jump-ahead for PCG64 streams.
//
// A stream is parallelised by giving each lane its own word offset: the state after
// d more words is A_d*s + G_d*inc (LCG jump-ahead; checked against numpy's PCG64.advance
// and against stepping in tests/test_oracle.py and tests/test_gpu_*.py).
//   c_A/c_G : d = 2^k, read with warp-uniform k      -> __constant__ (broadcast)
//   g_SA/g_SG: d = 0..JUMP_SMALL (1024), per-lane d    -> global (L1-cached)
#pragma once
#include "core.cuh"

namespace br {

__constant__ u128 c_A[64];
__constant__ u128 c_G[64];
__constant__ u128 c_LA[64];
__device__ u128 g_SA[JUMP_SMALL + 1];
__device__ u128 g_SG[JUMP_SMALL + 1];
__device__ u128 g_LSA[JUMP_SMALL + 1];

// state after d more updates (any d; cost popcount(d) affine steps)
__device__ __forceinline__ u128 jump(u128 s, u128 inc, uint64_t d) {
    int k = 0;
    while (d) {
        if (d & 1) s = mad128(s, c_A[k], mul128(c_G[k], inc));
        d >>= 1;
        ++k;
    }
    return s;
}

// state after d (0..JUMP_SMALL) more updates; d may differ per lane
__device__ __forceinline__ u128 jump_small(u128 s, u128 inc, int d) {
    u128 A = g_SA[d], G = g_SG[d];
    return mad128(s, A, mul128(G, inc));
}

// one PCG64 update + output (wordsource.py:85-89)
__device__ __forceinline__ uint64_t pcg_next(u128 &s, u128 inc) {
    s = mad128(s, mk128(PCG_MULT_HI, PCG_MULT_LO), inc);
    return xslrr(s);
}

}  // namespace br

namespace br {
// ---- generator-generic forms: `lh` selects Lehmer128 (increment 0) instead of PCG64.
// Every additive term carries the increment, so for Lehmer it vanishes and only the
// multiplier tables differ.
__device__ __forceinline__ bool is_lehmer(u128 inc) { return (inc.hi | inc.lo) == 0; }

__device__ __forceinline__ u128 gen_mult(bool lh) {
    return lh ? mk128(0, LEHMER_MULT) : mk128(PCG_MULT_HI, PCG_MULT_LO);
}

// output of a post-update state: XSL-RR (wordsource.py:87-89) or the top 64 bits (:65-67)
__device__ __forceinline__ uint64_t gen_out(u128 s, bool lh) { return lh ? s.hi : xslrr(s); }

__device__ __forceinline__ uint64_t gen_next(u128 &s, u128 inc, bool lh) {
    s = mad128(s, gen_mult(lh), inc);
    return gen_out(s, lh);
}

__device__ __forceinline__ u128 gen_jump(u128 s, u128 inc, uint64_t d, bool lh) {
    int k = 0;
    while (d) {
        if (d & 1) s = mad128(s, lh ? c_LA[k] : c_A[k], mul128(c_G[k], inc));
        d >>= 1;
        ++k;
    }
    return s;
}

// the affine map of a d-word jump: state' = A * state + C
__device__ __forceinline__ void gen_affine(uint64_t d, u128 inc, bool lh, u128 &A, u128 &C) {
    u128 a = mk128(0, 1), g = mk128(0, 0);
    int k = 0;
    while (d) {
        if (d & 1) {
            const u128 Ak = lh ? c_LA[k] : c_A[k];
            a = mul128(a, Ak);
            g = mad128(g, Ak, c_G[k]);
        }
        d >>= 1;
        ++k;
    }
    A = a;
    C = mul128(g, inc);
}

__device__ __forceinline__ u128 gen_jump_small(u128 s, u128 inc, int d, bool lh) {
    return mad128(s, lh ? g_LSA[d] : g_SA[d], mul128(g_SG[d], inc));
}

__device__ __forceinline__ u128 gen_SA(bool lh, int d) { return lh ? g_LSA[d] : g_SA[d]; }

__device__ __forceinline__ void gen_seed(uint64_t seed, u128 &s, u128 &inc, bool lh) {
    if (lh) lehmer_seed(seed, s, inc);
    else pcg_seed(seed, s, inc);
}
}  // namespace br
