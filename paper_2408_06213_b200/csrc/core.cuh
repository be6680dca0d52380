// core.cuh -- 128-bit arithmetic, device PCG64 and the Theorem-1 digit step.
//
// Reference semantics:
//   PCG64 (XSL-RR 128/64, output of the post-update state)  wordsource.py:71-89
//   splitmix64 seeding                                       wordsource.py:22-35, 80-83
//   one die of the digit chain (a_i, r_i) = b_i (x) r_{i-1}  batched.py:69-82
//
// sm_100a has no 64-bit multiplier: every 64-bit product is built from 32x32->64
// IMAD.WIDE.U32 partial products.  A die with a bound < 2^32 costs two of them, a PCG
// step (multiply by a 128-bit constant) about ten.  Everything here is plain integer
// CUDA; no tensor cores (there is no dense contraction on this path).
#pragma once
#include <stdint.h>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

namespace br {

struct u128 {
    uint64_t lo, hi;
};

__host__ __device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) {
    u128 r;
    r.lo = lo;
    r.hi = hi;
    return r;
}

__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// a*b mod 2^128
__host__ __device__ __forceinline__ u128 mul128(u128 a, u128 b) {
    u128 r;
    r.lo = a.lo * b.lo;
    r.hi = mulhi64(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
    return r;
}

__host__ __device__ __forceinline__ u128 add128(u128 a, u128 b) {
    u128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1u : 0u);
    return r;
}

// s*a + c mod 2^128.  On the device: a hand-written multiply-add carry chain over 32-bit
// limbs (16 PTX mad.lo/hi.cc, 25 SASS instructions).
__host__ __device__ __forceinline__ u128 mad128(u128 s, u128 a, u128 c) {
#ifdef __CUDA_ARCH__
    const uint32_t s0 = (uint32_t)s.lo, s1 = (uint32_t)(s.lo >> 32), s2 = (uint32_t)s.hi, s3 = (uint32_t)(s.hi >> 32);
    const uint32_t a0 = (uint32_t)a.lo, a1 = (uint32_t)(a.lo >> 32), a2 = (uint32_t)a.hi, a3 = (uint32_t)(a.hi >> 32);
    const uint32_t c0 = (uint32_t)c.lo, c1 = (uint32_t)(c.lo >> 32), c2 = (uint32_t)c.hi, c3 = (uint32_t)(c.hi >> 32);
    uint32_t r0, r1, r2, r3;
    asm("mad.lo.cc.u32 %0, %4, %8, %12;\n\t"
        "madc.lo.cc.u32 %1, %4, %9, %13;\n\t"
        "madc.lo.cc.u32 %2, %4, %10, %14;\n\t"
        "madc.lo.u32 %3, %4, %11, %15;\n\t"
        "mad.hi.cc.u32 %1, %4, %8, %1;\n\t"
        "madc.hi.cc.u32 %2, %4, %9, %2;\n\t"
        "madc.hi.u32 %3, %4, %10, %3;\n\t"
        "mad.lo.cc.u32 %1, %5, %8, %1;\n\t"
        "madc.lo.cc.u32 %2, %5, %9, %2;\n\t"
        "madc.lo.u32 %3, %5, %10, %3;\n\t"
        "mad.hi.cc.u32 %2, %5, %8, %2;\n\t"
        "madc.hi.u32 %3, %5, %9, %3;\n\t"
        "mad.lo.cc.u32 %2, %6, %8, %2;\n\t"
        "madc.lo.u32 %3, %6, %9, %3;\n\t"
        "mad.hi.u32 %3, %6, %8, %3;\n\t"
        "mad.lo.u32 %3, %7, %8, %3;"
        : "=&r"(r0), "=&r"(r1), "=&r"(r2), "=&r"(r3)
        : "r"(s0), "r"(s1), "r"(s2), "r"(s3), "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(c0), "r"(c1), "r"(c2),
          "r"(c3));
    u128 r;
    r.lo = ((uint64_t)r1 << 32) | r0;
    r.hi = ((uint64_t)r3 << 32) | r2;
    return r;
#else
    return add128(mul128(s, a), c);
#endif
}

// s*a + c mod 2^128 through unsigned __int128: nvcc emits 6 IMAD.WIDE.U32 (+1 .X) for the
// partial products and ~10 adds, 17 SASS instructions per step against 25 for mad128's
// chain.  Faster where the generator step is the bound (k = 1 and k >= 3 bulk rolls: 15% and
// 5%); at C2's register budget it spills and costs 2-4%, so mad128 stays the default.
__host__ __device__ __forceinline__ u128 mad128_wide(u128 s, u128 a, u128 c) {
    const unsigned __int128 x = ((unsigned __int128)s.hi << 64) | s.lo;
    const unsigned __int128 m = ((unsigned __int128)a.hi << 64) | a.lo;
    const unsigned __int128 d = ((unsigned __int128)c.hi << 64) | c.lo;
    const unsigned __int128 y = x * m + d;
    u128 r;
    r.lo = (uint64_t)y;
    r.hi = (uint64_t)(y >> 64);
    return r;
}

// s <- A*s + C
__host__ __device__ __forceinline__ u128 affine(u128 s, u128 A, u128 C) { return mad128(s, A, C); }

// PCG_MULTIPLIER, wordsource.py:19
static constexpr uint64_t PCG_MULT_HI = 0x2360ED051FC65DA4ull;
static constexpr uint64_t PCG_MULT_LO = 0x4385DF649FCCF645ull;
// LEHMER_MULTIPLIER, wordsource.py:18 (128-bit multiplicative generator, output = top 64 bits)
static constexpr uint64_t LEHMER_MULT = 0xDA942042E4DD58B5ull;

// XSL-RR output of a (post-update) state, wordsource.py:87-89
__host__ __device__ __forceinline__ uint64_t xslrr(u128 s) {
#ifdef __CUDA_ARCH__
    // rotate right by the top 6 bits with two funnel shifts (swap halves for rot >= 32)
    const uint32_t xl = (uint32_t)s.hi ^ (uint32_t)s.lo, xh = (uint32_t)(s.hi >> 32) ^ (uint32_t)(s.lo >> 32);
    const uint32_t rot = (uint32_t)(s.hi >> 58);
    const bool sw = rot & 32u;
    const uint32_t a = sw ? xh : xl, b = sw ? xl : xh;
    return ((uint64_t)__funnelshift_r(b, a, rot) << 32) | __funnelshift_r(a, b, rot);
#else
    uint64_t x = s.hi ^ s.lo;
    unsigned rot = (unsigned)(s.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
#endif
}

__host__ __device__ __forceinline__ uint64_t splitmix64_next(uint64_t &x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Pcg64Source.__init__ (wordsource.py:80-83)
__host__ __device__ __forceinline__ void pcg_seed(uint64_t seed, u128 &state, u128 &inc) {
    uint64_t x = seed;
    uint64_t z0 = splitmix64_next(x), z1 = splitmix64_next(x);
    uint64_t z2 = splitmix64_next(x), z3 = splitmix64_next(x);
    state = mk128(z0, z1);
    inc = mk128(z2, z3 | 1u);
}

// LehmerSource.__init__ (wordsource.py:61-63); the increment is 0, which is how a Lehmer
// stream is told apart from a PCG64 stream (whose increment is always odd)
__host__ __device__ __forceinline__ void lehmer_seed(uint64_t seed, u128 &state, u128 &inc) {
    uint64_t x = seed;
    uint64_t z0 = splitmix64_next(x), z1 = splitmix64_next(x);
    state = mk128(z0, z1 | 1u);
    inc = mk128(0, 0);
}

// per-array seed convention: first splitmix64 output of (s<<32)|a
__host__ __device__ __forceinline__ uint64_t array_seed(uint64_t run_seed, uint64_t a) {
    uint64_t x = (run_seed << 32) | a;
    return splitmix64_next(x);
}

// One die: (digit, r') = b (x) r for b < 2^32.  Two IMAD.WIDE.U32 partial products.
// The carry of b*r_lo is absorbed as the 64-bit addend of the second IMAD.WIDE:
// b*r_hi + (b*r_lo >> 32) < 2^64, so (digit, r') = (p1 >> 32, p1_lo : p0_lo).
__host__ __device__ __forceinline__ uint32_t die(uint32_t b, uint64_t &r) {
    const uint64_t p0 = (uint64_t)b * (uint32_t)r;
    const uint64_t p1 = (uint64_t)b * (uint32_t)(r >> 32) + (p0 >> 32);
    r = (p1 << 32) | (uint32_t)p0;
    return (uint32_t)(p1 >> 32);
}

// 2^64 mod b for 1 <= b < 2^64 (bounded.py:59-62); b == 0 encodes 2^64 -> 0
__host__ __device__ __forceinline__ uint64_t threshold64(uint64_t b) { return b ? (0 - b) % b : 0; }

// Jump tables: A_d = M^d, G_d = sum_{i<d} M^i so that state_{t+d} = A_d*state_t + G_d*inc.
// The direct tables cover every lane offset of a CTA (up to 1024 threads).
static constexpr int JUMP_SMALL = 1024;
struct JumpTables {
    u128 A[64], G[64];       // d = 2^k
    u128 SA[JUMP_SMALL + 1], SG[JUMP_SMALL + 1];  // d = 0..JUMP_SMALL (lane offsets, realignments)
    u128 LA[64], LSA[JUMP_SMALL + 1];             // Lehmer: multiplier powers M_L^(2^k), M_L^d
};

// Host construction (also used by the C-ABI host helpers)
inline void build_jump_tables(JumpTables &t) {
    u128 m = mk128(PCG_MULT_HI, PCG_MULT_LO);
    u128 g = mk128(0, 1);
    for (int k = 0; k < 64; ++k) {
        t.A[k] = m;
        t.G[k] = g;
        // (A,G)_{2d} = (A^2, (A+1) G)
        g = mul128(add128(m, mk128(0, 1)), g);
        m = mul128(m, m);
    }
    u128 lm = mk128(0, LEHMER_MULT);
    for (int k = 0; k < 64; ++k) {
        t.LA[k] = lm;
        lm = mul128(lm, lm);
    }
    u128 la = mk128(0, 1);
    for (int d = 0; d <= JUMP_SMALL; ++d) {
        t.LSA[d] = la;
        la = mul128(mk128(0, LEHMER_MULT), la);
    }
    u128 a = mk128(0, 1), gg = mk128(0, 0);
    u128 M = mk128(PCG_MULT_HI, PCG_MULT_LO);
    for (int d = 0; d <= JUMP_SMALL; ++d) {
        t.SA[d] = a;
        t.SG[d] = gg;
        gg = add128(mul128(M, gg), mk128(0, 1));  // G_{d+1} = M*G_d + 1
        a = mul128(M, a);
    }
}

}  // namespace br
