// chacha.cuh -- device ChaCha20 keystream words (wordsource.py:92-164).
//
// ChaChaSource emits the 64-bit words of the keystream: word q of block c is
// u32[2q] | u32[2q+1] << 32 of chacha_block(key, c, nonce) (64-bit counter in state words
// 12-13, 64-bit nonce in 14-15, 20 rounds).  The stream is counter based, so the "state"
// the kernels carry is a position, and every jump-ahead is an addition:
//
//   state s = number of words drawn so far (mod 2^67); the word a post-update state
//   outputs is keystream[s - 1]  -- the same post-update convention as gen_out for
//   PCG64/Lehmer, so the lane/jump bookkeeping of every kernel is unchanged
//   (jump by d = s + d, the 32-step advance is s*1 + 32).
//
// The key and nonce (derived from a seed by splitmix64, wordsource.py:147-153, or handed
// over in a br_chacha state) ride in registers (ChaKey).  Consumers:
//   * sequential ones (one thread walks consecutive words) keep the last block in
//     registers (ChaCursor): one block computation per 8 words;
//   * warp/CTA generation steps, where lane L needs word P+L, share a shared-memory window
//     of 8T words filled by T threads computing one block each (cha_fill), refilled when
//     the step's 32..256 words run past it, i.e. once every ~8 steps.
#pragma once
#include "core.cuh"

namespace br {

// inc.lo == 2 marks a ChaCha stream (PCG64 increments are odd, Lehmer's is 0); inc.hi is
// the nonce.  The 8 key words follow the 32-byte head of a device/host state (br_chacha).
static constexpr uint64_t CHACHA_TAG = 2;
// A replayed word sequence (wordsource.py:191-207 FixedSequenceSource, 64-bit words) is the
// same kind of position-addressed stream: word p is words[p] of a device array (inc.hi =
// its length, the first key slot = its address).  Words past the end read as 2^64 - 1, which
// every batch accepts (its final remainder is 2^64 - prod >= 2^64 mod prod), so a call that
// over-reads still terminates; the host then raises SourceExhausted from the position the
// call ended at.
static constexpr uint64_t WORDS_TAG = 4;

struct ChaKey {
    uint32_t k[8];
    uint64_t nonce;
    const uint64_t *words;  // non-null: replayed words instead of the ChaCha block function
    uint64_t nwords;
};

__host__ __device__ __forceinline__ bool is_chacha(u128 inc) { return inc.lo == CHACHA_TAG; }
// position-addressed streams: ChaCha keystreams and replayed word sequences
__host__ __device__ __forceinline__ bool is_posgen(u128 inc) {
    return inc.lo == CHACHA_TAG || inc.lo == WORDS_TAG;
}

__host__ __device__ __forceinline__ uint32_t rotl32(uint32_t v, int r) {
#ifdef __CUDA_ARCH__
    return __funnelshift_l(v, v, r);
#else
    return (v << r) | (v >> (32 - r));
#endif
}

#define BR_CHA_QR(a, b, c, d)  \
    a += b;                    \
    d = rotl32(d ^ a, 16);     \
    c += d;                    \
    b = rotl32(b ^ c, 12);     \
    a += b;                    \
    d = rotl32(d ^ a, 8);      \
    c += d;                    \
    b = rotl32(b ^ c, 7);

// wordsource.py:102-133 chacha_block (RFC 8439 block function, 64/64 counter/nonce split)
__host__ __device__ __forceinline__ void chacha_block(const ChaKey &K, uint64_t ctr, uint32_t out[16]) {
    uint32_t x0 = 0x61707865u, x1 = 0x3320646Eu, x2 = 0x79622D32u, x3 = 0x6B206574u;
    uint32_t x4 = K.k[0], x5 = K.k[1], x6 = K.k[2], x7 = K.k[3];
    uint32_t x8 = K.k[4], x9 = K.k[5], x10 = K.k[6], x11 = K.k[7];
    uint32_t x12 = (uint32_t)ctr, x13 = (uint32_t)(ctr >> 32);
    uint32_t x14 = (uint32_t)K.nonce, x15 = (uint32_t)(K.nonce >> 32);
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int r = 0; r < 10; ++r) {
        BR_CHA_QR(x0, x4, x8, x12)
        BR_CHA_QR(x1, x5, x9, x13)
        BR_CHA_QR(x2, x6, x10, x14)
        BR_CHA_QR(x3, x7, x11, x15)
        BR_CHA_QR(x0, x5, x10, x15)
        BR_CHA_QR(x1, x6, x11, x12)
        BR_CHA_QR(x2, x7, x8, x13)
        BR_CHA_QR(x3, x4, x9, x14)
    }
    out[0] = x0 + 0x61707865u;
    out[1] = x1 + 0x3320646Eu;
    out[2] = x2 + 0x79622D32u;
    out[3] = x3 + 0x6B206574u;
    out[4] = x4 + K.k[0];
    out[5] = x5 + K.k[1];
    out[6] = x6 + K.k[2];
    out[7] = x7 + K.k[3];
    out[8] = x8 + K.k[4];
    out[9] = x9 + K.k[5];
    out[10] = x10 + K.k[6];
    out[11] = x11 + K.k[7];
    out[12] = x12 + (uint32_t)ctr;
    out[13] = x13 + (uint32_t)(ctr >> 32);
    out[14] = x14 + (uint32_t)K.nonce;
    out[15] = x15 + (uint32_t)(K.nonce >> 32);
}

// wordsource.py:147-153 ChaChaSource.__init__: four splitmix64 outputs are the key (low
// half first), the fifth the nonce; counter 0 and an empty buffer = position 0.
__host__ __device__ __forceinline__ void chacha_seed(uint64_t seed, ChaKey &K) {
    uint64_t x = seed;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint64_t c = splitmix64_next(x);
        K.k[2 * i] = (uint32_t)c;
        K.k[2 * i + 1] = (uint32_t)(c >> 32);
    }
    K.nonce = splitmix64_next(x);
    K.words = nullptr;
    K.nwords = 0;
}

// the 8 words of block `blk` of either kind of position-addressed stream
__host__ __device__ __forceinline__ void cha_block_any(const ChaKey &K, uint64_t blk, uint32_t out[16]) {
    if (K.words) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint64_t idx = blk * 8 + q;
#ifdef __CUDA_ARCH__
            const uint64_t w = idx < K.nwords ? __ldg(K.words + idx) : ~0ull;
#else
            const uint64_t w = 0;  // host code never reads device words directly
#endif
            out[2 * q] = (uint32_t)w;
            out[2 * q + 1] = (uint32_t)(w >> 32);
        }
    } else {
        chacha_block(K, blk, out);
    }
}

// block counter of word position p: (p >> 3) mod 2^64 (the counter wraps like the
// reference's `& MASK64`, wordsource.py:160)
__host__ __device__ __forceinline__ uint64_t cha_block_of(u128 p) { return (p.hi << 61) | (p.lo >> 3); }

// word q (0..7) of a block held in registers, without dynamic register indexing
__host__ __device__ __forceinline__ uint64_t cha_pick(const uint32_t b[16], uint32_t q) {
    uint32_t lo = b[0], hi = b[1];
#pragma unroll
    for (int i = 1; i < 8; ++i) {
        if (q == (uint32_t)i) {
            lo = b[2 * i];
            hi = b[2 * i + 1];
        }
    }
    return ((uint64_t)hi << 32) | lo;
}

__host__ __device__ __forceinline__ u128 cha_prev(u128 s) {  // s - 1 mod 2^128
    u128 r;
    r.lo = s.lo - 1;
    r.hi = s.hi - (s.lo == 0 ? 1u : 0u);
    return r;
}

__host__ __device__ __forceinline__ u128 cha_add(u128 s, uint64_t d) {
    u128 r;
    r.lo = s.lo + d;
    r.hi = s.hi + (r.lo < s.lo ? 1u : 0u);
    return r;
}

// word output by post-update state s (keystream[s-1]): one full block, for rare/one-off use
__host__ __device__ __forceinline__ uint64_t cha_out(const ChaKey &K, u128 s) {
    const u128 p = cha_prev(s);
    uint32_t b[16];
    cha_block_any(K, cha_block_of(p), b);
    return cha_pick(b, (uint32_t)(p.lo & 7));
}

// sequential consumer: the last block stays in registers
struct ChaCursor {
    uint32_t b[16];
    uint64_t blk;
    bool valid;
};

__host__ __device__ __forceinline__ uint64_t cha_out_cached(const ChaKey &K, ChaCursor &c, u128 s) {
    const u128 p = cha_prev(s);
    const uint64_t blk = cha_block_of(p);
    if (!c.valid || blk != c.blk) {
        cha_block_any(K, blk, c.b);
        c.blk = blk;
        c.valid = true;
    }
    return cha_pick(c.b, (uint32_t)(p.lo & 7));
}

#ifdef __CUDACC__
// ---- shared-memory keystream window: T threads fill 8T words [W0, W0 + 8T), W0 % 8 == 0.
// Thread t computes block W0/8 + t and stores its 4 16-byte chunks swizzled
// (chunk c -> c ^ ((t >> 1) & 3)) so that the 16-byte stores of 8 neighbouring threads hit
// 8 distinct bank groups.
__device__ __forceinline__ uint32_t cha_win_index(uint32_t i) {  // logical word -> u64 slot
    const uint32_t t = i >> 3, c = (i >> 1) & 3;
    return (t << 3) | ((c ^ ((t >> 1) & 3)) << 1) | (i & 1);
}

__device__ __forceinline__ void cha_fill(uint64_t *win, const ChaKey &K, u128 W0, uint32_t t) {
    uint32_t b[16];
    cha_block_any(K, cha_block_of(W0) + t, b);
    uint4 *dst = reinterpret_cast<uint4 *>(win + 8 * t);
    const uint32_t sw = (t >> 1) & 3;
    dst[0 ^ sw] = make_uint4(b[0], b[1], b[2], b[3]);
    dst[1 ^ sw] = make_uint4(b[4], b[5], b[6], b[7]);
    dst[2 ^ sw] = make_uint4(b[8], b[9], b[10], b[11]);
    dst[3 ^ sw] = make_uint4(b[12], b[13], b[14], b[15]);
}

__device__ __forceinline__ uint64_t cha_win_word(const uint64_t *win, uint32_t rel) {
    return win[cha_win_index(rel)];
}

__device__ __forceinline__ u128 cha_sub(u128 s, uint32_t d) {
    u128 r;
    r.lo = s.lo - d;
    r.hi = s.hi - (s.lo < d ? 1u : 0u);
    return r;
}

// an initial window origin that forces a fill on first use (P - W0 wraps to a huge value)
__device__ __forceinline__ u128 cha_win_unset(u128 p) { return mk128(p.hi, p.lo + (1ull << 20)); }

// Warp form: lane `lane` wants word position p, where p - lane is the same for the whole
// warp.  Window = 256 words per warp; refilled (warp-uniform decision) when the warp's 32
// words run past it.
__device__ __forceinline__ uint64_t cha_warp_word(uint64_t *win, const ChaKey &K, u128 &W0, u128 p, uint32_t lane) {
    const u128 P = cha_sub(p, lane);
    if (P.lo - W0.lo > 256 - 32) {
        __syncwarp();
        W0 = mk128(P.hi, P.lo & ~7ull);
        cha_fill(win, K, W0, lane);
        __syncwarp();
    }
    return cha_win_word(win, (uint32_t)(p.lo - W0.lo));
}

// CTA form: thread L of G wants word p, p - L uniform over the CTA; window = 8G words.
template <int G>
__device__ __forceinline__ uint64_t cha_cta_word(uint64_t *win, const ChaKey &K, u128 &W0, u128 p, uint32_t L) {
    const u128 P = cha_sub(p, L);
    if (P.lo - W0.lo > 8 * G - G) {
        __syncthreads();
        W0 = mk128(P.hi, P.lo & ~7ull);
        cha_fill(win, K, W0, L);
        __syncthreads();
    }
    return cha_win_word(win, (uint32_t)(p.lo - W0.lo));
}

// key of a device stream state (state[0..3] = br_pcg64 head, state[4..7] = key words)
__device__ __forceinline__ ChaKey cha_key_of_state(const uint64_t *state) {
    ChaKey K;
    K.words = state[3] == WORDS_TAG ? reinterpret_cast<const uint64_t *>(state[4]) : nullptr;
    K.nwords = state[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint64_t w = state[4 + i];
        K.k[2 * i] = (uint32_t)w;
        K.k[2 * i + 1] = (uint32_t)(w >> 32);
    }
    K.nonce = state[2];
    return K;
}
#endif

}  // namespace br
