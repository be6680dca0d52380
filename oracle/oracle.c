/*
 * oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * Checker for the CUDA product; see oracle.h for the rules.  Each function follows the
 * cited reference code (paths relative to /root/reference/pkg/src/batchrand/) literally,
 * including the carried upper bound `u` of _run_batches, so that the simplifications the
 * GPU kernels make (per-batch exact thresholds, SURVEY finding 3) are checked against the
 * reference's own control flow rather than assumed.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

#define MASK64 0xFFFFFFFFFFFFFFFFull
/* wordsource.py:18-19 */
static const u128 LEHMER_MULT = (u128)0xDA942042E4DD58B5ull;
#define PCG_MULT_HI 0x2360ED051FC65DA4ull
#define PCG_MULT_LO 0x4385DF649FCCF645ull

static inline u128 mk(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }
static inline u128 mask_of(int bits) { return bits >= 64 ? (u128)MASK64 : (((u128)1 << bits) - 1); }

/* wordsource.py:22-35 splitmix64_stream (one step) */
uint64_t or_splitmix64_next(uint64_t *x) {
    *x += 0x9E3779B97F4A7C15ull;
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* wordsource.py:80-83 Pcg64Source.__init__ */
void or_source_pcg64(or_source *s, uint64_t seed) {
    memset(s, 0, sizeof(*s));
    s->kind = 0;
    s->word_bits = 64;
    uint64_t x = seed;
    uint64_t z0 = or_splitmix64_next(&x), z1 = or_splitmix64_next(&x);
    uint64_t z2 = or_splitmix64_next(&x), z3 = or_splitmix64_next(&x);
    s->state_hi = z0;
    s->state_lo = z1;
    s->inc_hi = z2;
    s->inc_lo = z3 | 1u;
}

/* wordsource.py:61-63 LehmerSource.__init__ */
void or_source_lehmer(or_source *s, uint64_t seed) {
    memset(s, 0, sizeof(*s));
    s->kind = 2;
    s->word_bits = 64;
    uint64_t x = seed;
    uint64_t z0 = or_splitmix64_next(&x), z1 = or_splitmix64_next(&x);
    s->state_hi = z0;
    s->state_lo = z1 | 1u;
}

/* wordsource.py:194-201 FixedSequenceSource.__init__ */
void or_source_fixed(or_source *s, const uint64_t *words, int64_t n, int32_t bits) {
    memset(s, 0, sizeof(*s));
    s->kind = 1;
    s->word_bits = bits;
    s->words = words;
    s->nwords = n;
}

/* wordsource.py:92-99 round pattern and constants */
static const int CHACHA_IDX[8][4] = {{0, 4, 8, 12}, {1, 5, 9, 13}, {2, 6, 10, 14}, {3, 7, 11, 15},
                                     {0, 5, 10, 15}, {1, 6, 11, 12}, {2, 7, 8, 13}, {3, 4, 9, 14}};
static inline uint32_t rotl32(uint32_t v, int r) { return (v << r) | (v >> (32 - r)); }

/* wordsource.py:102-133 chacha_block */
void or_chacha_block(const uint32_t key[8], uint64_t counter, uint64_t nonce, uint32_t out[16]) {
    uint32_t init[16] = {0x61707865u, 0x3320646Eu, 0x79622D32u, 0x6B206574u};
    for (int i = 0; i < 8; ++i) init[4 + i] = key[i];
    init[12] = (uint32_t)counter;
    init[13] = (uint32_t)(counter >> 32);
    init[14] = (uint32_t)nonce;
    init[15] = (uint32_t)(nonce >> 32);
    uint32_t x[16];
    memcpy(x, init, sizeof x);
    for (int r = 0; r < 10; ++r) {
        for (int q = 0; q < 8; ++q) {
            const int a = CHACHA_IDX[q][0], b = CHACHA_IDX[q][1], c = CHACHA_IDX[q][2], d = CHACHA_IDX[q][3];
            x[a] += x[b]; x[d] = rotl32(x[d] ^ x[a], 16);
            x[c] += x[d]; x[b] = rotl32(x[b] ^ x[c], 12);
            x[a] += x[b]; x[d] = rotl32(x[d] ^ x[a], 8);
            x[c] += x[d]; x[b] = rotl32(x[b] ^ x[c], 7);
        }
    }
    for (int i = 0; i < 16; ++i) out[i] = x[i] + init[i];
}

/* wordsource.py:147-153 ChaChaSource.__init__ */
void or_source_chacha(or_source *s, uint64_t seed) {
    memset(s, 0, sizeof(*s));
    s->kind = 3;
    s->word_bits = 64;
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) {
        uint64_t c = or_splitmix64_next(&x);
        s->key[2 * i] = (uint32_t)c;
        s->key[2 * i + 1] = (uint32_t)(c >> 32);
    }
    s->nonce = or_splitmix64_next(&x);
    s->counter = 0;
    s->pos = 16;
}

/* position arithmetic on the ChaCha source: the next word is word pos/2 of the buffered
 * block counter-1, or word 0 of block `counter` when the buffer is empty.  Skipping delta
 * words lands on block (P + delta) / 8 with the same refill rule as next_word. */
void or_chacha_advance(or_source *s, uint64_t delta) {
    /* absolute word position mod 2^67, as (block, word) */
    uint64_t blk = s->pos == 16 ? s->counter : s->counter - 1;
    uint64_t w = s->pos == 16 ? 0 : (uint64_t)(s->pos / 2);
    uint64_t t = w + (delta & 7);
    blk += (delta >> 3) + (t >> 3);
    w = t & 7;
    if (w == 0) {
        s->counter = blk;
        s->pos = 16;
    } else {
        or_chacha_block(s->key, blk, s->nonce, s->buf);
        s->counter = blk + 1;
        s->pos = (int32_t)(2 * w);
    }
}

int or_next_word(or_source *s, uint64_t *w) {
    if (s->kind == 0) {
        /* wordsource.py:85-89 Pcg64Source.next_word: update, then XSL-RR of the new state */
        u128 st = mk(s->state_hi, s->state_lo) * mk(PCG_MULT_HI, PCG_MULT_LO) +
                  mk(s->inc_hi, s->inc_lo);
        s->state_hi = (uint64_t)(st >> 64);
        s->state_lo = (uint64_t)st;
        unsigned rot = (unsigned)(st >> 122);
        uint64_t x = s->state_hi ^ s->state_lo;
        *w = (x >> rot) | (x << ((64 - rot) & 63));
    } else if (s->kind == 2) {
        /* wordsource.py:65-67 LehmerSource.next_word */
        u128 st = mk(s->state_hi, s->state_lo) * LEHMER_MULT;
        s->state_hi = (uint64_t)(st >> 64);
        s->state_lo = (uint64_t)st;
        *w = s->state_hi;
    } else if (s->kind == 3) {
        /* wordsource.py:155-164 ChaChaSource.next_word */
        if (s->pos == 16) {
            or_chacha_block(s->key, s->counter, s->nonce, s->buf);
            s->counter += 1;
            s->pos = 0;
        }
        *w = (uint64_t)s->buf[s->pos] | ((uint64_t)s->buf[s->pos + 1] << 32);
        s->pos += 2;
    } else {
        /* wordsource.py:202-207 FixedSequenceSource.next_word */
        if (s->cursor >= s->nwords) return OR_E_EXHAUSTED;
        *w = s->words[s->cursor++];
    }
    s->drawn++;
    return OR_OK;
}

/* O(log d) LCG jump-ahead (not in the reference; pinned against numpy PCG64.advance
 * and against stepping, tests/test_oracle.py). */
void or_pcg64_advance(or_source *s, uint64_t delta) {
    u128 acc_m = 1, acc_p = 0, cur_m = mk(PCG_MULT_HI, PCG_MULT_LO), cur_p = mk(s->inc_hi, s->inc_lo);
    while (delta) {
        if (delta & 1) {
            acc_m *= cur_m;
            acc_p = acc_p * cur_m + cur_p;
        }
        cur_p = (cur_m + 1) * cur_p;
        cur_m *= cur_m;
        delta >>= 1;
    }
    u128 st = acc_m * mk(s->state_hi, s->state_lo) + acc_p;
    s->state_hi = (uint64_t)(st >> 64);
    s->state_lo = (uint64_t)st;
}

/* Per-array seed convention: next(splitmix64_stream(((s<<32)|a) & MASK64)). */
uint64_t or_array_seed(uint64_t run_seed, uint64_t array_index) {
    uint64_t x = (run_seed << 32) | array_index;
    return or_splitmix64_next(&x);
}

/* bounded.py:107-119 falling_factorial */
static int ff128(uint64_t n, uint64_t k, int bits, u128 *out) {
    if (k > n) return OR_E_INVALID;
    u128 limit = (u128)1 << bits;
    u128 acc = 1;
    for (uint64_t f = n; f > n - k; --f) {
        /* acc <= 2^64 and f < 2^64: the product fits before the check only if acc*f
         * does not wrap 2^128; acc <= 2^bits <= 2^64 so acc*f < 2^128. */
        acc *= (u128)f;
        if (acc > limit) return OR_E_BOUND_OVERFLOW;
    }
    *out = acc;
    return OR_OK;
}

int or_falling_factorial(uint64_t n, uint64_t k, int32_t bits, uint64_t *lo, uint64_t *hi) {
    u128 v = 0;
    int st = ff128(n, k, bits, &v);
    if (st == OR_OK) {
        *lo = (uint64_t)v;
        *hi = (uint64_t)(v >> 64);
    }
    return st;
}

/* bounded.py:59-62 threshold: 2**bits mod b */
static u128 thresh128(u128 b, int bits) { return (((u128)1 << bits) - b) % b; }
uint64_t or_threshold(uint64_t b_lo, uint64_t b_hi, int32_t bits) {
    return (uint64_t)thresh128(mk(b_hi, b_lo), bits);
}

/* bounded.py:73-104 roll_single_traced */
int or_roll_single(or_source *s, uint64_t b_lo, uint64_t b_hi, uint64_t *value,
                   uint64_t *words, int32_t *remainder_ops) {
    int bits = s->word_bits;
    u128 b = mk(b_hi, b_lo);
    if (b < 1 || b > ((u128)1 << bits)) return OR_E_BOUND_OVERFLOW;
    u128 mask = mask_of(bits);
    uint64_t w;
    if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
    u128 p = b * w;
    u128 lo = p & mask;
    if (lo >= b) {
        *value = (uint64_t)(p >> bits);
        *words = 1;
        *remainder_ops = 0;
        return OR_OK;
    }
    u128 t = ((mask + 1) - b) % b;
    uint64_t nw = 1;
    while (lo < t) {
        if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
        p = b * w;
        lo = p & mask;
        nw++;
    }
    *value = (uint64_t)(p >> bits);
    *words = nw;
    *remainder_ops = 1;
    return OR_OK;
}

/* batched.py:69-82 digit_pass */
static u128 digit_pass128(uint64_t r0, const uint64_t *bases, int k, int bits, uint64_t *digits) {
    u128 mask = mask_of(bits);
    u128 r = r0;
    for (int i = 0; i < k; ++i) {
        u128 p = (u128)bases[i] * r;
        digits[i] = (uint64_t)(p >> bits);
        r = p & mask;
    }
    return r;
}

void or_digit_pass(uint64_t r0, const uint64_t *bases, int32_t k, int32_t bits,
                   uint64_t *digits, uint64_t *rk) {
    *rk = (uint64_t)digit_pass128(r0, bases, k, bits, digits);
}

/* mixed_radix.py:26-34 RadixBases.of validation + product */
static int radix_product(const uint64_t *bases, int k, int bits, u128 *prod) {
    if (k < 1) return OR_E_INVALID;
    for (int i = 0; i < k; ++i)
        if (bases[i] < 1) return OR_E_INVALID;
    u128 limit = (u128)1 << bits;
    u128 acc = 1;
    for (int i = 0; i < k; ++i) {
        /* math.prod then BoundEncoding.of: overflow of the exact product is the error;
         * keep the running product exact until it provably exceeds the limit */
        acc *= bases[i];
        if (acc > limit) {
            /* once above 2**bits with all remaining bases >= 1 the product stays above */
            return OR_E_BOUND_OVERFLOW;
        }
    }
    *prod = acc;
    return OR_OK;
}

/* batched.py:102-123 roll_batch */
int or_roll_batch(or_source *s, const uint64_t *bases, int32_t k, int32_t bits,
                  int32_t has_upper, uint64_t upper_lo, uint64_t upper_hi,
                  uint64_t *digits, uint64_t *words, int32_t *threshold_computed,
                  uint64_t *rk) {
    u128 b;
    int st = radix_product(bases, k, bits, &b);
    if (st) return st;
    uint64_t w;
    if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
    uint64_t nw = 1;
    u128 r = digit_pass128(w, bases, k, bits, digits);
    u128 u = mk(upper_hi, upper_lo);
    if ((has_upper && r >= u) || r >= b) {
        *words = nw;
        *threshold_computed = 0;
        *rk = (uint64_t)r;
        return OR_OK;
    }
    u128 t = (((u128)1 << bits) - b) % b;
    while (r < t) {
        if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
        nw++;
        r = digit_pass128(w, bases, k, bits, digits);
    }
    *words = nw;
    *threshold_computed = 1;
    *rk = (uint64_t)r;
    return OR_OK;
}

/* batched.py:85-99 roll_batch_known_threshold */
int or_roll_batch_known_threshold(or_source *s, const uint64_t *bases, int32_t k,
                                  int32_t bits, uint64_t t, uint64_t *digits,
                                  uint64_t *words, uint64_t *rk) {
    uint64_t nw = 0, w;
    for (;;) {
        if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
        nw++;
        u128 r = digit_pass128(w, bases, k, bits, digits);
        if (r >= t) {
            *words = nw;
            *rk = (uint64_t)r;
            return OR_OK;
        }
    }
}

/* shuffle.py:32-49 ShuffleSchedule.__post_init__ */
int or_schedule_validate(const uint64_t *lengths, const uint32_t *sizes, int32_t nent,
                         int32_t max_batch, int32_t bits) {
    if (nent < 1) return OR_E_INVALID;
    for (int i = 0; i + 1 < nent; ++i) {
        if (lengths[i] <= lengths[i + 1]) return OR_E_INVALID;
        if (sizes[i] >= sizes[i + 1]) return OR_E_INVALID;
    }
    if ((int64_t)sizes[nent - 1] != (int64_t)max_batch) return OR_E_INVALID;
    for (int i = 0; i < nent; ++i) {
        if ((uint64_t)sizes[i] > lengths[i]) return OR_E_INVALID;
        u128 f;
        int st = ff128(lengths[i], sizes[i], bits, &f);
        if (st) return st;
    }
    return OR_OK;
}

static inline void swap_elem(unsigned char *z, int eb, uint64_t i, uint64_t j) {
    if (eb == 4) {
        uint32_t *a = (uint32_t *)z, t = a[i];
        a[i] = a[j];
        a[j] = t;
    } else if (eb == 8) {
        uint64_t *a = (uint64_t *)z, t = a[i];
        a[i] = a[j];
        a[j] = t;
    } else {
        unsigned char tmp[64];
        memcpy(tmp, z + i * eb, eb);
        memcpy(z + i * eb, z + j * eb, eb);
        memcpy(z + j * eb, tmp, eb);
    }
}

/* shuffle.py:80-97 shuffle_unbatched */
int or_shuffle_unbatched(or_source *s, void *zv, int32_t eb, uint64_t n) {
    unsigned char *z = (unsigned char *)zv;
    int bits = s->word_bits;
    u128 mask = mask_of(bits), top = mask + 1;
    uint64_t w;
    for (uint64_t i = n ? n - 1 : 0; i >= 1 && n >= 2; --i) {
        u128 b = (u128)i + 1;
        if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
        u128 p = b * w, lo = p & mask;
        if (lo < b) {
            u128 t = (top - b) % b;
            while (lo < t) {
                if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
                p = b * w;
                lo = p & mask;
            }
        }
        swap_elem(z, eb, i, (uint64_t)(p >> bits));
        if (i == 1) break;
    }
    return OR_OK;
}

/* shuffle.py:228-266 shuffle_naive_batched (literal): pairs by division, then index 1 */
int or_shuffle_naive_batched(or_source *s, void *zv, int32_t eb, uint64_t n) {
    unsigned char *z = (unsigned char *)zv;
    int bits = s->word_bits;
    u128 mask = mask_of(bits), top = mask + 1;
    uint64_t w;
    if (n < 2) return OR_OK;
    uint64_t i = n - 1;
    if (i >= 2 && (u128)(i + 1) * i > top) return OR_E_BOUND_OVERFLOW;
    while (i >= 2) {
        u128 b = (u128)(i + 1) * i;
        if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
        u128 p = b * w, lo = p & mask;
        if (lo < b) {
            u128 t = (top - b) % b;
            while (lo < t) {
                if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
                p = b * w;
                lo = p & mask;
            }
        }
        u128 v = p >> bits;
        uint64_t j1 = (uint64_t)(v / i), j2 = (uint64_t)(v % i);
        swap_elem(z, eb, i, j1);
        i -= 1;
        swap_elem(z, eb, i, j2);
        i -= 1;
    }
    if (i == 1) {
        if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
        u128 p = (u128)2 * w, lo = p & mask;
        if (lo < 2) {
            u128 t = (top - 2) % 2;
            while (lo < t) {
                if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
                p = (u128)2 * w;
                lo = p & mask;
            }
        }
        swap_elem(z, eb, 1, (uint64_t)(p >> bits));
    }
    return OR_OK;
}

/* shuffle.py:100-134 _run_batches (literal, with the carried bound u) */
static int run_batches(or_source *s, unsigned char *z, int eb, uint64_t n, uint32_t k,
                       u128 *u_io, uint64_t count, int bits) {
    u128 mask = mask_of(bits);
    uint64_t js[128];
    u128 u = *u_io;
    uint64_t w;
    if (k > 128) return OR_E_INVALID;
    for (uint64_t c = 0; c < count; ++c) {
        if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
        u128 r = w;
        u128 b = n;
        for (uint32_t i = 0; i < k; ++i) {
            u128 p = b * r;
            js[i] = (uint64_t)(p >> bits);
            r = p & mask;
            b -= 1;
        }
        if (r < u) {
            int st = ff128(n, k, bits, &u);
            if (st) return st;
            u128 t = ((mask + 1) - u) % u;
            while (r < t) {
                if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
                r = w;
                b = n;
                for (uint32_t i = 0; i < k; ++i) {
                    u128 p = b * r;
                    js[i] = (uint64_t)(p >> bits);
                    r = p & mask;
                    b -= 1;
                }
            }
        }
        uint64_t i = n - 1;
        for (uint32_t m = 0; m < k; ++m) {
            swap_elem(z, eb, i, js[m]);
            i -= 1;
        }
        n -= k;
    }
    *u_io = u;
    return OR_OK;
}

/* shuffle.py:137-146 partial_shuffle_batch */
int or_partial_shuffle_batch(or_source *s, void *z, int32_t eb, uint64_t n, uint32_t k,
                             uint64_t u_lo, uint64_t u_hi, uint64_t *u_out_lo,
                             uint64_t *u_out_hi) {
    u128 u = mk(u_hi, u_lo);
    int st = run_batches(s, (unsigned char *)z, eb, n, k, &u, 1, s->word_bits);
    if (st) return st;
    *u_out_lo = (uint64_t)u;
    *u_out_hi = (uint64_t)(u >> 64);
    return OR_OK;
}

/* shuffle.py:149-225 shuffle_batched (literal).  check_bounds: shuffle.py:214-221. */
int or_shuffle_batched(or_source *s, void *zv, int32_t eb, uint64_t n,
                       const uint64_t *lengths, const uint32_t *sizes, int32_t nent,
                       int32_t bits, int32_t check_bounds) {
    unsigned char *z = (unsigned char *)zv;
    if (s->word_bits != bits) return OR_E_INVALID;
    uint64_t remaining = n;
    if (remaining < 2) return OR_OK;
    uint64_t top_length = lengths[0];
    u128 mask = mask_of(bits);
    uint64_t w;
    if (remaining > top_length) {
        u128 topw = mask + 1;
        for (uint64_t i = remaining - 1; i >= top_length; --i) {
            u128 b = (u128)i + 1;
            if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
            u128 p = b * w, lo = p & mask;
            if (lo < b) {
                u128 t = (topw - b) % b;
                while (lo < t) {
                    if (or_next_word(s, &w)) return OR_E_EXHAUSTED;
                    p = b * w;
                    lo = p & mask;
                }
            }
            swap_elem(z, eb, i, (uint64_t)(p >> bits));
            if (i == 0) break;
        }
        remaining = top_length;
    }
    int idx = 0;
    for (int pos = 0; pos < nent; ++pos) {
        if (lengths[pos] >= remaining) idx = pos;
        else break;
    }
    uint32_t k = sizes[idx];
    u128 u;
    int st = ff128(lengths[idx], k, bits, &u);
    if (st) return st;
    while (remaining > 1) {
        if (remaining < k) {
            k = (uint32_t)(remaining - 1);
            u128 uf;
            st = ff128(remaining, k, bits, &uf);
            if (st) return st;
            st = run_batches(s, z, eb, remaining, k, &uf, 1, bits);
            if (st) return st;
            break;
        }
        if (idx + 1 < nent && remaining <= lengths[idx + 1]) {
            idx += 1;
            k = sizes[idx];
            st = ff128(lengths[idx], k, bits, &u);
            if (st) return st;
            continue;
        }
        uint64_t count;
        if (idx + 1 < nent)
            count = (remaining - lengths[idx + 1] + k - 1) / k; /* -((next - rem) // k) */
        else
            count = remaining / k;
        if (check_bounds) {
            for (uint64_t c = 0; c < count; ++c) {
                u128 f;
                st = ff128(remaining, k, bits, &f);
                if (st) return st;
                if (u < f) return 9; /* AssertionError */
                st = run_batches(s, z, eb, remaining, k, &u, 1, bits);
                if (st) return st;
                remaining -= k;
            }
        } else {
            st = run_batches(s, z, eb, remaining, k, &u, count, bits);
            if (st) return st;
            remaining -= count * k;
        }
    }
    return OR_OK;
}

/* Word-free regime walk of shuffle_batched (shuffle.py:168-224). */
int64_t or_shuffle_trace(uint64_t n, const uint64_t *lengths, const uint32_t *sizes,
                         int32_t nent, int32_t bits, uint64_t *batch_n, uint32_t *batch_k,
                         int64_t cap) {
    int64_t nb = 0;
#define EMIT(NN, KK)                      \
    do {                                  \
        if (nb < cap) {                   \
            batch_n[nb] = (NN);           \
            batch_k[nb] = (KK);           \
        }                                 \
        nb++;                             \
    } while (0)
    uint64_t remaining = n;
    if (remaining < 2) return 0;
    uint64_t top_length = lengths[0];
    if (remaining > top_length) {
        for (uint64_t i = remaining - 1; i >= top_length; --i) {
            EMIT(i + 1, 1);
            if (i == 0) break;
        }
        remaining = top_length;
    }
    int idx = 0;
    for (int pos = 0; pos < nent; ++pos) {
        if (lengths[pos] >= remaining) idx = pos;
        else break;
    }
    uint32_t k = sizes[idx];
    (void)bits;
    while (remaining > 1) {
        if (remaining < k) {
            k = (uint32_t)(remaining - 1);
            EMIT(remaining, k);
            break;
        }
        if (idx + 1 < nent && remaining <= lengths[idx + 1]) {
            idx += 1;
            k = sizes[idx];
            continue;
        }
        uint64_t count = (idx + 1 < nent) ? (remaining - lengths[idx + 1] + k - 1) / k
                                          : remaining / k;
        for (uint64_t c = 0; c < count; ++c) {
            EMIT(remaining, k);
            remaining -= k;
        }
    }
#undef EMIT
    return nb;
}

int or_roll_batches(or_source *s, const uint32_t *bounds, int32_t k, int64_t nb,
                    uint32_t *rolls, uint8_t *words, uint8_t *flags, uint64_t *rk) {
    uint64_t bases[64], digits[64];
    if (k < 1 || k > 64) return OR_E_INVALID;
    for (int64_t i = 0; i < nb; ++i) {
        for (int m = 0; m < k; ++m) bases[m] = bounds[i * k + m];
        uint64_t nw, r;
        int32_t tc;
        int st = or_roll_batch(s, bases, k, 64, 0, 0, 0, digits, &nw, &tc, &r);
        if (st) return st;
        for (int m = 0; m < k; ++m) rolls[i * k + m] = (uint32_t)digits[m];
        if (words) words[i] = (uint8_t)(nw > 255 ? 255 : nw);
        if (flags) flags[i] = (uint8_t)tc;
        if (rk) rk[i] = r;
    }
    return OR_OK;
}

/* Bulk rolls on all host threads: the CPU baseline of the bench (not in the reference; the
 * results are or_roll_batches' exactly).  The batch range is split into contiguous chunks and
 * chunk c is rolled from the stream advanced to its first batch, as if no earlier batch had
 * been rejected.  Then, in chunk order, a chunk whose true first word differs (earlier chunks
 * consumed extra words) is rolled again from the right word.  PCG64 and ChaCha sources (O(log)
 * jump-ahead); any other source, or one thread, runs or_roll_batches. */
static void or_source_skip(or_source *s, uint64_t delta) {
    if (s->kind == 3) or_chacha_advance(s, delta);
    else or_pcg64_advance(s, delta);
    s->drawn += (int64_t)delta;
}

int or_roll_batches_mt(or_source *s, const uint32_t *bounds, int32_t k, int64_t nb, uint32_t *rolls,
                       uint8_t *words, uint8_t *flags, uint64_t *rk, int32_t nthreads) {
    int T = 1;
#ifdef _OPENMP
    T = nthreads > 0 ? nthreads : omp_get_max_threads();
#endif
    if ((s->kind != 0 && s->kind != 3) || T <= 1 || nb < (int64_t)T * 4096)
        return or_roll_batches(s, bounds, k, nb, rolls, words, flags, rk);
    if (T > 1024) T = 1024;
    int64_t extra[1024];
    int errs[1024];
    const or_source base = *s;
#ifdef _OPENMP
#pragma omp parallel for schedule(static, 1) num_threads(T)
#endif
    for (int c = 0; c < T; ++c) {
        const int64_t lo = nb * c / T, hi = nb * (c + 1) / T;
        or_source src = base;
        or_source_skip(&src, (uint64_t)lo);
        errs[c] = or_roll_batches(&src, bounds + lo * k, k, hi - lo, rolls + lo * k, words ? words + lo : NULL,
                                  flags ? flags + lo : NULL, rk ? rk + lo : NULL);
        extra[c] = (src.drawn - base.drawn) - hi;
    }
    uint64_t D = 0;
    for (int c = 0; c < T; ++c) {
        if (errs[c]) return errs[c];
        const int64_t lo = nb * c / T, hi = nb * (c + 1) / T;
        if (D != 0) {
            or_source src = base;
            or_source_skip(&src, (uint64_t)lo + D);
            const int st = or_roll_batches(&src, bounds + lo * k, k, hi - lo, rolls + lo * k, words ? words + lo : NULL,
                                           flags ? flags + lo : NULL, rk ? rk + lo : NULL);
            if (st) return st;
            extra[c] = (src.drawn - base.drawn) - hi - (int64_t)D;
        }
        D += (uint64_t)extra[c];
    }
    *s = base;
    or_source_skip(s, (uint64_t)nb + D);
    return OR_OK;
}

int or_gen_bounds(or_source *s, uint32_t *out, int64_t count, uint64_t lo, uint64_t span) {
    for (int64_t i = 0; i < count; ++i) {
        uint64_t v, nw;
        int32_t ro;
        int st = or_roll_single(s, span, 0, &v, &nw, &ro);
        if (st) return st;
        out[i] = (uint32_t)(lo + v);
    }
    return OR_OK;
}

/* batched.py:126-128 roll_batch_naive: roll_single on the product, then decode
 * (mixed_radix.py:53-67: divmod by the bases in reverse) */
int or_roll_batch_naive(or_source *s, const uint64_t *bases, int32_t k, uint64_t *digits) {
    u128 prod;
    int st = radix_product(bases, k, s->word_bits, &prod);
    if (st) return st;
    uint64_t v, words;
    int32_t ro;
    st = or_roll_single(s, (uint64_t)prod, (uint64_t)(prod >> 64), &v, &words, &ro);
    if (st) return st;
    u128 val = v;
    for (int m = k - 1; m >= 0; --m) {
        digits[m] = (uint64_t)(val % bases[m]);
        val /= bases[m];
    }
    return OR_OK;
}

/* segmented shuffle_naive_batched: array a shuffled with make_source(G, hash(run_seed, base + a)) */
int or_shuffle_naive_segmented(void *data, int32_t eb, int64_t num_arrays, uint64_t n, uint64_t run_seed,
                               int64_t base, uint32_t *words_out, int32_t nthreads, int32_t generator) {
    int err = OR_OK;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t a = 0; a < num_arrays; ++a) {
        or_source src;
        const uint64_t seed = or_array_seed(run_seed, (uint64_t)(base + a));
        if (generator == 2) or_source_chacha(&src, seed);
        else if (generator == 1) or_source_lehmer(&src, seed);
        else or_source_pcg64(&src, seed);
        int st = or_shuffle_naive_batched(&src, (unsigned char *)data + (size_t)a * n * eb, eb, n);
        if (st) err = st;
        if (words_out) words_out[a] = (uint32_t)src.drawn;
    }
    (void)nthreads;
    return err;
}

int or_shuffle_segmented(void *data, int32_t eb, int64_t num_arrays, uint64_t n,
                         uint64_t run_seed, int64_t base, const uint64_t *lengths,
                         const uint32_t *sizes, int32_t nent, uint32_t *words_out,
                         int32_t nthreads, int32_t unbatched) {
    return or_shuffle_segmented_gen(data, eb, num_arrays, n, run_seed, base, lengths, sizes, nent,
                                    words_out, nthreads, unbatched, 0);
}

int or_shuffle_segmented_gen(void *data, int32_t eb, int64_t num_arrays, uint64_t n,
                             uint64_t run_seed, int64_t base, const uint64_t *lengths,
                             const uint32_t *sizes, int32_t nent, uint32_t *words_out,
                             int32_t nthreads, int32_t unbatched, int32_t generator) {
    int err = OR_OK;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t a = 0; a < num_arrays; ++a) {
        or_source src;
        if (generator == 2)
            or_source_chacha(&src, or_array_seed(run_seed, (uint64_t)(base + a)));
        else if (generator == 1)
            or_source_lehmer(&src, or_array_seed(run_seed, (uint64_t)(base + a)));
        else
            or_source_pcg64(&src, or_array_seed(run_seed, (uint64_t)(base + a)));
        unsigned char *z = (unsigned char *)data + (size_t)a * n * eb;
        int st = unbatched ? or_shuffle_unbatched(&src, z, eb, n)
                           : or_shuffle_batched(&src, z, eb, n, lengths, sizes, nent, 64, 0);
        if (st) err = st;
        if (words_out) words_out[a] = (uint32_t)src.drawn;
    }
    (void)nthreads;
    return err;
}

void or_pcg64_fill(const or_source *s0, uint64_t offset, uint64_t *out, int64_t count) {
    const int64_t CH = 1 << 16;
    int64_t nch = (count + CH - 1) / CH;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t c = 0; c < nch; ++c) {
        or_source s = *s0;
        if (s.kind == 3)
            or_chacha_advance(&s, offset + (uint64_t)(c * CH));
        else
            or_pcg64_advance(&s, offset + (uint64_t)(c * CH));
        int64_t end = (c + 1) * CH < count ? (c + 1) * CH : count;
        for (int64_t i = c * CH; i < end; ++i) or_next_word(&s, &out[i]);
    }
}
