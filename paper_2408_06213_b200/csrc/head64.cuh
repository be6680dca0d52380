// head64.cuh -- the single-roll head of arrays of 2^32 or more elements (stream form).
//
// shuffle.py:175-190: above the schedule's top regime every position takes one roll,
// i = len-1 down to the top length, bound b = i + 1 (64-bit here), word-level rejection
// (lo < b, then redraw while lo < (2^64 - b) mod b).  This kernel runs the positions
// i >= stop (= 2^32 - 1); the rest of the array (below 2^32 - 1, bounds < 2^32) continues
// through the 32-bit kernels on the same stream, so the sequence of draws is the reference's.
//
// One CTA, G = 1024 steps per group (lane l: i = top - l, word W + l, all lanes jump-ahead
// states).  A rejection at lane f commits lanes < f and re-runs step top - f on the next
// word.  Targets are uniform on [0, i], i >= 2^32 - 1, so within a group a repeated target
// (~G^2 / 2^33) or a target among the group's own positions (~G^2 / 2^32) is rare: the
// group's swaps are independent and run in parallel unless a 4096-slot hash of the targets
// (exact, linear probing) or the position check finds a conflict, in which case thread 0
// applies the group's swaps in order.
#pragma once
#include "chacha.cuh"
#include "jump.cuh"

namespace br {

static constexpr int H64_T = 1024;
static constexpr uint32_t H64_SLOTS = 4096;

template <typename T>
__global__ void __launch_bounds__(H64_T) shuffle_head64_kernel(T *__restrict__ z, uint64_t n, uint64_t stop,
                                                               uint64_t *state_io, uint64_t *head_words,
                                                               uint64_t *rk_first) {
    __shared__ unsigned long long tbl[H64_SLOTS];  // target + 1 (0 = empty)
    __shared__ uint64_t J[H64_T];
    __shared__ uint32_t fmin, conflict;
    const int L = threadIdx.x;
    const u128 s0 = mk128(state_io[0], state_io[1]), inc = mk128(state_io[2], state_io[3]);
    const bool pos = is_posgen(inc);  // ChaCha / replayed words: the state is a word position
    const bool lh = !pos && is_lehmer(inc);
    ChaKey K;
    if (pos) K = cha_key_of_state(state_io);
    // lane state: its next output is word W + L (W = words consumed so far)
    u128 s = pos ? cha_add(s0, (uint64_t)L + 1) : gen_jump_small(s0, inc, L + 1, lh);
    const u128 AJ = gen_SA(lh, H64_T), CJ = mul128(g_SG[H64_T], inc);
    uint64_t top = n - 1, left = n - stop, extra = 0;  // positions stop .. top remain
    bool first = true;
    while (left > 0) {
        const uint64_t cnt = min((uint64_t)H64_T, left);
        for (uint32_t q = L; q < H64_SLOTS; q += H64_T) tbl[q] = 0ull;
        if (L == 0) {
            fmin = 0xFFFFFFFFu;
            conflict = 0;
        }
        __syncthreads();
        uint64_t i = 0, j = 0;
        bool act = (uint64_t)L < cnt;
        if (act) {
            i = top - (uint64_t)L;
            const uint64_t b = i + 1;  // i < n <= 2^64 - 1
            const uint64_t w = pos ? cha_out(K, s) : gen_out(s, lh);
            const uint64_t lo = b * w;
            j = __umul64hi(b, w);
            if (first && L == 0 && rk_first) *rk_first = lo;
            if (lo < b && lo < (0ull - b) % b) atomicMin(&fmin, (uint32_t)L);
        }
        __syncthreads();
        const uint32_t f = fmin;  // lanes >= f are not committed this round
        act = act && (uint32_t)L < f;
        const uint64_t nv = min(cnt, (uint64_t)f);
        if (act) {
            J[L] = j;
            if (j >= top - nv + 1 && j != i) conflict = 1;  // the target is another lane's position
            uint32_t h = (uint32_t)((j * 0x9E3779B97F4A7C15ull) >> 52);
            for (;;) {  // exact duplicate check (linear probing)
                const unsigned long long old = atomicCAS(&tbl[h], 0ull, (unsigned long long)(j + 1));
                if (old == 0ull) break;
                if (old == (unsigned long long)(j + 1)) {
                    conflict = 1;
                    break;
                }
                h = (h + 1) & (H64_SLOTS - 1);
            }
        }
        __syncthreads();
        if (!conflict) {
            if (act) {
                const T a = z[i], c = z[j];
                z[i] = c;
                z[j] = a;
            }
        } else if (L == 0) {
            for (uint64_t l = 0; l < nv; ++l) {
                const uint64_t ii = top - l, jj = J[l];
                const T a = z[ii];
                z[ii] = z[jj];
                z[jj] = a;
            }
        }
        first = false;
        if (f == 0xFFFFFFFFu) {  // every step of the group committed
            top -= cnt;
            left -= cnt;
            if (left) s = pos ? cha_add(s, H64_T) : mad128(s, AJ, CJ);
        } else {  // step top - f is re-drawn from the next word
            top -= f;
            left -= f;
            extra += 1;
            s = pos ? cha_add(s, (uint64_t)f + 1) : gen_jump_small(s, inc, (int)f + 1, lh);
        }
        __syncthreads();
    }
    if (L == 0) {
        const uint64_t words = (n - stop) + extra;
        const u128 sf = pos ? cha_add(s0, words) : gen_jump(s0, inc, words, lh);
        state_io[0] = sf.hi;
        state_io[1] = sf.lo;
        *head_words = words;
    }
}

__global__ void add_words_kernel(uint64_t *words, const uint64_t *more) {
    if (words) words[0] += more[0];
}

}  // namespace br
