/*
 * batchrand_b200.h -- C ABI of the B200-native batched-dice / segmented-shuffle path.
 *
 * Drop-in boundary for the hot path of the reference package
 * /root/reference/pkg/src/batchrand (arXiv 2408.06213).  The reference is pure Python
 * with no FFI; each entry point below states the reference function whose semantics it
 * reproduces bit-exactly (same words consumed, same digits, same permutation) and the
 * Python binding lives in paper_2408_06213_b200/batchrand.py (ctypes).  See
 * INTEGRATION.md for the binding a maintainer adds to the reference.
 *
 * Conventions
 *   - Plain C types only.  Pointers named *_dev are CUDA device pointers owned by the
 *     caller; `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Device entry points are asynchronous on `stream` and never synchronise the device,
 *     except the four marked SYNCHRONOUS below (br_state_download, br_roll_check and
 *     br_roll_batch64 synchronise `stream`; br_pcg64_next on a replayed-word state reads one
 *     word).  Shuffle plans are built on the device, stream-ordered, and cached; a cached
 *     plan is freed with cudaFreeAsync after every stream that used it has passed its last
 *     use.  Entry points return a status code; no C++ exception crosses the ABI.
 *     br_last_error() gives the thread-local message of the last failure.
 *   - Generator state that evolves across calls lives in device memory (br_pcg64 in
 *     *_dev buffers) so that back-to-back calls need no host round trip.
 *   - Word width is 64 bits (PCG64 XSL-RR 128/64, wordsource.py:71-89); items are 4 or 8
 *     bytes.  The stream forms take any n (shuffle.py:175-190: the single rolls above
 *     2^32 - 1 run in a 64-bit head kernel, the rest on the 32-bit kernels); the segmented
 *     forms take n < 2^32 (BR_E_UNSUPPORTED otherwise) and the naive ones raise
 *     BR_E_BOUND_OVERFLOW once the pair product passes 2^64 (shuffle.py:240-241).
 *   - There is no CPU fallback: without a CUDA device every device entry point returns
 *     BR_E_CUDA.
 */
#ifndef BATCHRAND_B200_H
#define BATCHRAND_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BR_ABI_VERSION 3

/* Status codes.  Python mapping (errors.py:4-37): */
#define BR_OK 0
#define BR_E_INVALID 1        /* ValueError            (shuffle.py:163-167, shuffle.py:35-48) */
#define BR_E_BOUND_OVERFLOW 2 /* BoundOverflow         (bounded.py:115-118, mixed_radix.py:33) */
#define BR_E_EXHAUSTED 3      /* SourceExhausted       (wordsource.py:203-204) */
#define BR_E_CUDA 4           /* RuntimeError (CUDA error / no device) */
#define BR_E_UNSUPPORTED 5    /* TypeError/NotImplementedError (size or source not handled) */

/* Generator state.  PCG64 (wordsource.py:71-89): 128-bit LCG state and ODD increment.
 * Lehmer128 (wordsource.py:51-67): 128-bit odd state, increment 0 -- an increment of 0 is
 * how every entry point below tells a Lehmer stream from a PCG64 stream. */
typedef struct br_pcg64 {
    uint64_t state_hi, state_lo;
    uint64_t inc_hi, inc_lo;
} br_pcg64;

/* ChaCha20 keystream (wordsource.py:136-164): a br_pcg64 head followed by the key.
 *   head.state = absolute position of the next word (ChaChaSource: counter*8 when the
 *                buffer is empty, else (counter-1)*8 + _pos/2); the next word is 64-bit
 *                word (position % 8) of block (position / 8) mod 2^64
 *   head.inc_hi = nonce, head.inc_lo = BR_CHACHA_TAG (even and non-zero, so no PCG64 or
 *                Lehmer state carries it)
 * Every entry point taking a br_pcg64* (host or device) reads the 64-byte br_chacha when
 * it sees the tag, so a ChaCha state buffer must be a whole br_chacha. */
#define BR_CHACHA_TAG 2
typedef struct br_chacha {
    br_pcg64 head;
    uint32_t key[8];
} br_chacha;

/* One regime of a ShuffleSchedule: (max_length, batch_size) (shuffle.py:22-30). */
typedef struct br_regime {
    uint64_t max_length;
    uint32_t batch_size;
    uint32_t reserved;
} br_regime;

/* One run of consecutive batches of a compiled plan: `count` batches of size k, the first
 * at remaining length start_n, each next one at start_n - k*c (shuffle.py:100-134). */
typedef struct br_segment {
    uint64_t start_n;
    uint32_t k;
    uint32_t reserved;
    uint64_t count;
} br_segment;

int br_abi_version(void);
const char *br_last_error(void);
/* number of visible CUDA devices (0 when none); never fails */
int br_device_count(void);

/* ---------------------------------------------------------------- host generator helpers */
/* wordsource.py:22-35 splitmix64_stream, one step */
uint64_t br_splitmix64_next(uint64_t *x);
/* wordsource.py:80-83 Pcg64Source.__init__ */
void br_pcg64_seed(uint64_t seed, br_pcg64 *out);
/* wordsource.py:61-63 LehmerSource.__init__ (increment 0) */
void br_lehmer_seed(uint64_t seed, br_pcg64 *out);
/* wordsource.py:147-153 ChaChaSource.__init__ (position 0) */
void br_chacha_seed(uint64_t seed, br_chacha *out);
/* wordsource.py:191-207 FixedSequenceSource with 64-bit words: a stream that replays the
 * `nwords` words at words_dev (device memory, kept alive by the caller for every call that
 * uses the state).  head.state = position of the next word, head.inc_hi = nwords,
 * head.inc_lo = BR_WORDS_TAG, key[0..1] = the address.  Words past the end read as
 * 2^64 - 1 (accepted by every batch, so the call terminates): the caller raises
 * SourceExhausted when a call ends at a position beyond nwords. */
#define BR_WORDS_TAG 4
int br_words_state(const uint64_t *words_dev, uint64_t nwords, br_chacha *out);
/* wordsource.py:85-89 Pcg64Source.next_word / :65-67 LehmerSource.next_word /
 * :155-164 ChaChaSource.next_word / a replayed word (synchronous device read), told apart
 * by the increment */
uint64_t br_pcg64_next(br_pcg64 *st);
/* O(log d) jump-ahead by `delta` words (numpy PCG64.advance semantics; ChaCha: position + d) */
void br_pcg64_advance(br_pcg64 *st, uint64_t delta);
/* Per-array seed convention: first splitmix64 output of ((run_seed << 32) | a) mod 2^64 */
uint64_t br_array_seed(uint64_t run_seed, uint64_t array_index);

/* ---------------------------------------------------------------- host plan helpers */
/* shuffle.py:32-49 ShuffleSchedule.__post_init__ (word_bits must be 64). */
int br_schedule_validate(const br_regime *entries, int n_entries, uint32_t max_batch, int word_bits);
/* bounded.py:107-119 falling_factorial; *hi is 1 only for the value 2^64. */
int br_falling_factorial(uint64_t n, uint32_t k, uint64_t *lo, uint64_t *hi);
/* Regime walk of shuffle_batched (shuffle.py:168-224): writes at most `cap` segments,
 * returns the number of segments (<0: -status).  n_batches_out = batches without
 * rejections = words consumed by an all-accept run. */
int64_t br_plan_build(uint64_t n, const br_regime *entries, int n_entries, br_segment *out,
                      int64_t cap, uint64_t *n_batches_out);

/* ---------------------------------------------------------------- device: generator */
/* out_dev[i] = word (offset + i) of the stream `st` (host struct, not modified). */
int br_pcg64_fill(uint64_t *out_dev, int64_t count, const br_pcg64 *st, uint64_t offset,
                  void *stream);
/* Copy a host state to/from device memory on `stream`.  Upload is asynchronous (the host
 * struct is copied into pinned staging before the call returns) and copies a whole br_chacha for a ChaCha state;
 * download is SYNCHRONOUS (it synchronises `stream`) and copies the 32-byte head (the key
 * never changes). */
int br_state_upload(br_pcg64 *state_dev, const br_pcg64 *st, void *stream);
int br_state_download(br_pcg64 *st, const br_pcg64 *state_dev, void *stream);

/* ---------------------------------------------------------------- device: batched rolls */
/* Bulk form of batched.py:102-123 roll_batch:
 *   for i in range(num_batches):
 *       r = roll_batch(src, BatchSpec(RadixBases.of(bounds[i*k:(i+1)*k])))
 *       rolls[i*k:(i+1)*k] = r.digits; words[i] = min(r.words_consumed, 255)
 *       flags[i] = r.threshold_computed; final_rk[i] = r.final_remainder
 * with src the stream in *state_dev (PCG64, Lehmer or ChaCha; advanced in place by the
 * words consumed).
 * bounds are u32 (>= 1); flags_dev / final_rk_dev may be NULL.  bounds_dev and rolls_dev
 * must be 16-byte aligned, words_dev and final_rk_dev 8-byte aligned (BR_E_INVALID otherwise).  `workspace_dev` is
 * br_roll_workspace_bytes() of zero-initialised device memory, reusable across calls on
 * one stream (calls sharing a workspace must be stream-ordered).  Invalid bounds (a zero
 * bound -> ValueError, product > 2^64 -> BoundOverflow) are reported through
 * br_roll_check(), which synchronises; the state is then left unchanged. */
size_t br_roll_workspace_bytes(void);
int br_roll_batches(const uint32_t *bounds_dev, int k, int64_t num_batches, br_pcg64 *state_dev,
                    uint32_t *rolls_dev, uint8_t *words_dev, uint8_t *flags_dev,
                    uint64_t *final_rk_dev, void *workspace_dev, void *stream);
/* The two launches of br_roll_batches issued separately (phase 1: the speculative main
 * kernel, phase 2: the exact fixup + state advance); phase 1 must be followed by phase 2 on
 * the same stream.  Used by bench.py to time the main kernel alone. */
int br_roll_batches_phase(const uint32_t *bounds_dev, int k, int64_t num_batches,
                          br_pcg64 *state_dev, uint32_t *rolls_dev, uint8_t *words_dev,
                          uint8_t *flags_dev, uint64_t *final_rk_dev, void *workspace_dev,
                          int phase, void *stream);
/* roll_batch_naive (batched.py:126-128) in the same bulk form: one Lemire draw on the
 * product of the k bounds, digits by division (mixed_radix.py:53-67).  Same words, digits
 * and acceptance as br_roll_batches (Theorem 1); the division-based baseline of the paper.
 * Status through br_roll_check as for br_roll_batches. */
int br_roll_batches_naive(const uint32_t *bounds_dev, int k, int64_t num_batches, br_pcg64 *state_dev,
                          uint32_t *rolls_dev, uint8_t *words_dev, uint8_t *flags_dev,
                          uint64_t *final_rk_dev, void *workspace_dev, void *stream);
/* SYNCHRONOUS: synchronises `stream`, returns the deferred status of the last br_roll_batches on this
 * workspace (BR_OK / BR_E_INVALID / BR_E_BOUND_OVERFLOW) and clears it.  *extra_words (may
 * be NULL) receives the words consumed beyond one per batch (rejections). */
int br_roll_check(void *workspace_dev, void *stream, uint64_t *extra_words);

/* One roll_batch (batched.py:102-123) with 64-bit bases -- any base below 2^64, product at
 * most 2^64 -- on the stream in *state_dev (any generator kind; advanced in place), or, with
 * state_dev NULL, one digit_pass (batched.py:69-82) of the word *r0_dev.  out_dev receives
 * k + 3 u64: the digits, the words consumed, threshold_computed (0/1), the final remainder.
 * A base of 0 encodes 2^64 (the full range, bounded.py:35-56).  The bulk entry points take
 * u32 bounds; this is the drop-in path for wider ones.  SYNCHRONOUS: reads the k bases back
 * to check the product before the launch. */
int br_roll_batch64(const uint64_t *bases_dev, int k, br_pcg64 *state_dev, const uint64_t *r0_dev,
                    uint64_t *out_dev, void *stream);

/* batched.py:69-82 digit_pass over many words (no generator): for word i with bases
 * bounds[i*k:(i+1)*k] (u32), digits[i*k+m] and the final remainder rk[i] (rk may be NULL). */
int br_digit_pass(const uint64_t *words_dev, const uint32_t *bounds_dev, int k, int64_t count,
                  uint32_t *digits_dev, uint64_t *rk_dev, void *stream);

/* ---------------------------------------------------------------- device: shuffles */
/* shuffle.py:149-225 shuffle_batched(src, z, schedule) on one device array of n elements
 * (elem_bytes 4 or 8), src = the stream in *state_dev (PCG64, Lehmer or ChaCha; advanced
 * in place).
 * unbatched != 0 runs shuffle.py:80-97 shuffle_unbatched instead (schedule ignored).
 * words_dev (may be NULL) receives the words consumed (u64). */
int br_shuffle_stream(void *z_dev, int elem_bytes, uint64_t n, br_pcg64 *state_dev,
                      const br_regime *entries, int n_entries, int unbatched,
                      uint64_t *words_dev, void *stream);
/* Same with an explicit plan (e.g. one partial batch, shuffle.py:137-146): the segments
 * are run in order on z[0:n].  rk_first_dev (may be NULL) receives the final remainder of
 * the FIRST word drawn (what _run_batches compares with the carried bound u). */
int br_shuffle_stream_segments(void *z_dev, int elem_bytes, uint64_t n, br_pcg64 *state_dev,
                               const br_segment *segs, int n_segs, uint64_t *words_dev,
                               uint64_t *rk_first_dev, void *stream);
/* Many independent shuffles: array a (0 <= a < num_arrays) of n elements at
 * data_dev + a*n*elem_bytes is shuffled in place by
 *     shuffle_batched(make_source(G, br_array_seed(run_seed, array_index_base + a)), z)
 * with G = "pcg64" (generator 0), "lehmer" (generator 1) or "chacha" (generator 2).
 * array_index_base lets shards of one job run on different GPUs with no exchange.
 * words_dev (may be NULL) receives words consumed per array (u32). */
int br_shuffle_segmented(void *data_dev, int elem_bytes, int64_t num_arrays, uint64_t n,
                         uint64_t run_seed, int64_t array_index_base, const br_regime *entries,
                         int n_entries, int generator, uint32_t *words_dev, void *stream);

/* shuffle.py:228-266 shuffle_naive_batched(src, z): Fisher-Yates two indices at a time,
 * one draw on (i+1)*i split by division, a single roll on 2 for a leftover index 1.
 * Stream form (as br_shuffle_stream) and the segmented form (as br_shuffle_segmented). */
int br_shuffle_naive_stream(void *z_dev, int elem_bytes, uint64_t n, br_pcg64 *state_dev,
                            uint64_t *words_dev, void *stream);
int br_shuffle_naive_segmented(void *data_dev, int elem_bytes, int64_t num_arrays, uint64_t n,
                               uint64_t run_seed, int64_t array_index_base, int generator,
                               uint32_t *words_dev, void *stream);

/* Kernel-selection report for the last device call on this thread (diagnostics). */
const char *br_last_kernel(void);
/* Free cached device plans (all devices). */
void br_release(void);

#ifdef __cplusplus
}
#endif
#endif
