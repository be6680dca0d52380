// capi.cu -- C ABI (include/batchrand_b200.h): host plan compiler, plan cache, launches.
//
// One translation unit: the kernels (roll.cuh, shuffle.cuh) and the jump-table symbols
// they read live here so no relocatable device code is needed.
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/batchrand_b200.h"
#include "chacha.cuh"
#include "core.cuh"
#include "jump.cuh"
#include "roll.cuh"
#include "shuffle.cuh"
#include "stage_shuffle.cuh"
#include "head64.cuh"
#include "warp_shuffle.cuh"

using namespace br;

namespace {

thread_local std::string g_err;
thread_local std::string g_kernel;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(BR_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));  \
    } while (0)

typedef unsigned __int128 h128;


const JumpTables &host_tables() {
    static JumpTables t;
    static std::once_flag once;
    std::call_once(once, [] { build_jump_tables(t); });
    return t;
}

struct DeviceInfo {
    bool ready = false;
    int sms = 0;
    bool coop = false;
};
std::mutex g_mu;
std::map<int, DeviceInfo> g_dev;

int ensure_device(int *dev_out, DeviceInfo *info_out) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(BR_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    std::lock_guard<std::mutex> lk(g_mu);
    DeviceInfo &d = g_dev[dev];
    if (!d.ready) {
        const JumpTables &t = host_tables();
        CK(cudaMemcpyToSymbol(c_A, t.A, sizeof(t.A)));
        CK(cudaMemcpyToSymbol(c_G, t.G, sizeof(t.G)));
        CK(cudaMemcpyToSymbol(g_SA, t.SA, sizeof(t.SA)));
        CK(cudaMemcpyToSymbol(g_SG, t.SG, sizeof(t.SG)));
        CK(cudaMemcpyToSymbol(c_LA, t.LA, sizeof(t.LA)));
        CK(cudaMemcpyToSymbol(g_LSA, t.LSA, sizeof(t.LSA)));
        CK(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
        // stream-ordered scratch (cudaMallocAsync) stays mapped in the pool between calls
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = 16ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
        int coop = 0;
        CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        d.coop = coop != 0;
        d.ready = true;
    }
    *dev_out = dev;
    *info_out = d;
    return BR_OK;
}

// ---------------------------------------------------------------- plan compiler
// Regime walk of shuffle_batched (shuffle.py:168-224); head of single rolls above the top
// regime (shuffle.py:175-190) becomes one k=1 segment.
int build_segments(uint64_t n, const br_regime *e, int ne, std::vector<br_segment> &segs, uint64_t &nbatches) {
    segs.clear();
    nbatches = 0;
    if (n < 2) return BR_OK;
    if (ne < 1 || !e) return fail(BR_E_INVALID, "schedule needs at least one regime");
    uint64_t remaining = n;
    const uint64_t top = e[0].max_length;
    auto push = [&](uint64_t start, uint32_t k, uint64_t count) {
        br_segment s;
        s.start_n = start;
        s.k = k;
        s.reserved = 0;
        s.count = count;
        segs.push_back(s);
        nbatches += count;
    };
    if (remaining > top) {
        push(remaining, 1, remaining - top);
        remaining = top;
    }
    int idx = 0;
    for (int pos = 0; pos < ne; ++pos) {
        if (e[pos].max_length >= remaining) idx = pos;
        else break;
    }
    uint32_t k = e[idx].batch_size;
    while (remaining > 1) {
        if (remaining < k) {
            push(remaining, (uint32_t)(remaining - 1), 1);
            break;
        }
        if (idx + 1 < ne && remaining <= e[idx + 1].max_length) {
            ++idx;
            k = e[idx].batch_size;
            continue;
        }
        uint64_t count = (idx + 1 < ne) ? (remaining - e[idx + 1].max_length + k - 1) / k : remaining / k;
        if (count == 0 || k == 0) return fail(BR_E_INVALID, "degenerate schedule");
        push(remaining, k, count);
        remaining -= count * k;
    }
    return BR_OK;
}

int ff_checked(uint64_t n, uint64_t k, h128 *out) {
    if (k > n) return BR_E_INVALID;
    h128 acc = 1, lim = (h128)1 << 64;
    for (uint64_t f = n; f > n - k; --f) {
        acc *= f;
        if (acc > lim) return BR_E_BOUND_OVERFLOW;
    }
    *out = acc;
    return BR_OK;
}

// ---------------------------------------------------------------- device plans
// A plan is built ON THE DEVICE, stream-ordered, from its segment list (at most MAX_SEGS
// entries, passed by value): plan_build_kernel writes the segments, the exact threshold
// 2^64 mod ff(n_b, k_b) of every batch and, for n < 2^16, the warp kernels' batch records.  No
// host copy, no host memory per batch, no synchronisation.  Plans are cached per (device,
// segments, n, naive) and shared by later calls on any stream (they wait for the build event);
// each is reference-counted and, once evicted and unused, freed with cudaFreeAsync after an
// event of every stream that used it -- never while a launched kernel can still read it.
struct PlanSegs {
    DevSeg s[MAX_SEGS];
    uint32_t nseg, nbatches, brec;
};

__global__ void plan_build_kernel(PlanSegs ps, DevSeg *__restrict__ segs_out, uint64_t *__restrict__ thresh,
                                  uint4 *__restrict__ brec) {
    const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (t0 < ps.nseg) segs_out[t0] = ps.s[t0];
    for (uint32_t b = t0; b < ps.nbatches; b += gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = ps.nseg - 1;  // last segment with first_batch <= b
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (ps.s[mid].first_batch <= b) lo = mid;
            else hi = mid - 1;
        }
        const DevSeg S = ps.s[lo];
        const uint32_t nb = S.start_n - (b - S.first_batch) * S.k;
        unsigned __int128 f = 1;  // ff(nb, k) <= 2^64, checked on the host for the segment start
        for (uint32_t m = 0; m < S.k; ++m) f *= (uint64_t)(nb - m);
        const uint64_t f64 = (uint64_t)f;
        const uint64_t t = (f >> 64) ? 0 : (0 - f64) % f64;  // bounded.py:59-62 (2^64 mod ff)
        thresh[b] = t;
        if (ps.brec) brec[b] = make_uint4((uint32_t)t, (uint32_t)(t >> 32), nb, S.k);
    }
}

cudaStream_t free_stream(int dev) {
    static std::mutex mu;
    static std::map<int, cudaStream_t> streams;
    std::lock_guard<std::mutex> lk(mu);
    auto it = streams.find(dev);
    if (it != streams.end()) return it->second;
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) s = nullptr;
    streams[dev] = s;
    return s;
}

struct PlanStore {
    int dev = -1;
    void *mem = nullptr;
    size_t bytes = 0;
    DevPlan plan{};
    uint64_t nbatches = 0;
    cudaEvent_t built = nullptr;
    std::mutex mu;
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;  // last use per stream

    // make `st` wait for the build (a no-op once it has completed)
    int ready_on(cudaStream_t st) {
        if (built) CK(cudaStreamWaitEvent(st, built, 0));
        return BR_OK;
    }
    // record that kernels reading this plan were queued on `st`
    void used(cudaStream_t st) {
        std::lock_guard<std::mutex> lk(mu);
        for (auto &u : uses)
            if (u.first == st) {
                cudaEventRecord(u.second, st);
                return;
            }
        if (uses.size() >= 16) {  // many streams: retire the oldest record (a host wait on a past event)
            cudaEventSynchronize(uses.front().second);
            cudaEventDestroy(uses.front().second);
            uses.erase(uses.begin());
        }
        cudaEvent_t ev = nullptr;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            cudaStreamSynchronize(st);  // cannot track it: make the use complete instead
            return;
        }
        cudaEventRecord(ev, st);
        uses.emplace_back(st, ev);
    }
    ~PlanStore() {
        if (!mem) return;
        int cur = -1;
        if (cudaGetDevice(&cur) != cudaSuccess) return;  // runtime gone (process exit)
        cudaSetDevice(dev);
        cudaStream_t fs = free_stream(dev);
        for (auto &u : uses) {
            cudaStreamWaitEvent(fs, u.second, 0);
            cudaEventDestroy(u.second);
        }
        if (built) {
            cudaStreamWaitEvent(fs, built, 0);
            cudaEventDestroy(built);
        }
        cudaFreeAsync(mem, fs);
        cudaGetLastError();
        cudaSetDevice(cur);
    }
};
using PlanRef = std::shared_ptr<PlanStore>;

struct PlanCache {
    std::map<std::pair<int, std::string>, PlanRef> map;
    std::list<std::pair<int, std::string>> lru;  // front = most recent
    size_t bytes = 0;
};
// never destroyed: plan destructors must not run after the CUDA runtime has shut down
PlanCache &plan_cache() {
    static PlanCache *c = new PlanCache;
    return *c;
}
constexpr size_t PLAN_CACHE_MAX = 4096;          // plans
constexpr size_t PLAN_CACHE_BYTES = 1ull << 30;  // device bytes over all cached plans
constexpr size_t PLAN_ITEM_BYTES = 256ull << 20; // larger plans serve their call and are freed

// Plan of segments `segs` for length n on the current device, ready on stream `st`.
int get_plan(uint64_t n, const std::vector<br_segment> &segs, bool naive, cudaStream_t st, PlanRef *out) {
    int dev;
    DeviceInfo di;
    int e0 = ensure_device(&dev, &di);
    if (e0) return e0;
    std::string key((const char *)segs.data(), segs.size() * sizeof(br_segment));
    key.append((const char *)&n, sizeof(n));
    key.push_back(naive ? 'N' : 'B');
    const auto ck = std::make_pair(dev, key);
    PlanCache &pc = plan_cache();
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = pc.map.find(ck);
        if (it != pc.map.end()) {
            *out = it->second;
            pc.lru.remove(ck);
            pc.lru.push_front(ck);
        }
    }
    if (*out) return (*out)->ready_on(st);
    if (segs.size() > (size_t)MAX_SEGS) return fail(BR_E_UNSUPPORTED, "plan has too many segments");
    PlanSegs ps{};
    uint64_t fb = 0, steps = 0;
    uint32_t maxk = 0;
    for (const br_segment &s : segs) {
        if (s.start_n >= (1ull << 32)) return fail(BR_E_UNSUPPORTED, "arrays of 2^32 or more elements");
        if (s.k == 0 || (uint64_t)s.k * s.count > s.start_n)
            return fail(BR_E_INVALID, "segment runs past the start of the array");
        h128 f;  // ff(n_b, k) grows with n_b: the segment's first batch is its largest
        int e = ff_checked(s.start_n, s.k, &f);
        if (e) return fail(e, "falling factorial of a batch exceeds 2^64");
        DevSeg &d = ps.s[ps.nseg++];
        d.start_n = (uint32_t)s.start_n;
        d.k = s.k;
        d.count = (uint32_t)s.count;
        d.first_batch = (uint32_t)fb;
        maxk = std::max(maxk, s.k);
        fb += s.count;
        steps += (uint64_t)s.k * s.count;
        if (fb >= (1ull << 32)) return fail(BR_E_UNSUPPORTED, "too many batches");
    }
    ps.nbatches = (uint32_t)fb;
    ps.brec = n < 65536 ? 1u : 0u;
    const size_t off = (ps.nseg * sizeof(DevSeg) + 15) & ~(size_t)15;
    const size_t boff = off + ((fb * sizeof(uint64_t) + 15) & ~(size_t)15);
    const size_t bytes = boff + (ps.brec ? fb * sizeof(uint4) : 0) + 16;
    auto p = std::make_shared<PlanStore>();
    p->dev = dev;
    p->bytes = bytes;
    CK(cudaMallocAsync(&p->mem, bytes, st));
    char *base = (char *)p->mem;
    const int threads = 256;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((fb + threads - 1) / threads, (uint64_t)di.sms * 8));
    plan_build_kernel<<<grid, threads, 0, st>>>(ps, (DevSeg *)base, (uint64_t *)(base + off),
                                                ps.brec ? (uint4 *)(base + boff) : nullptr);
    CK(cudaGetLastError());
    CK(cudaEventCreateWithFlags(&p->built, cudaEventDisableTiming));
    CK(cudaEventRecord(p->built, st));
    p->plan.n = (uint32_t)n;
    p->plan.nbatches = (uint32_t)fb;
    p->plan.nseg = ps.nseg;
    p->plan.max_k = maxk;
    p->plan.lo = (uint32_t)(n > steps ? n - steps : 0);
    p->plan.naive = naive ? 1u : 0u;
    p->plan.segs = (const DevSeg *)base;
    p->plan.thresh = (const uint64_t *)(base + off);
    p->plan.brec = ps.brec ? (const uint4 *)(base + boff) : nullptr;
    p->nbatches = fb;
    if (bytes <= PLAN_ITEM_BYTES) {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = pc.map.find(ck);
        if (it != pc.map.end()) {  // another thread built it meanwhile: keep theirs, ours dies after use
            pc.lru.remove(ck);
        } else {
            pc.bytes += bytes;
        }
        if (it == pc.map.end()) pc.map[ck] = p;
        pc.lru.push_front(ck);
        while ((pc.bytes > PLAN_CACHE_BYTES || pc.map.size() > PLAN_CACHE_MAX) && pc.lru.size() > 1) {
            auto victim = pc.lru.back();
            pc.lru.pop_back();
            auto v = pc.map.find(victim);
            if (v != pc.map.end()) {
                pc.bytes -= v->second->bytes;
                pc.map.erase(v);  // freed (stream-ordered) once no caller holds it
            }
        }
    }
    *out = p;
    return BR_OK;
}

__global__ void pcg_fill_kernel(uint64_t *__restrict__ out, int64_t count, u128 s0, u128 inc, uint64_t offset) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t per = (((count + nwarps - 1) / nwarps) + 31) & ~(int64_t)31;
    const int64_t wb = warp * per, we = min(wb + per, count);
    if (wb >= we) return;
    const bool lh = is_lehmer(inc);
    u128 s = gen_jump(s0, inc, offset + (uint64_t)wb, lh);
    s = gen_jump_small(s, inc, lane + 1, lh);
    const u128 A32 = gen_SA(lh, 32), C32 = mul128(g_SG[32], inc);
    for (int64_t b0 = wb; b0 < we; b0 += 32) {
        const int64_t i = b0 + lane;
        if (i < we) out[i] = gen_out(s, lh);
        s = mad128(s, A32, C32);
    }
}

// ChaCha keystream words: thread t computes block (P0 + offset)/8 + t and writes the
// words of it that fall in [0, count).
__global__ void cha_fill_kernel(uint64_t *__restrict__ out, int64_t count, ChaKey K, u128 p0) {
    const uint32_t q0 = (uint32_t)(p0.lo & 7);  // word of the first block that is out[0]
    const int64_t nblk = ((int64_t)q0 + count + 7) >> 3;
    const uint64_t blk0 = cha_block_of(p0);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nblk; t += (int64_t)gridDim.x * blockDim.x) {
        uint32_t b[16];
        cha_block_any(K, blk0 + (uint64_t)t, b);
        const int64_t i0 = t * 8 - q0;  // out index of word 0 of this block
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int64_t i = i0 + q;
            if (i >= 0 && i < count) out[i] = ((uint64_t)b[2 * q + 1] << 32) | b[2 * q];
        }
    }
}

// One batch with 64-bit bases (batched.py:69-123 with bases up to 2^64, product <= 2^64,
// checked by the caller): the sequential roll_batch on one thread, any generator kind.  The
// bulk kernels take u32 bounds; this is the drop-in path for wider bases (roll_single with a
// bound above 2^32, RadixBases with a base above 2^32).  With state == nullptr it is a plain
// digit pass of the word *r0 (digit_pass).  out: digits[k], words, threshold_computed, rk.
__global__ void roll_one64_kernel(const uint64_t *__restrict__ bases, int k, uint64_t prod, int full,
                                  uint64_t *state, const uint64_t *r0, uint64_t *out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const bool stream = state != nullptr;
    u128 s = mk128(0, 0), inc = mk128(0, 0);
    bool pos = false, lh = false;
    ChaKey ck;
    ChaCursor cur;
    cur.valid = false;
    if (stream) {
        s = mk128(state[0], state[1]);
        inc = mk128(state[2], state[3]);
        pos = is_posgen(inc);
        lh = is_lehmer(inc);
        if (pos) ck = cha_key_of_state(state);
    }
    uint64_t words = 0, r = 0, t = 0;
    bool tc = false;
    for (;;) {
        uint64_t w;
        if (!stream) {
            w = *r0;
        } else if (pos) {
            s = cha_add(s, 1);
            w = cha_out_cached(ck, cur, s);
        } else {
            w = gen_next(s, inc, lh);
        }
        ++words;
        r = w;
        for (int m = 0; m < k; ++m) {
            const uint64_t b = bases[m];
            if (b == 0) {  // the base 2^64 (alone in a batch): digit = r, remainder 0
                out[m] = r;
                r = 0;
            } else {
                out[m] = __umul64hi(b, r);
                r = b * r;
            }
        }
        if (!stream) break;
        if (words == 1) {  // batched.py:116-119: the threshold only if r_k < product
            if (!full && r >= prod) break;
            tc = true;
            t = full ? 0 : (0 - prod) % prod;
        }
        if (r >= t) break;
    }
    out[k] = words;
    out[k + 1] = tc ? 1 : 0;
    out[k + 2] = r;
    if (stream) {
        state[0] = s.hi;
        state[1] = s.lo;
    }
}

// position-addressed streams (ChaCha keystream or replayed words): 64-byte states
inline bool host_is_chacha(const br_pcg64 *st) { return st->inc_lo == CHACHA_TAG || st->inc_lo == WORDS_TAG; }

inline ChaKey host_cha_key(const br_pcg64 *st) {
    const br_chacha *c = reinterpret_cast<const br_chacha *>(st);
    ChaKey K;
    for (int i = 0; i < 8; ++i) K.k[i] = c->key[i];
    K.nonce = st->inc_hi;
    K.words = nullptr;
    K.nwords = 0;
    if (st->inc_lo == WORDS_TAG) {
        uint64_t addr;
        memcpy(&addr, c->key, sizeof addr);
        K.words = reinterpret_cast<const uint64_t *>(addr);
        K.nwords = st->inc_hi;
    }
    return K;
}

int grid_for(const DeviceInfo &di, const void *kernel, int threads, size_t smem, int64_t work_blocks) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    int64_t g = (int64_t)per_sm * di.sms;
    if (work_blocks < g) g = work_blocks;
    return (int)(g < 1 ? 1 : g);
}

// Generator of each state buffer as last uploaded by br_state_upload: picks the main roll
// kernel.  Only a hint -- the kernels check the tag and fall back (see roll.cuh mark_main).
std::mutex g_kind_mu;
std::map<const void *, bool> g_is_chacha;

void note_state_kind(const void *dev, bool chacha) {
    std::lock_guard<std::mutex> lk(g_kind_mu);
    if (g_is_chacha.size() >= 65536) g_is_chacha.clear();  // only a hint: forgetting is safe
    g_is_chacha[dev] = chacha;
}

bool state_is_chacha(const void *dev) {
    std::lock_guard<std::mutex> lk(g_kind_mu);
    auto it = g_is_chacha.find(dev);
    return it != g_is_chacha.end() && it->second;
}

template <int K>
int launch_roll(const RollArgs &a, const DeviceInfo &di, cudaStream_t st, int phase) {
    const int threads = 256;
    const bool cha = (phase & 1) && state_is_chacha(a.state);
    if (cha) {
        const int64_t warps = (a.nb + 255) / 256;  // a 256-word keystream window per warp
        int grid = grid_for(di, (const void *)roll_cha_kernel<K>, threads, 0, (warps + 7) / 8);
        roll_cha_kernel<K><<<grid, threads, 0, st>>>(a);
        CK(cudaGetLastError());
    } else if (phase & 1) {
        int64_t work_blocks = (a.nb + 8 * 512 - 1) / (8 * 512);
        if constexpr (K <= 2) {
            const void *kp = a.flags ? (a.rk ? (const void *)roll_fast_kernel<K, true, true>
                                             : (const void *)roll_fast_kernel<K, true, false>)
                                     : (a.rk ? (const void *)roll_fast_kernel<K, false, true>
                                             : (const void *)roll_fast_kernel<K, false, false>);
            if (K == 2 && a.naive)  // division digits (k = 1 has nothing to divide)
                kp = a.flags ? (a.rk ? (const void *)roll_fast_kernel<K, true, true, true>
                                     : (const void *)roll_fast_kernel<K, true, false, true>)
                             : (a.rk ? (const void *)roll_fast_kernel<K, false, true, true>
                                     : (const void *)roll_fast_kernel<K, false, false, true>);
            int grid = grid_for(di, kp, threads, 0, work_blocks);
            RollArgs b = a;
            void *args[] = {&b};
            CK(cudaLaunchKernel(kp, dim3(grid), dim3(threads), args, 0, st));
        } else {
            int grid = grid_for(di, (const void *)roll_main_kernel<K>, threads, 0, work_blocks);
            roll_main_kernel<K><<<grid, threads, 0, st>>>(a);
        }
        CK(cudaGetLastError());
    }
    if (phase & 2) {
        // fixup: one block per SM, launched as a programmatic dependent of the main kernel so
        // its launch latency overlaps the main kernel's tail.  Its grid barrier (only reached
        // when a batch was rejected) needs every block co-resident, which only a cooperative
        // launch guarantees (other streams, MPS SM limits or green contexts can hold SMs), so
        // the cooperative attribute is the default; BR_ROLL_FIXUP=plain drops it (A/B only).
        if (di.sms * (threads / 32) > ROLL_MAX_WARPS) return fail(BR_E_UNSUPPORTED, "more SMs than the roll workspace covers");
        RollArgs b = a;
        void *args[] = {&b};
        cudaLaunchConfig_t cfg = {};
        const char *fx = getenv("BR_ROLL_FIXUP");
        const bool coop = !(fx && !strcmp(fx, "plain"));
        cfg.gridDim = dim3(di.sms);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = st;
        cudaLaunchAttribute attrs[2];
        attrs[0].id = cudaLaunchAttributeCooperative;
        attrs[0].val.cooperative = 1;
        attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attrs;
        cfg.numAttrs = (phase & 1) ? 2 : 1;
        if (!coop) {
            attrs[0] = attrs[1];
            cfg.numAttrs = (phase & 1) ? 1 : 0;
        }
        cudaError_t e = cudaLaunchKernelExC(&cfg, (const void *)roll_fixup_kernel<K>, args);
        if (e != cudaSuccess && (phase & 1)) {  // programmatic serialization refused: launch without it
            cudaGetLastError();
            attrs[0].id = cudaLaunchAttributeCooperative;
            attrs[0].val.cooperative = 1;
            cfg.numAttrs = coop ? 1 : 0;
            e = cudaLaunchKernelExC(&cfg, (const void *)roll_fixup_kernel<K>, args);
        }
        if (e != cudaSuccess) return fail(BR_E_CUDA, std::string("fixup launch: ") + cudaGetErrorString(e));
    }
    g_kernel = std::string(cha ? "roll_cha_kernel<" : K <= 2 ? "roll_fast_kernel<" : "roll_main_kernel<") +
               std::to_string(K) + ">+roll_fixup_kernel";
    return BR_OK;
}

constexpr uint32_t SMALL_SMEM_MAX = 64 * 1024;   // per 128-thread block
constexpr uint32_t MID_SMEM_MAX = 200 * 1024;    // per warp
constexpr uint32_t WARP_SMEM_MAX = 48 * 1024;    // warp kernel: several arrays per SM or none
constexpr uint32_t WARP_SMEM_DEFAULT = 16 * 1024; // warp kernel by default (measured crossover)
#ifndef LARGE_W
#define LARGE_W 16  // C5: 12.2 ms (8 warps: 12.9, 4 warps: 17.5)
#endif
#ifndef CTA_W
#define CTA_W 4
#endif
#ifndef RES_W
#define RES_W 8
#endif
#ifndef RES_WS
#define RES_WS 16  // single-array stream calls: one CTA, as wide as its window allows
#endif

// BR_SHUFFLE_KERNEL=small|resolve|idx|warp|hash|mid|stage|large|global restricts the dispatch below to one
// shuffle kernel where it is eligible (tests cover every kernel; A/B timing).  Unset: the
// first eligible kernel in the order below.
enum { K_ANY = 0, K_SMALL, K_RESOLVE, K_HASH, K_MID, K_LARGE, K_GLOBAL, K_WARP, K_IDX, K_STAGE };
int forced_kernel() {
    const char *e = getenv("BR_SHUFFLE_KERNEL");
    if (!e || !*e) return K_ANY;
    static const char *names[] = {"", "small", "resolve", "hash", "mid", "large", "global", "warp", "idx", "stage"};
    for (int i = 1; i <= K_STAGE; ++i)
        if (!strcmp(e, names[i])) return i;
    return K_ANY;
}

// staging buffers per CTA of the index-permutation kernel (BR_IDX_STAGES, default 2)
int idx_stages() {
    const char *e = getenv("BR_IDX_STAGES");
    const int v = e ? atoi(e) : 2;
    return v >= 8 ? 8 : (v >= 4 ? 4 : (v >= 2 ? 2 : 1));  // a power of two: ticket slots are tk % 32
}

inline bool allow(int k) {
    const int f = forced_kernel();
    return f == K_ANY || f == k;
}

template <typename T>
int launch_shuffle(void *data, int64_t num_arrays, uint64_t n, const PlanStore &cp, bool segmented,
                   uint64_t run_seed, int64_t base, uint32_t *words32, uint64_t *state_dev, uint64_t *words64,
                   uint64_t *rk_first, int gen, const DeviceInfo &di, cudaStream_t st) {
    const uint32_t stride = (uint32_t)(n | 1u);
    const int tpb = 64;  // 2 warps: many small blocks per SM overlap their load/compute/store phases
    const size_t small_smem = (size_t)tpb * stride * sizeof(T);
    // n <= 64: u8 index permutations in a transposed (conflict-free) layout, payload applied per warp
    if (allow(K_SMALL) && segmented && cp.plan.max_k <= 8 && n <= 64 && !getenv("BR_SMALL_ROWS")) {
        auto kern = n == 64 ? (gen == 2 ? shuffle_small_idx_kernel<T, true, 64> : shuffle_small_idx_kernel<T, false, 64>)
                            : (gen == 2 ? shuffle_small_idx_kernel<T, true> : shuffle_small_idx_kernel<T, false>);
        const int64_t blocks = (num_arrays + SMI_T - 1) / SMI_T;
        kern<<<(unsigned)blocks, SMI_T, 0, st>>>((T *)data, num_arrays, cp.plan, run_seed, base, words32, gen);
        CK(cudaGetLastError());
        g_kernel = std::string("shuffle_small_idx_kernel<u") + std::to_string(8 * sizeof(T)) + ">";
        return BR_OK;
    }
    if (allow(K_SMALL) && segmented && cp.plan.max_k <= 8 && small_smem <= SMALL_SMEM_MAX / 2) {
        auto kern = gen == 2 ? shuffle_small_kernel<T, true> : shuffle_small_kernel<T, false>;
        CK(cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)small_smem));
        int64_t blocks = (num_arrays + tpb - 1) / tpb;
        // q / n == umulhi(q, ceil(2^32 / n)) exactly for q < 2^32 / n (spans are < 2^16 elements)
        const uint32_t magic = (uint32_t)((((uint64_t)1 << 32) + n - 1) / n);
        const int vec_ok = ((n * sizeof(T)) % 16 == 0 && ((uintptr_t)data & 15) == 0) ? 1 : 0;
        kern<<<(unsigned)blocks, tpb, small_smem, st>>>((T *)data, num_arrays, cp.plan, stride, magic, vec_ok, run_seed,
                                                        base, words32, gen);
        CK(cudaGetLastError());
        g_kernel = std::string("shuffle_small_kernel<u") + std::to_string(8 * sizeof(T)) + ">";
        return BR_OK;
    }
    // closed-form resolution (shuffle_resolve_kernel): the single-array stream calls, where one
    // CTA's latency is the whole call and it needs ~10 barriers instead of 5 per 128 steps;
    // for many arrays the hashed groups win, so there only on request
    const bool res_fit = n <= 65535 && resolve_smem_bytes<T>((uint32_t)n) <= MID_SMEM_MAX;
    if (res_fit && (forced_kernel() == K_RESOLVE || (!segmented && forced_kernel() == K_ANY))) {
        const size_t rsmem = resolve_smem_bytes<T>((uint32_t)n);
        const void *kp;
        int threads;
        if (segmented) {
            kp = gen == 2 ? (const void *)shuffle_resolve_kernel<T, RES_W, 1> : (const void *)shuffle_resolve_kernel<T, RES_W, 0>;
            threads = 32 * RES_W;
        } else {
            kp = (const void *)shuffle_resolve_kernel<T, RES_WS, 2>;
            threads = 32 * RES_WS;
        }
        CK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem));
        int grid = segmented ? grid_for(di, kp, threads, rsmem, num_arrays) : 1;
        int use_tma = (((uintptr_t)data | (n * sizeof(T))) & 15) == 0 ? 1 : 0;
        int seg = segmented ? 1 : 0;
        T *dp = (T *)data;
        DevPlan plan = cp.plan;
        void *args[] = {&dp, &num_arrays, &plan, &run_seed, &base, &words32, &state_dev, &words64, &rk_first, &use_tma,
                        &seg, &gen};
        CK(cudaLaunchKernel(kp, dim3(grid), dim3(threads), args, rsmem, st));
        g_kernel = std::string("shuffle_resolve_kernel<u") + std::to_string(8 * sizeof(T)) + "," +
                   std::to_string(threads / 32) + ">";
        return BR_OK;
    }
    const uint32_t zbytes = (uint32_t)((n * sizeof(T) + 15) & ~(uint64_t)15);
    // one warp per array (warp_shuffle.cuh): the default for many arrays of up to 16 KB
    // (12 arrays per SM; C4 1.93 vs 2.49 ms for the hash kernel).  Beyond that too few
    // arrays fit per SM and the CTA groups of the hash kernel win.
    // u16 index permutations, one CTA of NW warps per SM sharing staging buffers
    // (warp_shuffle.cuh shuffle_idx_kernel).  By default when that gives at least 12 arrays
    // per SM and 1.5x the warp kernel's (C4: 20 vs 12 arrays per SM, 1.84 vs 1.93 ms; u64[4096]:
    // 17 per SM, 1.19 ms vs 1.59 for the hash kernel); DESIGN.md section 4.
    if ((forced_kernel() == K_IDX || forced_kernel() == K_ANY) && cp.plan.brec && segmented && n <= 65536 &&
        (uint64_t)cp.plan.max_k * 32 + 64 <= WRING) {
        const int cm = gen == 2 ? 1 : 0;
        const void *kp = gen == 2 ? (const void *)shuffle_idx_kernel<T, 1> : (const void *)shuffle_idx_kernel<T, 0>;
        int dev = 0, optin = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        const int nstage = idx_stages();
        const size_t selems = (n + 3) & ~(uint64_t)3;
        const size_t sbytes = (selems * sizeof(T) + 15) & ~(size_t)15;
        const size_t per_warp = ((2 * n + 15) & ~(uint64_t)15) + idx_warp_fixed(cm);
        const size_t fixed = (size_t)nstage * sbytes + IDX_CTL_BYTES;
        if ((size_t)optin > fixed + per_warp) {
            int nw = (int)std::min<size_t>(24, ((size_t)optin - fixed) / per_warp);
            // arrays per SM the one-warp-per-array kernel would hold (0: not eligible)
            const size_t zb = (n * sizeof(T) + 15) & ~(uint64_t)15;
            const int warp_chains = zb <= WARP_SMEM_DEFAULT ? (int)std::min<size_t>(32, (size_t)optin / (zb + 2656)) : 0;
            // arrays per SM of the hash kernel (one CTA per array, payload + tables + reserve)
            const size_t hash_cta = zb + sizeof(LargeShared<T, CTA_W, uint16_t, CRING, HASH_HB>) + 1024;
            const int hash_ctas = (int)((size_t)optin / hash_cta);
            // measured (idx vs the alternative, arrays per SM and ms): u32[4096] 20 vs 12 (warp),
            // 1.46 vs 1.52; u32[8192] 9 vs 6 (hash), 1.30 vs 1.45; u32[9000] 8 vs 4, 0.74 vs 0.95;
            // u32[10000] 7 vs 4, 0.93 vs 1.05; u32[12000] 5 vs 3, 1.61 vs 1.55; u64[8192] 5 vs 3,
            // 1.19 vs 1.60 (the hash kernel holds 8-byte payloads, the index kernel u16 indices)
            const bool pick = forced_kernel() == K_IDX || (nw >= 12 && 2 * nw >= 3 * warp_chains) ||
                              (zb > WARP_SMEM_DEFAULT && (nw >= 6 || sizeof(T) == 8) && 2 * nw >= 3 * hash_ctas);
            const int64_t need = (num_arrays + di.sms - 1) / di.sms;  // warps per SM that have work
            if (need < nw) nw = (int)std::max<int64_t>(1, need);
            if (pick) {
                const size_t smem = fixed + (size_t)nw * per_warp;
                CK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                const int64_t ctas = (num_arrays + nw - 1) / nw;
                const int grid = (int)std::min<int64_t>(ctas, di.sms);
                int use_tma = (((uintptr_t)data | (n * sizeof(T))) & 15) == 0 ? 1 : 0;
                if (const char *he = getenv("BR_IDX_HOLD_US")) use_tma |= std::min(1000, std::max(0, atoi(he))) << 8;  // test knob
                T *dp = (T *)data;
                DevPlan plan = cp.plan;
                int ns = nstage;
                void *args[] = {&dp, &num_arrays, &plan, &run_seed, &base, &words32, (void *)&use_tma, &gen, &ns};
                CK(cudaLaunchKernel(kp, dim3(grid), dim3(32 * nw), args, smem, st));
                g_kernel = std::string("shuffle_idx_kernel<u") + std::to_string(8 * sizeof(T)) + "," + std::to_string(nw) +
                           ">";
                return BR_OK;
            }
        }
    }
    const bool warp_fit = cp.plan.brec && segmented && zbytes <= WARP_SMEM_MAX &&
                          (uint64_t)cp.plan.max_k * 32 + 64 <= WRING;
    if (warp_fit && (forced_kernel() == K_WARP || (forced_kernel() == K_ANY && zbytes <= WARP_SMEM_DEFAULT))) {
        auto kern = gen == 2 ? shuffle_warp_kernel<T, true, 1> : shuffle_warp_kernel<T, true, 0>;
        const void *kp = (const void *)kern;
        CK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zbytes));
        const int grid = grid_for(di, kp, 32, zbytes, num_arrays);
        const int use_tma = (((uintptr_t)data | (n * sizeof(T))) & 15) == 0 ? 1 : 0;
        kern<<<grid, 32, zbytes, st>>>((T *)data, num_arrays, cp.plan, run_seed, base, words32, state_dev, words64,
                                       rk_first, use_tma, gen);
        CK(cudaGetLastError());
        g_kernel = std::string("shuffle_warp_kernel<u") + std::to_string(8 * sizeof(T)) + ">";
        return BR_OK;
    }
    const uint32_t hbytes = (uint32_t)((n + 15) & ~(uint64_t)15);  // lane-id table indexed by target
    const size_t smem = (size_t)zbytes + hbytes;
    const size_t csmem = (size_t)zbytes;  // payload only; the rest is static
    if (allow(K_HASH) && n < 65536 && csmem <= MID_SMEM_MAX &&
        (uint64_t)cp.plan.max_k * 32 * CTA_W + 32 * CTA_W <= CRING) {
        constexpr int W = CTA_W;
        auto kern = !segmented ? shuffle_cta_hash_kernel<T, W, 2>
                               : (gen == 2 ? shuffle_cta_hash_kernel<T, W, 1> : shuffle_cta_hash_kernel<T, W, 0>);
        const void *kp = (const void *)kern;
        CK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
        int grid = segmented ? grid_for(di, kp, 32 * W, csmem, num_arrays) : 1;
        const int use_tma = (((uintptr_t)data | (n * sizeof(T))) & 15) == 0 ? 1 : 0;
        kern<<<grid, 32 * W, csmem, st>>>((T *)data, num_arrays, cp.plan, run_seed, base, words32, state_dev, words64,
                                          rk_first, use_tma, segmented ? 1 : 0, gen);
        CK(cudaGetLastError());
        g_kernel = std::string("shuffle_cta_hash_kernel<u") + std::to_string(8 * sizeof(T)) + "," +
                   std::to_string(W) + ">";
        return BR_OK;
    }
    if (allow(K_MID) && n <= 65536 && smem <= MID_SMEM_MAX && cp.plan.max_k <= 30) {
        auto kern = !segmented ? shuffle_mid_kernel<T, false, 2>
                               : (gen == 2 ? shuffle_mid_kernel<T, true, 1> : shuffle_mid_kernel<T, true, 0>);
        const void *kp = (const void *)kern;
        CK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int grid = segmented ? grid_for(di, kp, 32, smem, num_arrays) : 1;
        const int use_tma = (((uintptr_t)data | (n * sizeof(T))) & 15) == 0 ? 1 : 0;
        kern<<<grid, 32, smem, st>>>((T *)data, num_arrays, cp.plan, zbytes, run_seed, base, words32, state_dev,
                                     words64, rk_first, use_tma, gen);
        CK(cudaGetLastError());
        g_kernel = std::string("shuffle_mid_kernel<u") + std::to_string(8 * sizeof(T)) + ">";
        return BR_OK;
    }
    // many arrays beyond shared memory: the stage pipeline (stage_shuffle.cuh), one CTA per
    // array, every random access in shared memory.  PCG64/Lehmer streams, full plans, n <= 2^20
    // (C5: 9.2 ms against 12.2 for the CTA-group kernel on the array in global memory).
    const bool sp_fit = segmented && gen != 2 && cp.plan.lo <= 1 && n > 1 && n <= (uint64_t)SP_MAXNB * SP_B &&
                        cp.plan.max_k <= 8;
    if (sp_fit && (forced_kernel() == K_STAGE || forced_kernel() == K_ANY)) {
        const size_t smem = sizeof(SpShared<T>);
        const void *kp = (const void *)shuffle_stage_kernel<T>;
        CK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int grid = grid_for(di, kp, SP_T, smem, num_arrays);
        const size_t cta = sp_cta_bytes((uint32_t)n);
        const uint32_t vstride = (uint32_t)((n + 7) & ~(uint64_t)7);  // 16-byte aligned areas
        const size_t per_array = (size_t)vstride * (sizeof(T) + 2) + 4;
        // arrays per launch pair: every CTA busy, value areas of at most ~4 GB
        const int64_t chunk = std::min<int64_t>(num_arrays, std::max<int64_t>(grid, (int64_t)((4ull << 30) / per_array)));
        const size_t cta_total = (cta * (size_t)grid + 255) & ~(size_t)255;
        const size_t val_bytes = ((size_t)chunk * vstride * sizeof(T) + 255) & ~(size_t)255;
        const size_t slot_bytes = ((size_t)chunk * vstride * 2 + 255) & ~(size_t)255;
        unsigned char *scratch = nullptr;
        CK(cudaMallocAsync((void **)&scratch, cta_total + val_bytes + slot_bytes + (size_t)chunk * 4, st));
        T *val = (T *)(scratch + cta_total);
        uint16_t *slot = (uint16_t *)(scratch + cta_total + val_bytes);
        uint32_t *flags = (uint32_t *)(scratch + cta_total + val_bytes + slot_bytes);
        const int use_tma = (((uintptr_t)data | (n * sizeof(T))) & 15) == 0 && !getenv("BR_SP_NOTMA") ? 1 : 0;
        const void *gk = (const void *)shuffle_stage_gather_kernel<T>;
        const int ggrid = grid_for(di, gk, SPG_T, 0, chunk * (int64_t)((n + SP_B - 1) / SP_B));
        // flagged arrays (a tile larger than a chunk) are re-shuffled from their untouched payload
        constexpr int LW = LARGE_W;
        const void *fk = (const void *)shuffle_cta_large_kernel<T, LW, 0>;  // PCG64 and Lehmer
        const size_t fsmem = large_smem_bytes<T, LW>(false);
        CK(cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem));
        cudaError_t le = cudaSuccess;
#ifdef SP_CHECK
        if (getenv("BR_SP_STOP")) {
            int v = atoi(getenv("BR_SP_STOP")), ph = getenv("BR_SP_PHASE") ? atoi(getenv("BR_SP_PHASE")) : 99;
            cudaMemcpyToSymbol(g_sp_stop, &v, 4);
            cudaMemcpyToSymbol(g_sp_phase, &ph, 4);
        }
#endif
        for (int64_t a0 = 0; a0 < num_arrays && le == cudaSuccess; a0 += chunk) {
            int64_t na = std::min(chunk, num_arrays - a0);
            T *dp = (T *)data + a0 * (int64_t)n;
            DevPlan plan = cp.plan;
            int g = gen;
            size_t cb = cta;
            int64_t b0 = base + a0;
            uint32_t *w32 = words32 ? words32 + a0 : nullptr;
            int tma = use_tma;
            uint32_t vs = vstride;
            le = cudaMemsetAsync(flags, 0, (size_t)na * 4, st);
            void *args[] = {&dp, &na, &plan, &run_seed, &b0, &w32, &g, &scratch, &cb, &val, &slot, &vs, &flags, &tma};
            if (le == cudaSuccess)
                le = cudaLaunchKernel(kp, dim3((unsigned)std::min<int64_t>(grid, na)), dim3(SP_T), args, smem, st);
            const bool dbg = getenv("BR_SP_DEBUG") != nullptr;
            if (dbg && le == cudaSuccess && (le = cudaStreamSynchronize(st)) != cudaSuccess)
                return fail(BR_E_CUDA, std::string("stage kernel: ") + cudaGetErrorString(le));
#ifdef SP_CHECK
            if (dbg) {
                unsigned h[8];
                cudaMemcpyFromSymbol(h, g_sp_dbg, sizeof(h));
                fprintf(stderr, "SP_CHECK line %u: %u %u %08x blk %u\n", h[0], h[1], h[2], h[3], h[4]);
            }
#endif
            if (le == cudaSuccess) {
                uint32_t nn = (uint32_t)n;
                void *gargs[] = {&dp, &na, &nn, &val, &slot, &vs, &flags};
                le = cudaLaunchKernel(gk, dim3(ggrid), dim3(SPG_T), gargs, 0, st);
                if (dbg && le == cudaSuccess && (le = cudaStreamSynchronize(st)) != cudaSuccess)
                    return fail(BR_E_CUDA, std::string("gather kernel: ") + cudaGetErrorString(le));
            }
            if (le == cudaSuccess) {
                uint64_t *nul = nullptr;
                int seg1 = 1;
                const uint32_t *only = flags;
                void *fargs[] = {&dp, &na, &plan, &run_seed, &b0, &w32, &nul, &nul, &nul, &seg1, &g, (void *)&only};
                le = cudaLaunchKernel(fk, dim3((unsigned)std::min<int64_t>(na, (int64_t)di.sms * 8)), dim3(32 * LW),
                                      fargs, fsmem, st);
            }
        }
        CK(cudaFreeAsync(scratch, st));
        if (le != cudaSuccess) return fail(BR_E_CUDA, std::string("stage kernel launch: ") + cudaGetErrorString(le));
        g_kernel = std::string("shuffle_stage_kernel<u") + std::to_string(8 * sizeof(T)) + ">";
        return BR_OK;
    }
    // large arrays: one CTA per array, targets generated in-CTA, array in global memory
    if (allow(K_LARGE) && (uint64_t)cp.plan.max_k * 32 * LARGE_W + 32 * LARGE_W <= large_ring(LARGE_W)) {
        constexpr int W = LARGE_W;
        const int grid = segmented ? (int)std::min<int64_t>(num_arrays, (int64_t)di.sms * 8) : 1;
        auto kern = !segmented ? shuffle_cta_large_kernel<T, W, 2>
                               : (gen == 2 ? shuffle_cta_large_kernel<T, W, 1> : shuffle_cta_large_kernel<T, W, 0>);
        // dynamic shared memory: the CTA's tables and the ChaCha keystream window when there is one
        const size_t wsmem = large_smem_bytes<T, W>(!segmented || gen == 2);
        CK(cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem));
        kern<<<grid, 32 * W, wsmem, st>>>((T *)data, num_arrays, cp.plan, run_seed, base, words32, state_dev, words64,
                                          rk_first, segmented ? 1 : 0, gen, nullptr);
        CK(cudaGetLastError());
        g_kernel = std::string("shuffle_cta_large_kernel<u") + std::to_string(8 * sizeof(T)) + "," +
                   std::to_string(W) + ">";
        return BR_OK;
    }
    // large arrays, exotic schedules: targets (u32 per position) into scratch, then warp-group apply
    {
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(num_arrays, (int64_t)((1ull << 31) / (n * 4))));
        uint32_t *J = nullptr;
        CK(cudaMallocAsync((void **)&J, (size_t)chunk * n * sizeof(uint32_t), st));
        for (int64_t a0 = 0; a0 < num_arrays; a0 += chunk) {
            const int64_t na = std::min(chunk, num_arrays - a0);
            const int grid_gen = (int)std::min<int64_t>(na, (int64_t)di.sms * 16);
            if (segmented) {
                auto kern = gen == 2 ? shuffle_large_gen_kernel<true, 1> : shuffle_large_gen_kernel<true, 0>;
                kern<<<grid_gen, 32, 0, st>>>(na, cp.plan, run_seed, base + a0, J, words32 ? words32 + a0 : nullptr,
                                              state_dev, words64, rk_first, gen);
            } else {
                shuffle_large_gen_kernel<false, 2><<<1, 32, 0, st>>>(1, cp.plan, run_seed, base, J, nullptr,
                                                                      state_dev, words64, rk_first, gen);
            }
            const uint32_t lim = cp.plan.lo > 1 ? cp.plan.lo : 1;
            shuffle_large_apply_kernel<T><<<(int)std::min<int64_t>(na, (int64_t)di.sms * 16), 32, 0, st>>>(
                (T *)data + a0 * (int64_t)n, na, (uint32_t)n, lim, J);
            CK(cudaGetLastError());
        }
        CK(cudaFreeAsync(J, st));
        g_kernel = std::string("shuffle_large_gen_kernel+shuffle_large_apply_kernel<u") + std::to_string(8 * sizeof(T)) +
                   ">";
        return BR_OK;
    }
}

int shuffle_common(void *data, int eb, int64_t num_arrays, uint64_t n, const std::vector<br_segment> &segs,
                   bool segmented, uint64_t run_seed, int64_t base, uint32_t *words32, br_pcg64 *state_dev,
                   uint64_t *words64, uint64_t *rk_first, int gen, void *stream, bool naive = false) {
    if (gen < 0 || gen > 2) return fail(BR_E_UNSUPPORTED, "generator must be 0 (pcg64), 1 (lehmer) or 2 (chacha)");
    if (eb != 4 && eb != 8) return fail(BR_E_UNSUPPORTED, "elem_bytes must be 4 or 8");
    if (num_arrays < 0) return fail(BR_E_INVALID, "num_arrays < 0");
    int dev;
    DeviceInfo di;
    int stt = ensure_device(&dev, &di);
    if (stt) return stt;
    cudaStream_t st = (cudaStream_t)stream;
    // arrays of 2^32 or more elements (shuffle.py:175-190): the single-roll head above
    // 2^32 - 1 runs in shuffle_head64_kernel on the stream, the rest below it continues here
    // (BR_HEAD64_STOP lowers the split for tests on small arrays)
    uint64_t hstop = (1ull << 32) - 1;
    if (const char *e = getenv("BR_HEAD64_STOP")) hstop = std::min<uint64_t>(hstop, strtoull(e, nullptr, 10));
    if (n > hstop && !naive && hstop >= 1) {
        if (segmented) return fail(BR_E_UNSUPPORTED, "segmented arrays of 2^32 or more elements (shuffle each through the stream form)");
        if (segs.empty() || segs[0].k != 1 || segs[0].start_n != n || segs[0].count < n - hstop)
            return fail(BR_E_UNSUPPORTED, "arrays of 2^32 or more elements need single rolls above 2^32 - 1");
        if (!data) return fail(BR_E_INVALID, "null data pointer");
        if (!state_dev) return fail(BR_E_INVALID, "null state pointer");
        std::vector<br_segment> rest(segs);
        rest[0].start_n = hstop;
        rest[0].count -= n - hstop;
        if (rest[0].count == 0) rest.erase(rest.begin());
        uint64_t *hw = nullptr;
        CK(cudaMallocAsync((void **)&hw, sizeof(uint64_t), st));
        if (eb == 4)
            shuffle_head64_kernel<uint32_t><<<1, H64_T, 0, st>>>((uint32_t *)data, n, hstop, (uint64_t *)state_dev, hw,
                                                                 rk_first);
        else
            shuffle_head64_kernel<uint64_t><<<1, H64_T, 0, st>>>((uint64_t *)data, n, hstop, (uint64_t *)state_dev, hw,
                                                                 rk_first);
        cudaError_t le = cudaGetLastError();
        int r = le == cudaSuccess ? BR_OK : fail(BR_E_CUDA, std::string("head kernel: ") + cudaGetErrorString(le));
        if (r == BR_OK) {
            r = shuffle_common(data, eb, 1, hstop, rest, false, 0, 0, nullptr, state_dev, words64, nullptr, gen, stream,
                               false);
            const std::string rest_kernel = g_kernel;
            if (r == BR_OK && words64) add_words_kernel<<<1, 1, 0, st>>>(words64, hw);
            g_kernel = "shuffle_head64_kernel+" + rest_kernel;
        }
        cudaFreeAsync(hw, st);
        return r;
    }
    if (n >= (1ull << 32)) {
        if (naive && n > (1ull << 32)) return fail(BR_E_BOUND_OVERFLOW, "pair product exceeds 2**64");
        return fail(BR_E_UNSUPPORTED, "arrays of 2^32 or more elements");
    }
    if (segs.empty() || num_arrays == 0) {  // n < 2: nothing to do, no words consumed
        if (segmented && words32 && num_arrays > 0) CK(cudaMemsetAsync(words32, 0, num_arrays * sizeof(uint32_t), st));
        if (!segmented && words64) CK(cudaMemsetAsync(words64, 0, sizeof(uint64_t), st));
        g_kernel = "none";
        return BR_OK;
    }
    if (!data) return fail(BR_E_INVALID, "null data pointer");
    if (!segmented && !state_dev) return fail(BR_E_INVALID, "null state pointer");
    PlanRef cp;
    stt = get_plan(n, segs, naive, st, &cp);
    if (stt) return stt;
    const int r = eb == 4 ? launch_shuffle<uint32_t>(data, num_arrays, n, *cp, segmented, run_seed, base, words32,
                                                     (uint64_t *)state_dev, words64, rk_first, gen, di, st)
                          : launch_shuffle<uint64_t>(data, num_arrays, n, *cp, segmented, run_seed, base, words32,
                                                     (uint64_t *)state_dev, words64, rk_first, gen, di, st);
    cp->used(st);  // the plan outlives every kernel queued above (stream-ordered free)
    return r;
}

}  // namespace

extern "C" {

int br_abi_version(void) { return BR_ABI_VERSION; }
const char *br_last_error(void) { return g_err.c_str(); }
const char *br_last_kernel(void) { return g_kernel.c_str(); }

int br_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

uint64_t br_splitmix64_next(uint64_t *x) { return splitmix64_next(*x); }

void br_pcg64_seed(uint64_t seed, br_pcg64 *out) {
    u128 s, inc;
    pcg_seed(seed, s, inc);
    out->state_hi = s.hi;
    out->state_lo = s.lo;
    out->inc_hi = inc.hi;
    out->inc_lo = inc.lo;
}

void br_lehmer_seed(uint64_t seed, br_pcg64 *out) {
    u128 s, inc;
    lehmer_seed(seed, s, inc);
    out->state_hi = s.hi;
    out->state_lo = s.lo;
    out->inc_hi = inc.hi;
    out->inc_lo = inc.lo;
}

void br_chacha_seed(uint64_t seed, br_chacha *out) {
    ChaKey K;
    chacha_seed(seed, K);
    out->head.state_hi = 0;
    out->head.state_lo = 0;
    out->head.inc_hi = K.nonce;
    out->head.inc_lo = CHACHA_TAG;
    for (int i = 0; i < 8; ++i) out->key[i] = K.k[i];
}

int br_words_state(const uint64_t *words_dev, uint64_t nwords, br_chacha *out) {
    if (!out || (nwords && !words_dev)) return fail(BR_E_INVALID, "null words");
    memset(out, 0, sizeof *out);
    out->head.inc_hi = nwords;
    out->head.inc_lo = WORDS_TAG;
    const uint64_t addr = reinterpret_cast<uint64_t>(words_dev);
    memcpy(out->key, &addr, sizeof addr);
    return BR_OK;
}

uint64_t br_pcg64_next(br_pcg64 *st) {
    if (st->inc_lo == WORDS_TAG) {  // one replayed word, read back from the device
        const uint64_t p = st->state_lo;
        st->state_lo = p + 1;
        if (p >= st->inc_hi || st->state_hi) return ~0ull;  // past the end: as on the device
        uint64_t w = 0;
        cudaMemcpy(&w, host_cha_key(st).words + p, sizeof w, cudaMemcpyDeviceToHost);
        return w;
    }
    if (host_is_chacha(st)) {
        const u128 s = add128(mk128(st->state_hi, st->state_lo), mk128(0, 1));
        st->state_hi = s.hi;
        st->state_lo = s.lo;
        return cha_out(host_cha_key(st), s);
    }
    u128 s = mk128(st->state_hi, st->state_lo);
    const bool lh = (st->inc_hi | st->inc_lo) == 0;
    s = add128(mul128(s, lh ? mk128(0, LEHMER_MULT) : mk128(PCG_MULT_HI, PCG_MULT_LO)), mk128(st->inc_hi, st->inc_lo));
    st->state_hi = s.hi;
    st->state_lo = s.lo;
    return lh ? s.hi : xslrr(s);
}

void br_pcg64_advance(br_pcg64 *st, uint64_t delta) {
    if (host_is_chacha(st)) {
        const u128 s = add128(mk128(st->state_hi, st->state_lo), mk128(0, delta));
        st->state_hi = s.hi;
        st->state_lo = s.lo;
        return;
    }
    const JumpTables &t = host_tables();
    u128 s = mk128(st->state_hi, st->state_lo), inc = mk128(st->inc_hi, st->inc_lo);
    const bool lh = (inc.hi | inc.lo) == 0;
    for (int k = 0; delta; ++k, delta >>= 1)
        if (delta & 1) s = add128(mul128(lh ? t.LA[k] : t.A[k], s), mul128(t.G[k], inc));
    st->state_hi = s.hi;
    st->state_lo = s.lo;
}

uint64_t br_array_seed(uint64_t run_seed, uint64_t a) { return array_seed(run_seed, a); }

int br_falling_factorial(uint64_t n, uint32_t k, uint64_t *lo, uint64_t *hi) {
    h128 v;
    int st = ff_checked(n, k, &v);
    if (st) return fail(st, st == BR_E_INVALID ? "need 0 <= k <= n" : "falling factorial exceeds 2**64");
    *lo = (uint64_t)v;
    *hi = (uint64_t)(v >> 64);
    return BR_OK;
}

int br_schedule_validate(const br_regime *e, int ne, uint32_t max_batch, int word_bits) {
    if (word_bits != 64) return fail(BR_E_UNSUPPORTED, "device path supports 64-bit words only");
    if (ne < 1 || !e) return fail(BR_E_INVALID, "schedule needs at least one regime");
    for (int i = 0; i + 1 < ne; ++i) {
        if (e[i].max_length <= e[i + 1].max_length) return fail(BR_E_INVALID, "regime lengths must strictly decrease");
        if (e[i].batch_size >= e[i + 1].batch_size) return fail(BR_E_INVALID, "batch sizes must strictly increase");
    }
    if (e[ne - 1].batch_size != max_batch) return fail(BR_E_INVALID, "last batch size != max_batch");
    for (int i = 0; i < ne; ++i) {
        if ((uint64_t)e[i].batch_size > e[i].max_length) return fail(BR_E_INVALID, "batch size exceeds regime length");
        h128 f;
        int st = ff_checked(e[i].max_length, e[i].batch_size, &f);
        if (st) return fail(st, "regime product exceeds 2**64");
    }
    return BR_OK;
}

int64_t br_plan_build(uint64_t n, const br_regime *entries, int n_entries, br_segment *out, int64_t cap,
                      uint64_t *n_batches_out) {
    std::vector<br_segment> segs;
    uint64_t nb = 0;
    int st = build_segments(n, entries, n_entries, segs, nb);
    if (st) return -st;
    for (int64_t i = 0; i < (int64_t)segs.size() && i < cap; ++i) out[i] = segs[i];
    if (n_batches_out) *n_batches_out = nb;
    return (int64_t)segs.size();
}

int br_pcg64_fill(uint64_t *out_dev, int64_t count, const br_pcg64 *st, uint64_t offset, void *stream) {
    if (count < 0 || !st) return fail(BR_E_INVALID, "bad arguments");
    int dev;
    DeviceInfo di;
    int s = ensure_device(&dev, &di);
    if (s) return s;
    if (count == 0) return BR_OK;
    if (!out_dev) return fail(BR_E_INVALID, "null output");
    if (host_is_chacha(st)) {
        const u128 p0 = add128(mk128(st->state_hi, st->state_lo), mk128(0, offset));
        const int64_t nblk = (int64_t)((p0.lo & 7) + (uint64_t)count + 7) >> 3;
        int grid = grid_for(di, (const void *)cha_fill_kernel, 256, 0, (nblk + 255) / 256);
        cha_fill_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(out_dev, count, host_cha_key(st), p0);
        CK(cudaGetLastError());
        g_kernel = "cha_fill_kernel";
        return BR_OK;
    }
    int64_t blocks = (count + 256 * 32 - 1) / (256 * 32);
    int grid = grid_for(di, (const void *)pcg_fill_kernel, 256, 0, blocks);
    pcg_fill_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(out_dev, count, mk128(st->state_hi, st->state_lo),
                                                             mk128(st->inc_hi, st->inc_lo), offset);
    CK(cudaGetLastError());
    g_kernel = "pcg_fill_kernel";
    return BR_OK;
}

int br_state_upload(br_pcg64 *state_dev, const br_pcg64 *st, void *stream) {
    if (!state_dev || !st) return fail(BR_E_INVALID, "null state");
    const size_t bytes = host_is_chacha(st) ? sizeof(br_chacha) : sizeof(br_pcg64);
    // through a per-thread ring of pinned 64-byte slots: the copy is a true async DMA (a
    // pageable source would make the driver wait for the stream) and the caller's struct may
    // go away at once.  A slot is reused only after the event of its previous copy (a host
    // wait only if 64 uploads are still queued)
    struct Ring {
        br_chacha *slots = nullptr;
        cudaEvent_t ev[64] = {};
        int dev[64];
        unsigned next = 0;
    };
    thread_local Ring ring;
    if (!ring.slots) CK(cudaHostAlloc((void **)&ring.slots, 64 * sizeof(br_chacha), cudaHostAllocPortable));
    const unsigned i = ring.next++ & 63u;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (ring.ev[i]) {
        CK(cudaEventSynchronize(ring.ev[i]));
        if (ring.dev[i] != dev) {  // events belong to a device
            cudaEventDestroy(ring.ev[i]);
            ring.ev[i] = nullptr;
        }
    }
    if (!ring.ev[i]) CK(cudaEventCreateWithFlags(&ring.ev[i], cudaEventDisableTiming));
    ring.dev[i] = dev;
    memcpy(&ring.slots[i], st, bytes);
    CK(cudaMemcpyAsync(state_dev, &ring.slots[i], bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
    CK(cudaEventRecord(ring.ev[i], (cudaStream_t)stream));
    note_state_kind(state_dev, host_is_chacha(st));
    return BR_OK;
}

int br_state_download(br_pcg64 *st, const br_pcg64 *state_dev, void *stream) {
    if (!state_dev || !st) return fail(BR_E_INVALID, "null state");
    CK(cudaMemcpyAsync(st, state_dev, sizeof(br_pcg64), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    return BR_OK;
}

size_t br_roll_workspace_bytes(void) { return sizeof(RollWs); }

int br_roll_batches(const uint32_t *bounds, int k, int64_t nb, br_pcg64 *state_dev, uint32_t *rolls,
                    uint8_t *words, uint8_t *flags, uint64_t *final_rk, void *ws, void *stream) {
    return br_roll_batches_phase(bounds, k, nb, state_dev, rolls, words, flags, final_rk, ws, 3, stream);
}

static int roll_batches_impl(const uint32_t *bounds, int k, int64_t nb, br_pcg64 *state_dev, uint32_t *rolls,
                      uint8_t *words, uint8_t *flags, uint64_t *final_rk, void *ws, int phase, int naive,
                      void *stream) {
    if (phase < 1 || phase > 3) return fail(BR_E_INVALID, "phase must be 1, 2 or 3");
    if (nb < 0) return fail(BR_E_INVALID, "num_batches < 0");
    if (k < 1) return fail(BR_E_INVALID, "at least one base is required");
    if (k > 8) return fail(BR_E_UNSUPPORTED, "batches of more than 8 dice are not supported on the device path");
    int dev;
    DeviceInfo di;
    int s = ensure_device(&dev, &di);
    if (s) return s;
    if (nb == 0) {
        g_kernel = "none";
        return BR_OK;
    }
    if (!bounds || !state_dev || !rolls || !words || !ws) return fail(BR_E_INVALID, "null pointer argument");
    if ((((uintptr_t)bounds | (uintptr_t)rolls) & 15) != 0) return fail(BR_E_INVALID, "bounds/rolls must be 16-byte aligned");
    // the fast kernels store words in 8-byte vectors and final remainders as u64: a misaligned
    // pointer would fault (a sticky error) instead of raising
    if ((((uintptr_t)words | (uintptr_t)final_rk) & 7) != 0)
        return fail(BR_E_INVALID, "words/final_remainder must be 8-byte aligned");
    if (!di.coop) return fail(BR_E_CUDA, "device lacks cooperative launch");
    RollArgs a;
    a.bounds = bounds;
    a.k = k;
    a.nb = nb;
    a.state = (uint64_t *)state_dev;
    a.rolls = rolls;
    a.words = words;
    a.flags = flags;
    a.rk = final_rk;
    a.ws = (RollWs *)ws;
    a.naive = naive;
    cudaStream_t st = (cudaStream_t)stream;
    switch (k) {
        case 1: return launch_roll<1>(a, di, st, phase);
        case 2: return launch_roll<2>(a, di, st, phase);
        case 3: return launch_roll<3>(a, di, st, phase);
        case 4: return launch_roll<4>(a, di, st, phase);
        case 5: return launch_roll<5>(a, di, st, phase);
        case 6: return launch_roll<6>(a, di, st, phase);
        case 7: return launch_roll<7>(a, di, st, phase);
        default: return launch_roll<8>(a, di, st, phase);
    }
}

int br_roll_batches_phase(const uint32_t *bounds, int k, int64_t nb, br_pcg64 *state_dev, uint32_t *rolls,
                          uint8_t *words, uint8_t *flags, uint64_t *final_rk, void *ws, int phase, void *stream) {
    return roll_batches_impl(bounds, k, nb, state_dev, rolls, words, flags, final_rk, ws, phase, 0, stream);
}

int br_roll_batches_naive(const uint32_t *bounds, int k, int64_t nb, br_pcg64 *state_dev, uint32_t *rolls,
                          uint8_t *words, uint8_t *flags, uint64_t *final_rk, void *ws, void *stream) {
    return roll_batches_impl(bounds, k, nb, state_dev, rolls, words, flags, final_rk, ws, 3, 1, stream);
}

int br_roll_check(void *ws, void *stream, uint64_t *extra_words) {
    if (!ws) return fail(BR_E_INVALID, "null workspace");
    RollWs h;  // the header only (the fixup's per-warp records are scratch)
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    CK(cudaMemcpy(&h, ws, offsetof(RollWs, rec), cudaMemcpyDeviceToHost));
    if (extra_words) *extra_words = h.extra;
    if (h.error) {
        unsigned zero = 0;
        CK(cudaMemcpy((char *)ws + offsetof(RollWs, error), &zero, sizeof(zero), cudaMemcpyHostToDevice));
        return fail((int)h.error, h.error == BR_E_INVALID ? "bases must be positive" : "product of bounds exceeds 2**64");
    }
    return BR_OK;
}

int br_digit_pass(const uint64_t *words, const uint32_t *bounds, int k, int64_t count, uint32_t *digits, uint64_t *rk,
                  void *stream) {
    if (k < 1 || count < 0) return fail(BR_E_INVALID, "bad arguments");
    int dev;
    DeviceInfo di;
    int s = ensure_device(&dev, &di);
    if (s) return s;
    if (count == 0) return BR_OK;
    if (!words || !bounds || !digits) return fail(BR_E_INVALID, "null pointer argument");
    int64_t blocks = (count + 255) / 256;
    int grid = grid_for(di, (const void *)digit_pass_kernel, 256, 0, blocks);
    digit_pass_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(words, bounds, k, count, digits, rk);
    CK(cudaGetLastError());
    g_kernel = "digit_pass_kernel";
    return BR_OK;
}

int br_roll_batch64(const uint64_t *bases_dev, int k, br_pcg64 *state_dev, const uint64_t *r0_dev,
                    uint64_t *out_dev, void *stream) {
    if (k < 1 || k > 64) return fail(BR_E_INVALID, "1 <= k <= 64 bases");
    if (!bases_dev || !out_dev || (!state_dev && !r0_dev)) return fail(BR_E_INVALID, "null pointer argument");
    int dev;
    DeviceInfo di;
    int s = ensure_device(&dev, &di);
    if (s) return s;
    std::vector<uint64_t> b(k);
    CK(cudaMemcpyAsync(b.data(), bases_dev, k * sizeof(uint64_t), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    h128 prod = 1;
    for (int m = 0; m < k; ++m) {  // mixed_radix.py:28-35: product <= 2^64 (a 0 here encodes 2^64)
        prod *= b[m] ? (h128)b[m] : ((h128)1 << 64);
        if (prod > ((h128)1 << 64)) return fail(BR_E_BOUND_OVERFLOW, "product of the bases exceeds 2^64");
    }
    const int full = prod == ((h128)1 << 64) ? 1 : 0;
    roll_one64_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(bases_dev, k, (uint64_t)prod, full, (uint64_t *)state_dev,
                                                          r0_dev, out_dev);
    CK(cudaGetLastError());
    g_kernel = "roll_one64_kernel";
    return BR_OK;
}

int br_shuffle_stream(void *z, int eb, uint64_t n, br_pcg64 *state_dev, const br_regime *entries, int ne,
                      int unbatched, uint64_t *words_dev, void *stream) {
    std::vector<br_segment> segs;
    uint64_t nb = 0;
    if (unbatched) {
        if (n >= 2) {
            br_segment s;
            s.start_n = n;
            s.k = 1;
            s.reserved = 0;
            s.count = n - 1;
            segs.push_back(s);
        }
    } else {
        int st = build_segments(n, entries, ne, segs, nb);
        if (st) return st;
    }
    return shuffle_common(z, eb, 1, n, segs, false, 0, 0, nullptr, state_dev, words_dev, nullptr, 0, stream);
}

int br_shuffle_stream_segments(void *z, int eb, uint64_t n, br_pcg64 *state_dev, const br_segment *segs, int nseg,
                               uint64_t *words_dev, uint64_t *rk_first_dev, void *stream) {
    if (nseg < 0 || (nseg > 0 && !segs)) return fail(BR_E_INVALID, "bad segment list");
    std::vector<br_segment> v(segs, segs + nseg);
    for (const br_segment &s : v) {
        if (s.k < 1 || s.count < 1) return fail(BR_E_INVALID, "segment with k < 1 or count < 1");
        if (s.start_n > n || (uint64_t)s.k * s.count > s.start_n)
            return fail(BR_E_INVALID, "segment runs outside the array");
    }
    return shuffle_common(z, eb, 1, n, v, false, 0, 0, nullptr, state_dev, words_dev, rk_first_dev, 0, stream);
}

int br_shuffle_segmented(void *data, int eb, int64_t num_arrays, uint64_t n, uint64_t run_seed, int64_t base,
                         const br_regime *entries, int ne, int generator, uint32_t *words_dev, void *stream) {
    std::vector<br_segment> segs;
    uint64_t nb = 0;
    int st = build_segments(n, entries, ne, segs, nb);
    if (st) return st;
    return shuffle_common(data, eb, num_arrays, n, segs, true, run_seed, base, words_dev, nullptr, nullptr, nullptr,
                          generator, stream);
}

// shuffle.py:228-266 shuffle_naive_batched as a plan: pairs (i, i-1) from the top while
// i >= 2, then a single roll on 2 if index 1 is left.
static void naive_segments(uint64_t n, std::vector<br_segment> &segs) {
    if (n < 2) return;
    br_segment s{};
    s.start_n = n;
    s.k = 2;
    s.count = (n - 1) / 2;
    if (s.count) segs.push_back(s);
    if ((n - 1) & 1) {
        br_segment t{};
        t.start_n = 2;
        t.k = 1;
        t.count = 1;
        segs.push_back(t);
    }
}

int br_shuffle_naive_stream(void *z, int eb, uint64_t n, br_pcg64 *state_dev, uint64_t *words_dev, void *stream) {
    std::vector<br_segment> segs;
    naive_segments(n, segs);
    return shuffle_common(z, eb, 1, n, segs, false, 0, 0, nullptr, state_dev, words_dev, nullptr, 0, stream, true);
}

int br_shuffle_naive_segmented(void *data, int eb, int64_t num_arrays, uint64_t n, uint64_t run_seed, int64_t base,
                               int generator, uint32_t *words_dev, void *stream) {
    std::vector<br_segment> segs;
    naive_segments(n, segs);
    return shuffle_common(data, eb, num_arrays, n, segs, true, run_seed, base, words_dev, nullptr, nullptr, nullptr,
                          generator, stream, true);
}

void br_release(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    PlanCache &pc = plan_cache();
    pc.map.clear();  // each plan is freed (stream-ordered) once no caller holds it
    pc.lru.clear();
    pc.bytes = 0;
}

}  // extern "C"
