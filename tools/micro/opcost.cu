// Microbenchmark: throughput cost of the cost model's operations on B200.
// Every thread runs a dependent chain of one operation; the whole GPU is filled, so the time
// per operation is the machine throughput cost, as the cost model wants it.  Printed as JSON:
//   die          one batched die, (digit, r') = b (x) r            (core.cuh die)
//   pcg64_word   one PCG64 step + XSL-RR output                    (mad128_wide + xslrr)
//   lehmer_word  one Lehmer128 step + top word
//   chacha_word  one ChaCha20 block / 8                            (chacha.cuh)
//   mod64        2^64 mod b for a 64-bit b (the threshold remainder)
//   div64_32     a 64-by-32-bit quotient + remainder (the naive pair split)
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_2408_06213_b200/csrc opcost.cu -o opcost
#include <cuda_runtime.h>

#include <cstdio>

#include "chacha.cuh"
#include "core.cuh"

using namespace br;

constexpr int ITERS = 4096;

__global__ void k_die(uint64_t *out, uint32_t seed) {
    uint64_t r = 0x9E3779B97F4A7C15ull * (threadIdx.x + 1 + blockIdx.x * 977ull + seed);
    uint32_t acc = 0, b = 1000 + threadIdx.x;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        acc += die(b, r);
        b += 3;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ r;
}

__global__ void k_pcg(uint64_t *out, uint32_t seed) {
    u128 s = mk128(seed, threadIdx.x + blockIdx.x * 977ull), inc = mk128(0x5851F42D4C957F2Dull, 0x14057B7EF767814Full);
    const u128 M = mk128(PCG_MULT_HI, PCG_MULT_LO);
    uint64_t acc = 0;
#pragma unroll 8
    for (int i = 0; i < ITERS; ++i) {
        s = mad128_wide(s, M, inc);
        acc += xslrr(s);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_lehmer(uint64_t *out, uint32_t seed) {
    u128 s = mk128(seed, (threadIdx.x + blockIdx.x * 977ull) | 1);
    const u128 M = mk128(0, LEHMER_MULT), Z = mk128(0, 0);
    uint64_t acc = 0;
#pragma unroll 8
    for (int i = 0; i < ITERS; ++i) {
        s = mad128_wide(s, M, Z);
        acc += s.hi;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_chacha(uint64_t *out, uint32_t seed) {
    ChaKey K;
    chacha_seed(seed + threadIdx.x + blockIdx.x * 977ull, K);
    uint32_t acc = 0;
    for (int i = 0; i < ITERS / 8; ++i) {
        uint32_t b[16];
        chacha_block(K, (uint64_t)i, b);
#pragma unroll
        for (int q = 0; q < 16; ++q) acc += b[q];
        K.k[0] ^= acc;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_mod64(uint64_t *out, uint32_t seed) {
    uint64_t p = 0x0123456789ABCDEFull + threadIdx.x * 7919ull + blockIdx.x + seed, acc = 0;
#pragma unroll 4
    for (int i = 0; i < ITERS; ++i) {
        acc += (0 - p) % p;
        p += acc & 0xFFFF;
        p |= 1ull << 40;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_div(uint64_t *out, uint32_t seed) {
    uint64_t v = 0xFEDCBA9876543210ull ^ (threadIdx.x + blockIdx.x * 977ull + seed), acc = 0;
    uint32_t d = 100000 + threadIdx.x;
#pragma unroll 4
    for (int i = 0; i < ITERS; ++i) {
        const uint64_t q = v / d;
        acc += q + (v - q * d);
        v = (v ^ acc) | (1ull << 63);
        d += 2;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// peak of the partial-product instruction itself: 8 independent IMAD.WIDE.U32 chains per thread
__global__ void k_imad_wide(uint64_t *out, uint32_t seed) {
    uint64_t acc[8];
    uint32_t m = 0x9E3779B9u + threadIdx.x + seed;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = (uint64_t)(threadIdx.x + c * 7919u + blockIdx.x);
#pragma unroll 4
    for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = (uint64_t)(uint32_t)acc[c] * m + (acc[c] >> 32);
    }
    uint64_t x = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) x ^= acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

template <typename F>
double run(F kern, uint64_t *out, int grid, int threads, double ops_per_thread) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<grid, threads>>>(out, 1);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) kern<<<grid, threads>>>(out, 2 + r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e6 / 5 / ((double)grid * threads * ops_per_thread);  // ns per op, whole GPU
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 256, grid = sms * 8;
    uint64_t *out;
    cudaMalloc(&out, (size_t)grid * threads * sizeof(uint64_t));
    const double die = run(k_die, out, grid, threads, ITERS);
    const double pcg = run(k_pcg, out, grid, threads, ITERS);
    const double leh = run(k_lehmer, out, grid, threads, ITERS);
    const double cha = run(k_chacha, out, grid, threads, ITERS);  // ITERS/8 blocks = ITERS words
    const double mod = run(k_mod64, out, grid, threads, ITERS);
    const double dv = run(k_div, out, grid, threads, ITERS);
    const double iw = run(k_imad_wide, out, grid, threads, ITERS);  // ITERS/8 x 8 chains
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        fprintf(stderr, "cuda error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    printf("{\"device_sms\": %d, \"grid\": %d, \"threads\": %d, \"ns_per_op\": {\"die\": %.6g, \"pcg64_word\": %.6g, "
           "\"lehmer_word\": %.6g, \"chacha_word\": %.6g, \"mod64\": %.6g, \"div64_32\": %.6g}, "
           "\"in_dice\": {\"pcg64_word\": %.4g, \"lehmer_word\": %.4g, \"chacha_word\": %.4g, \"mod64\": %.4g, "
           "\"div64_32\": %.4g}, \"imad_wide_per_s\": %.6g, \"method\": \"dependent chains on every thread of %d x %d "
           "threads, CUDA events, 5 launches after warm-up; ns per op of the whole GPU; imad_wide_per_s = IMAD.WIDE.U32 "
           "(32x32+64 -> 64) throughput with 8 independent chains per thread\"}\n",
           sms, grid, threads, die, pcg, leh, cha, mod, dv, pcg / die, leh / die, cha / die, mod / die, dv / die,
           1e9 / iw, grid, threads);
    return 0;
}
