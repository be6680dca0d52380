// Microbenchmark: shared-memory bandwidth of B200 (roofline denominator for the smem-staged
// shuffles).  Every warp reads (LDS.32, lanes on consecutive words: conflict-free) and writes
// back its own slice of a 32 KB block buffer; bytes moved = 4 per lane access.  Printed as JSON.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a smem_bw.cu -o smem_bw
#include <cuda_runtime.h>

#include <cstdio>

constexpr int ITERS = 4096;
constexpr int WORDS = 8192;  // 32 KB per block

__global__ void __launch_bounds__(1024) k_lds(unsigned *out, unsigned seed) {
    __shared__ unsigned buf[WORDS];
    for (int i = threadIdx.x; i < WORDS; i += blockDim.x) buf[i] = i * seed;
    __syncthreads();
    volatile unsigned *vb = buf;  // every access is issued
    unsigned acc = 0, idx = threadIdx.x;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        acc += vb[idx];
        idx = (idx + 1024) & (WORDS - 1);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(1024) k_sts(unsigned *out, unsigned seed) {
    __shared__ unsigned buf[WORDS];
    volatile unsigned *vb = buf;
    unsigned idx = threadIdx.x, v = seed + threadIdx.x;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        vb[idx] = v;
        v += 3;
        idx = (idx + 1024) & (WORDS - 1);
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = buf[(threadIdx.x * 7) & (WORDS - 1)];
}

template <typename F>
double run(F kern, unsigned *out, int grid, int threads) {
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
    return (double)grid * threads * ITERS * 4.0 * 5 / (ms * 1e-3) / 1e9;  // GB/s
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int threads = 1024, grid = sms * 2;
    unsigned *out;
    cudaMalloc(&out, (size_t)grid * threads * sizeof(unsigned));
    const double ld = run(k_lds, out, grid, threads);
    const double st = run(k_sts, out, grid, threads);
    if (cudaDeviceSynchronize() != cudaSuccess) return 1;
    printf("{\"device_sms\": %d, \"lds32_gbs\": %.1f, \"sts32_gbs\": %.1f, \"analytic_gbs\": %.1f, \"method\": \"conflict-free "
           "LDS.32 / STS.32 loops, %d x %d threads, 32 KB per block, CUDA events over 5 launches after warm-up; analytic = "
           "SMs x 128 B/clk x max SM clock\"}\n",
           sms, ld, st, sms * 128.0 * clk * 1e3 / 1e9, grid, threads);
    return 0;
}
