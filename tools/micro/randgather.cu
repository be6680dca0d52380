// Microbenchmark: random 8-byte gathers / scatters / atomics over buffers of various sizes
// (L2-resident vs HBM-resident) on one GPU.  Dev tool; informs the large-array design.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__global__ void gather(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, uint64_t nmask, int64_t count, uint32_t salt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t j = ((uint64_t)hash32((uint32_t)i ^ salt) * 2654435761ull + hash32((uint32_t)(i >> 32) + salt)) & nmask;
    dst[i] = src[j];
  }
}
__global__ void scatter(uint64_t* __restrict__ dst, uint64_t nmask, int64_t count, uint32_t salt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t j = ((uint64_t)hash32((uint32_t)i ^ salt) * 2654435761ull) & nmask;
    dst[j] = i;
  }
}
__global__ void amin(uint32_t* __restrict__ dst, uint64_t nmask, int64_t count, uint32_t salt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t j = ((uint64_t)hash32((uint32_t)i ^ salt) * 2654435761ull) & nmask;
    atomicMin(dst + j, (uint32_t)i);
  }
}
// random read-modify-write of one 8-byte element (the access pair of a Fisher-Yates step on
// an HBM-resident array: z[j] is read, then written back)
__global__ void rmw(uint64_t* __restrict__ z, uint64_t nmask, int64_t count, uint32_t salt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t j = ((uint64_t)hash32((uint32_t)i ^ salt) * 2654435761ull + hash32((uint32_t)(i >> 32) + salt)) & nmask;
    z[j] = z[j] + i;
  }
}
__global__ void copy(const uint4* __restrict__ s, uint4* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) d[i] = s[i];
}
int main() {
  const int64_t count = 1 << 27;   // accesses per launch
  uint64_t *src, *dst; uint32_t* am;
  size_t maxbytes = 4ull << 30;
  cudaMalloc(&src, maxbytes); cudaMalloc(&dst, count * 8); cudaMalloc(&am, maxbytes);
  cudaMemset(src, 1, maxbytes); cudaMemset(am, 0xff, maxbytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int grid = 148 * 16, block = 256;
  for (size_t mb : {16, 32, 64, 96, 128, 256, 1024, 2048, 4096}) {
    uint64_t n = (mb << 20) / 8, nmask = n - 1;
    float best[4] = {1e9, 1e9, 1e9, 1e9};
    for (int rep = 0; rep < 4; ++rep) {
      float t;
      cudaEventRecord(a); gather<<<grid, block>>>(src, dst, nmask, count, rep); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t, a, b); best[0] = t < best[0] ? t : best[0];
      cudaEventRecord(a); scatter<<<grid, block>>>(src, nmask, count, rep); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t, a, b); best[1] = t < best[1] ? t : best[1];
      cudaEventRecord(a); amin<<<grid, block>>>(am, (((uint64_t)mb << 20) / 4) - 1, count, rep); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t, a, b); best[2] = t < best[2] ? t : best[2];
      cudaEventRecord(a); rmw<<<grid, block>>>(src, nmask, count, rep); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t, a, b); best[3] = t < best[3] ? t : best[3];
    }
    printf("buffer %5zu MB: gather %.2f G acc/s (%.0f GB/s useful)  scatter %.2f G acc/s  atomicMin32 %.2f G acc/s\n", mb,
           count / best[0] / 1e6, count * 8.0 / best[0] / 1e6, count / best[1] / 1e6, count / best[2] / 1e6);
    printf("{\"buffer_mb\": %zu, \"gather_per_s\": %.4g, \"scatter_per_s\": %.4g, \"atomicmin32_per_s\": %.4g, \"rmw_per_s\": %.4g}\n", mb,
           count / best[0] * 1e3, count / best[1] * 1e3, count / best[2] * 1e3, count / best[3] * 1e3);
  }
  float t; int64_t nn = (1ll << 30) / 16;
  for (int rep = 0; rep < 3; ++rep) { cudaEventRecord(a); copy<<<grid, block>>>((uint4*)src, (uint4*)am, nn); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t, a, b); }
  printf("copy 1 GiB: %.0f GB/s (read+write)\n", 2.0 * (1ll << 30) / t / 1e6);
  // L2-resident copy
  nn = (32ll << 20) / 16;
  float bt = 1e9;
  for (int rep = 0; rep < 20; ++rep) { cudaEventRecord(a); copy<<<grid, block>>>((uint4*)src, (uint4*)am, nn); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t, a, b); bt = t < bt ? t : bt; }
  printf("copy 32 MiB (L2): %.0f GB/s (read+write)\n", 2.0 * (32ll << 20) / bt / 1e6);
  return 0;
}
