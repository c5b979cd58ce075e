// Microbenchmark: L2 RED throughput for a gram-histogram-like scatter
// (n random u32 increments into `bins` counters), and the pure key read.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void gen(uint32_t* k, int64_t n, uint32_t bins, uint32_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    k[i] = x % bins;
  }
}
template <int MODE>
__global__ void scatter(const uint32_t* __restrict__ k, int64_t n, uint32_t* h, uint32_t* sink) {
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = __ldg(k + i);
    if (MODE == 0) atomicAdd(h + key, 1u);
    else acc += key;
  }
  if (MODE == 1 && acc == 0xdeadbeef) sink[0] = acc;
}
int main() {
  const int64_t n = 100000000;
  uint32_t *k, *h, *sink;
  cudaMalloc(&k, n * 4); cudaMalloc(&h, 64 << 20); cudaMalloc(&sink, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  uint32_t bins_list[] = {1336336, 33000, 4000000};
  for (uint32_t bins : bins_list) {
    gen<<<1184, 256>>>(k, n, bins, 7);
    for (int mode = 0; mode < 2; ++mode) {
      for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
        float best = 1e9;
        for (int r = 0; r < 3; ++r) {
          cudaMemset(h, 0, bins * 4);
          cudaEventRecord(a);
          if (mode == 0) scatter<0><<<grid, 256>>>(k, n, h, sink);
          else scatter<1><<<grid, 256>>>(k, n, h, sink);
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf("bins %u mode %s grid %d: %.3f ms  (%.1f G ops/s)\n", bins, mode ? "read" : "red", grid, best, n / best / 1e6);
      }
    }
  }
  return 0;
}
