// Microbenchmark: throughput of global reductions (RED.ADD.U32, result unused) into an
// L2-resident table on B200: N updates at hashed positions of a table of T counters.
// Used to decide whether a pass can build the next pass's digit totals with one global
// reduction per record instead of a separate count pass.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bw red_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return (uint32_t)x;
}

__global__ void k_red(uint64_t N, uint32_t mask, uint32_t* __restrict__ t) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(t + (mix(i) & mask), 1u);
}
// runs of 16 equal high bits: the (d1, d2) pattern of a first-pass tile (d1 from the
// slot order, d2 random): consecutive lanes hit the same 1 KB row, random columns
__global__ void k_red_rows(uint64_t N, uint32_t mask, uint32_t* __restrict__ t) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(t + ((((uint32_t)(i >> 4) * 2654435761u) << 10 | (mix(i) & 1023u)) & mask), 1u);
}

int main() {
  const uint64_t N = 500000000ull;
  uint32_t* t;
  cudaMalloc(&t, 64u << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (uint32_t T : {1u << 18, 1u << 20, 1u << 22}) {
    for (int kind = 0; kind < 2; ++kind) {
      for (int w = 0; w < 2; ++w) {
        cudaMemset(t, 0, (size_t)T * 4);
        cudaEventRecord(e0);
        if (kind == 0) k_red<<<148 * 8, 512>>>(N, T - 1, t);
        else k_red_rows<<<148 * 8, 512>>>(N, T - 1, t);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (w) printf("%s table %8u counters: %8.3f ms  %7.1f G red/s  err=%s\n", kind ? "rows  " : "random", T, ms,
                      N / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
