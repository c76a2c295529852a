// Microbenchmark: is a short-run radix scatter bound by the DRAM write-back pattern or
// by L2 transactions?  The same scatter (runs of `per` records per bucket per 4,096-record
// tile, 3 arrays K 8 B / V 8 B / P 4 B) is timed
//   global   into a full-size destination (every line written back to HBM), and
//   chunked  chunk by chunk into one L2-sized region that the next chunk overwrites
//            (C records, 20*C bytes), optionally followed per chunk by a coalesced
//            "consume" copy of the region to the full-size output and an L2 discard of
//            the region (the leaf stage of a bucket-at-a-time pipeline).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_scatter l2_scatter.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int TILE = 4096;

// tile `tile` of a chunk of n records (nb buckets of n/nb records) scattered into dst
__global__ void __launch_bounds__(512, 2) k_pattern(uint64_t n, int per, uint64_t nb,
                                                    const uint64_t* __restrict__ k,
                                                    const double* __restrict__ v,
                                                    const uint32_t* __restrict__ p,
                                                    uint64_t* __restrict__ ko, double* __restrict__ vo,
                                                    uint32_t* __restrict__ po) {
  const uint64_t tile = blockIdx.x;
  const uint64_t base = tile * TILE;
  uint64_t acc = 0;
  double vacc = 0;
  uint32_t pacc = 0;
#pragma unroll
  for (int r = 0; r < TILE / 512; ++r) {
    acc += __ldcs(k + base + r * 512 + threadIdx.x);
    vacc += __ldcs(v + base + r * 512 + threadIdx.x);
    pacc += __ldcs(p + base + r * 512 + threadIdx.x);
  }
  const uint64_t stride = n / nb;
#pragma unroll 4
  for (int q = threadIdx.x; q < TILE; q += 512) {
    const uint64_t bk = (uint64_t)(q / per) % nb;
    const uint64_t d = bk * stride + (tile * per + q % per) % stride;
    ko[d] = acc + q;
    vo[d] = vacc + q;
    po[d] = pacc + q;
  }
}

__device__ __forceinline__ void discard_l2(const void* a) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
}

// coalesced copy of the region to the output; optionally discard the region's lines
template <bool DISCARD>
__global__ void __launch_bounds__(512) k_consume(uint64_t n, const uint64_t* __restrict__ k,
                                                 const double* __restrict__ v,
                                                 const uint32_t* __restrict__ p,
                                                 uint64_t* __restrict__ ko, double* __restrict__ vo,
                                                 uint32_t* __restrict__ po) {
  for (uint64_t i = blockIdx.x * 512ull + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 512) {
    ko[i] = k[i];
    vo[i] = v[i];
    po[i] = p[i];
  }
  if (DISCARD) {
    __syncthreads();
    // lines of this CTA's iterations: 16 keys / 32 indices per 128-B line
    for (uint64_t i = (blockIdx.x * 512ull + threadIdx.x) * 16; i < n; i += (uint64_t)gridDim.x * 512 * 16) {
      discard_l2(k + i);
      discard_l2(v + i);
      if ((i & 31) == 0) discard_l2(p + i);
    }
  }
}

int main() {
  const uint64_t N = 256ull << 20;
  uint64_t *k, *ko, *tk;
  double *v, *vo, *tv;
  uint32_t *p, *po, *tp;
  cudaMalloc(&k, N * 8);
  cudaMalloc(&v, N * 8);
  cudaMalloc(&p, N * 4);
  cudaMalloc(&ko, N * 8);
  cudaMalloc(&vo, N * 8);
  cudaMalloc(&po, N * 4);
  const uint64_t CMAX = 8ull << 20;
  cudaMalloc(&tk, CMAX * 8);
  cudaMalloc(&tv, CMAX * 8);
  cudaMalloc(&tp, CMAX * 4);
  cudaMemset(k, 1, N * 8);
  cudaMemset(v, 2, N * 8);
  cudaMemset(p, 3, N * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](const char* name, int per, uint64_t C, auto launch) {
    launch();
    cudaEventRecord(e0);
    const int R = 3;
    for (int r = 0; r < R; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= R;
    printf("%-22s run=%3d chunk=%5lluK %8.3f ms  %7.1f GB/s (40 B/rec)  err=%s\n", name, per,
           (unsigned long long)(C >> 10), ms, 40.0 * N / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  time("copy", 0, N, [&] { k_consume<false><<<148 * 4, 512>>>(N, k, v, p, ko, vo, po); });
  for (int per : {16, 8, 4}) {
    const uint64_t nb = TILE / per;
    time("global scatter", per, N,
         [&] { k_pattern<<<N / TILE, 512>>>(N, per, nb, k, v, p, ko, vo, po); });
    for (uint64_t C : {1ull << 20, 2ull << 20, 4ull << 20}) {
      time("chunked scatter", per, C, [&] {
        for (uint64_t c = 0; c < N; c += C)
          k_pattern<<<C / TILE, 512>>>(C, per, nb, k + c, v + c, p + c, tk, tv, tp);
      });
      time("chunked scat+consume", per, C, [&] {
        for (uint64_t c = 0; c < N; c += C) {
          k_pattern<<<C / TILE, 512>>>(C, per, nb, k + c, v + c, p + c, tk, tv, tp);
          k_consume<false><<<148 * 2, 512>>>(C, tk, tv, tp, ko + c, vo + c, po + c);
        }
      });
      time("chunked scat+cons+disc", per, C, [&] {
        for (uint64_t c = 0; c < N; c += C) {
          k_pattern<<<C / TILE, 512>>>(C, per, nb, k + c, v + c, p + c, tk, tv, tp);
          k_consume<true><<<148 * 2, 512>>>(C, tk, tv, tp, ko + c, vo + c, po + c);
        }
      });
    }
    time("global scat+consume", per, N, [&] {
      k_pattern<<<N / TILE, 512>>>(N, per, nb, k, v, p, ko, vo, po);
      k_consume<false><<<148 * 4, 512>>>(N, ko, vo, po, k, v, p);
    });
  }
  return 0;
}
