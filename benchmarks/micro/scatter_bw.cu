// Microbenchmark: achieved HBM bandwidth of scatter write patterns on B200 (sm_100a).
// A (key, value) stream of N records is moved to a bucketed layout: record j of tile t
// (4096 records) goes to bucket j % B, after the records of earlier tiles in that
// bucket -- the write pattern of one radix pass with B digits of uniformly spread keys.
//   copy        out[i] = in[i] (the copy roofline of the same bytes)
//   direct      each thread stores its record straight to its destination
//   staged      the tile is reordered in shared memory, then runs are stored
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scatter_bw scatter_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int TILE = 4096;

__device__ __forceinline__ uint64_t dest_of(uint64_t i, uint64_t N, int B) {
  const uint64_t t = i / TILE, j = i % TILE;
  const uint64_t per = TILE / B;  // records per bucket per tile
  return (j % B) * (N / B) + t * per + j / B;
}

__global__ void k_copy(uint64_t N, const uint64_t* __restrict__ k, const double* __restrict__ v,
                       uint64_t* __restrict__ ko, double* __restrict__ vo) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
    ko[i] = __ldcs(k + i);
    vo[i] = __ldcs(v + i);
  }
}

template <int IPT>
__global__ void __launch_bounds__(256) k_direct(uint64_t N, int B, const uint64_t* __restrict__ k,
                                                const double* __restrict__ v, uint64_t* __restrict__ ko,
                                                double* __restrict__ vo) {
  const uint64_t base = (uint64_t)blockIdx.x * 256 * IPT;
  uint64_t kk[IPT];
  double vv[IPT];
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const uint64_t i = base + it * 256 + threadIdx.x;
    kk[it] = i < N ? __ldcs(k + i) : 0;
    vv[it] = i < N ? __ldcs(v + i) : 0;
  }
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const uint64_t i = base + it * 256 + threadIdx.x;
    if (i < N) {
      const uint64_t d = dest_of(i, N, B);
      ko[d] = kk[it];
      vo[d] = vv[it];
    }
  }
}

// Reads are coalesced tile loads (kept alive through a checksum); writes go to the
// bucketed destinations in output-slot order (runs of TILE/B records), no shared
// memory, so only the HBM write pattern differs from a copy.
template <bool P3>
__global__ void __launch_bounds__(256, 2) k_pattern(uint64_t N, int per, const uint64_t* __restrict__ k,
                                                    const double* __restrict__ v, uint64_t* __restrict__ ko,
                                                    double* __restrict__ vo, uint32_t* __restrict__ po,
                                                    uint64_t nb) {
  // runs of `per` records per bucket per tile, nb buckets, bucket regions N/nb apart
  const uint64_t tile = blockIdx.x;
  const uint64_t base = tile * TILE;
  uint64_t acc = 0;
  double vacc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    acc += __ldcs(k + base + r * 256 + threadIdx.x);
    vacc += __ldcs(v + base + r * 256 + threadIdx.x);
  }
  const uint64_t stride = N / nb;
#pragma unroll 4
  for (int p = threadIdx.x; p < TILE; p += 256) {
    const uint64_t bk = (uint64_t)(p / per) % nb;
    const uint64_t d = bk * stride + (tile * per + p % per) % stride;
    ko[d] = acc + p;
    vo[d] = vacc + p;
    if (P3) po[d] = (uint32_t)(acc + p);
  }
}

// Same pattern with (K', V) interleaved as one 16-byte record per slot (one STG.128) and
// the position in its own array: the record layout an interleaved intermediate would use.
__global__ void __launch_bounds__(256, 2) k_pattern_kv(uint64_t N, int per, const uint64_t* __restrict__ k,
                                                       const double* __restrict__ v, uint4* __restrict__ kvo,
                                                       uint32_t* __restrict__ po, uint64_t nb) {
  const uint64_t tile = blockIdx.x;
  const uint64_t base = tile * TILE;
  uint64_t acc = 0;
  double vacc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    acc += __ldcs(k + base + r * 256 + threadIdx.x);
    vacc += __ldcs(v + base + r * 256 + threadIdx.x);
  }
  const uint64_t stride = N / nb;
  const uint64_t vb = (uint64_t)__double_as_longlong(vacc);
#pragma unroll 4
  for (int p = threadIdx.x; p < TILE; p += 256) {
    const uint64_t bk = (uint64_t)(p / per) % nb;
    const uint64_t d = bk * stride + (tile * per + p % per) % stride;
    const uint64_t a = acc + p, b = vb + p;
    kvo[d] = make_uint4((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32));
    po[d] = (uint32_t)a;
  }
}

int main() {
  const uint64_t N = 256ull << 20;  // 256 Mi records: 4 GiB in, 4 GiB out
  uint64_t *k, *ko;
  double *v, *vo;
  cudaMalloc(&k, N * 8);
  cudaMalloc(&v, N * 8);
  cudaMalloc(&ko, N * 8 + (64ull << 20));
  cudaMalloc(&vo, N * 8 + (64ull << 20));
  cudaMemset(k, 1, N * 8);
  cudaMemset(v, 2, N * 8);

  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](const char* name, int B, auto launch) {
    for (int w = 0; w < 2; ++w) launch();
    cudaEventRecord(e0);
    const int R = 5;
    for (int r = 0; r < R; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= R;
    printf("%-10s run=%4d  %8.3f ms  %7.1f GB/s(r16+w16)  err=%s\n", name, B, ms, 32.0 * N / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  time("copy", 0, [&] { k_copy<<<148 * 8, 512>>>(N, k, v, ko, vo); });
  uint32_t* po;
  cudaMalloc(&po, N * 4 + (64ull << 20));
  uint4* kvo;
  cudaMalloc(&kvo, N * 16 + (64ull << 20));
  for (int per : {64, 16, 13, 8, 4}) {
    const uint64_t nb = TILE / per;
    time(per == 13 ? "2arr r13" : "2arr", per, [&] { k_pattern<false><<<N / TILE, 256>>>(N, per, k, v, ko, vo, po, nb); });
    time(per == 13 ? "3arr r13" : "3arr", per, [&] { k_pattern<true><<<N / TILE, 256>>>(N, per, k, v, ko, vo, po, nb); });
    time(per == 13 ? "kv+p r13" : "kv+p", per, [&] { k_pattern_kv<<<N / TILE, 256>>>(N, per, k, v, kvo, po, nb); });
  }
  return 0;
}
