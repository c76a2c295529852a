// mdt.cu — flattened LCO matrix -> compressed matrix datatypes.
//
// PAPER.md §5.2 (lines 325-331): a sparse tensor product first (1) permutes and flattens
// every operand into an LCO matrix in the order the chosen algorithm needs -- the
// permutation hot path of this library -- then (2) converts each LCO matrix to a matrix
// datatype (MDT): CSC/CSR, or the doubly compressed DCSC/DCSR of Buluc and Gilbert when
// the compressed dimension exceeds the NNZ (hyper-sparsity).
// An LCO matrix sorted major-first has key K = major * n_minor + minor, so compression
// never sorts:
//   singly (CSR / CSC):  ptr[n_major + 1], ptr[r] = first position whose major >= r; a
//                        nonzero that starts a new major writes the pointers of every
//                        empty major before it, so each entry is written exactly once;
//   doubly (DCSR / DCSC): ids[nz] of the non-empty majors and ptr[nz + 1]: a stream
//                        compaction of the positions that start a major (tile counts,
//                        one scan, tile-local ranks) -- memory O(nnz), never O(n_major).
// Both write minor[nnz] = K mod n_minor; the values array is the LCO's, unchanged.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "device_common.cuh"
#include "launch.h"
#include "lco_internal.h"

namespace lco {

constexpr int kCmThreads = 256;
constexpr int kCmItems = 16;
constexpr int kCmTile = kCmThreads * kCmItems;

__global__ void k_compress_singly(uint64_t nnz, const uint64_t* __restrict__ keys, FastDiv dmin,
                                  uint64_t n_minor, uint64_t n_major, uint64_t* __restrict__ ptr,
                                  uint64_t* __restrict__ minor) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const uint64_t k = __ldg(keys + i);
    const uint64_t r = fdiv(dmin, k);
    minor[i] = k - r * n_minor;
    const uint64_t rp = i ? fdiv(dmin, __ldg(keys + i - 1)) : ~0ull;  // ~0 + 1 = 0
    for (uint64_t x = rp + 1; x <= r; ++x) ptr[x] = i;
    if (i == nnz - 1)
      for (uint64_t x = r + 1; x <= n_major; ++x) ptr[x] = nnz;
  }
}

// Tile pass of the doubly compressed form: count (WRITE = false) or write the non-empty
// majors of tile t at toff[t] + tile-local rank.
template <bool WRITE>
__global__ void __launch_bounds__(kCmThreads) k_compress_doubly(uint64_t nnz,
                                                                const uint64_t* __restrict__ keys,
                                                                FastDiv dmin, uint64_t n_minor,
                                                                uint32_t* __restrict__ tcount,
                                                                const uint64_t* __restrict__ toff,
                                                                uint64_t* __restrict__ ids,
                                                                uint64_t* __restrict__ ptr,
                                                                uint64_t* __restrict__ minor) {
  __shared__ uint32_t s_warp[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t base = (uint64_t)blockIdx.x * kCmTile + (uint64_t)tid * kCmItems;
  uint64_t maj[kCmItems];
  uint32_t flags = 0, cnt = 0;
  uint64_t prev = base > 0 && base - 1 < nnz ? fdiv(dmin, __ldg(keys + base - 1)) : ~0ull;
#pragma unroll
  for (int it = 0; it < kCmItems; ++it) {
    const uint64_t i = base + it;
    if (i < nnz) {
      const uint64_t k = __ldg(keys + i);
      maj[it] = fdiv(dmin, k);
      if (WRITE) minor[i] = k - maj[it] * n_minor;
      const bool start = i == 0 || maj[it] != prev;
      flags |= (start ? 1u : 0u) << it;
      cnt += start ? 1u : 0u;
      prev = maj[it];
    }
  }
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < kCmThreads / 32 ? s_warp[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kCmThreads / 32) s_warp[lane] = wi - w;
    if (!WRITE && lane == kCmThreads / 32 - 1) tcount[blockIdx.x] = wi;
  }
  __syncthreads();
  if (!WRITE) return;
  uint64_t pos = toff[blockIdx.x] + s_warp[warp] + incl - cnt;
#pragma unroll
  for (int it = 0; it < kCmItems; ++it) {
    const uint64_t i = base + it;
    if (i < nnz && ((flags >> it) & 1u)) {
      ids[pos] = maj[it];
      ptr[pos] = i;
      ++pos;
    }
    if (i == nnz - 1) ptr[pos] = nnz;  // pos == number of non-empty majors here
  }
}

size_t compress_ctrl_bytes(uint64_t nnz) {
  const uint64_t nt = (nnz + kCmTile - 1) / kCmTile;
  return (nt * 4 + 255) / 256 * 256 + nt * 8 + 256;
}

cudaError_t run_compress(uint64_t nnz, const uint64_t* keys, uint64_t n_major, uint64_t n_minor,
                         int doubly, uint64_t* ptr, uint64_t* ids, uint64_t* minor,
                         uint64_t* n_nonempty, void* ctrl, const Launch& L) {
  const FastDiv dmin = make_fastdiv(n_minor);
  cudaError_t e;
  if (!doubly) {
    if (nnz == 0) return cudaMemsetAsync(ptr, 0, (n_major + 1) * 8, L.stream);
    if (L.mark) L.mark(L.ctx, "k_compress_singly");
    const uint64_t grid = umin64((nnz + 255) / 256, 148 * 16);
    k_compress_singly<<<(unsigned)grid, 256, 0, L.stream>>>(nnz, keys, dmin, n_minor, n_major,
                                                            ptr, minor);
    return cudaGetLastError();
  }
  if (nnz == 0) {
    if ((e = cudaMemsetAsync(ptr, 0, 8, L.stream)) != cudaSuccess) return e;
    return cudaMemsetAsync(n_nonempty, 0, 8, L.stream);
  }
  const uint64_t nt = (nnz + kCmTile - 1) / kCmTile;
  char* cb = static_cast<char*>(ctrl);
  uint32_t* tcount = reinterpret_cast<uint32_t*>(cb);
  uint64_t* toff = reinterpret_cast<uint64_t*>(cb + (nt * 4 + 255) / 256 * 256);
  if (L.mark) L.mark(L.ctx, "k_compress_count");
  k_compress_doubly<false><<<(unsigned)nt, kCmThreads, 0, L.stream>>>(
      nnz, keys, dmin, n_minor, tcount, nullptr, nullptr, nullptr, nullptr);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = run_count_scan(tcount, nt, toff, n_nonempty, L)) != cudaSuccess) return e;
  if (L.mark) L.mark(L.ctx, "k_compress_write");
  k_compress_doubly<true><<<(unsigned)nt, kCmThreads, 0, L.stream>>>(nnz, keys, dmin, n_minor,
                                                                     tcount, toff, ids, ptr, minor);
  return cudaGetLastError();
}

}  // namespace lco
