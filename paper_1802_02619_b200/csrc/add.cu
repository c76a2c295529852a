// add.cu — index-matched addition of two LCO tensors.
//
// PAPER.md:212-214 §3.2: adding c^(y)_{ijlk} and c^(x)_{jikl} of Eq (2.3) needs one of
// them "re-sorted into the {1,0,3,2} lexicographical order" (a permutation, the hot
// path of this library), after which the addition itself is a single merge of two
// sorted LIV streams.  C = A + sign * permute(B, match):
//   lco_permute moves B into A's order (B');
//   k_merge_split   merge-path split of every tile of kMTile merged positions (binary
//                   search of the co-rank, ties take A first);
//   k_merge<false>  per tile: count of outputs (a B' element whose key equals the A
//                   element merged just before it is folded into that element);
//   k_merge_scan    exclusive scan of the tile counts, total -> nnz_c;
//   k_merge<true>   per tile: writes keys and values (A-only: a, B-only: sign * b,
//                   both: a + sign * b, one IEEE addition; explicit zeros kept).
// Every thread merges kMItems consecutive positions from shared-memory copies of the
// tile's A and B' key ranges; the merged output is ascending because both inputs are.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "device_common.cuh"
#include "launch.h"
#include "lco_internal.h"

namespace lco {

constexpr int kMThreads = 256;
constexpr int kMItems = 16;
constexpr int kMTile = kMThreads * kMItems;

// co-rank: number of A elements among the first d merged (ties: A first)
__device__ __forceinline__ uint64_t co_rank(uint64_t d, const uint64_t* a, uint64_t na,
                                            const uint64_t* b, uint64_t nb) {
  uint64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) <= __ldg(b + (d - mid - 1))) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_merge_split(const uint64_t* __restrict__ a, uint64_t na,
                              const uint64_t* __restrict__ b, uint64_t nb, uint64_t ntiles,
                              uint64_t* __restrict__ split) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  const uint64_t d = t * kMTile < na + nb ? t * kMTile : na + nb;
  split[t] = co_rank(d, a, na, b, nb);
}

// One thread merges the positions [dl, de) of its tile and returns the number of
// outputs; with WRITE it also stores one recipe per output at rec[base + x]:
//   type 0: A element ia; type 1: A element ia + sign * B' element ib (ib may lie past
//   the tile's B' range, then it is read from global memory); type 2: B' element ib.
// A B' element equal to the A element merged just before it has already been added into
// that element and produces no output.
constexpr uint32_t kRecA = 0u, kRecAB = 1u, kRecB = 2u;

template <bool WRITE, class KA, class KB>
__device__ __forceinline__ uint32_t merge_run(uint32_t dl, uint32_t de, uint32_t ia, uint32_t ib,
                                              uint64_t i0, uint64_t j0, uint64_t na, uint64_t nb,
                                              KA keyA, KB keyB, uint32_t* rec, uint32_t base) {
  uint32_t cnt = 0;
  for (uint32_t p = dl; p < de; ++p) {
    const uint64_t gi = i0 + ia, gj = j0 + ib;
    const bool takeA = gi < na && (gj >= nb || keyA(gi) <= keyB(gj));
    if (takeA) {
      if (WRITE) {
        const bool both = gj < nb && keyB(gj) == keyA(gi);  // B' partner merges just after
        rec[base + cnt] = ((both ? kRecAB : kRecA) << 30) | (ia << 15) | ib;
      }
      ++cnt;
      ++ia;
    } else {
      if (!(gi > 0 && keyA(gi - 1) == keyB(gj))) {
        if (WRITE) rec[base + cnt] = (kRecB << 30) | (ia << 15) | ib;
        ++cnt;
      }
      ++ib;
    }
  }
  return cnt;
}

// Block-wide exclusive scan of one count per thread; returns this thread's base and the
// block total in *total.
__device__ __forceinline__ uint32_t merge_block_scan(uint32_t cnt, uint32_t* s_warp,
                                                     uint32_t* total) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < kMThreads / 32 ? s_warp[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kMThreads / 32) s_warp[lane] = wi - w;
    if (lane == kMThreads / 32 - 1) s_warp[31] = wi;
  }
  __syncthreads();
  *total = s_warp[31];
  return s_warp[warp] + incl - cnt;
}

constexpr size_t merge_smem(bool write) {
  return (size_t)kMTile * 8 + (write ? (size_t)kMTile * (8 + 4) : 0);
}

// Tile t of kMTile merged positions.  Count mode: the tile's output count.  Write mode:
// keys and values of the tile's A and B' ranges are staged in shared memory, every
// thread records its outputs' recipes, then the block writes the tile's outputs
// contiguously (coalesced) at toff[t].
template <bool WRITE>
__global__ void __launch_bounds__(kMThreads) k_merge(const uint64_t* __restrict__ a,
                                                     const double* __restrict__ va, uint64_t na,
                                                     const uint64_t* __restrict__ b,
                                                     const double* __restrict__ vb, uint64_t nb,
                                                     double sign, const uint64_t* __restrict__ split,
                                                     uint32_t* __restrict__ tcount,
                                                     const uint64_t* __restrict__ toff,
                                                     uint64_t* __restrict__ kc,
                                                     double* __restrict__ vc) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem);   // the tile's A keys, then its B' keys
  double* sv = reinterpret_cast<double*>(sk + kMTile);  // WRITE: their values
  uint32_t* rec = reinterpret_cast<uint32_t*>(sv + kMTile);  // WRITE: output recipes
  __shared__ uint32_t s_warp[32];
  const int tid = threadIdx.x;
  const uint64_t t = blockIdx.x;
  const uint64_t d0 = t * kMTile, n = na + nb;
  const uint64_t d1 = d0 + kMTile < n ? d0 + kMTile : n;
  const uint64_t i0 = split[t], i1 = split[t + 1];
  const uint64_t j0 = d0 - i0, j1 = d1 - i1;
  const uint32_t la = (uint32_t)(i1 - i0), lb = (uint32_t)(j1 - j0);
  uint64_t* sa = sk;
  uint64_t* sb = sk + la;
  for (uint32_t x = tid; x < la; x += kMThreads) {
    sa[x] = __ldg(a + i0 + x);
    if (WRITE) sv[x] = __ldg(va + i0 + x);
  }
  for (uint32_t x = tid; x < lb; x += kMThreads) {
    sb[x] = __ldg(b + j0 + x);
    if (WRITE) sv[la + x] = __ldg(vb + j0 + x);
  }
  __syncthreads();
  // this thread's diagonal inside the tile, co-rank by binary search in shared memory
  const uint32_t dl = min((uint32_t)(d1 - d0), (uint32_t)(tid * kMItems));
  const uint32_t de = min((uint32_t)(d1 - d0), dl + kMItems);
  uint32_t lo = dl > lb ? dl - lb : 0, hi = dl < la ? dl : la;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (sa[mid] <= sb[dl - mid - 1]) lo = mid + 1;
    else hi = mid;
  }
  const uint32_t ia = lo, ib = dl - lo;
  // keys just outside the tile's ranges come from global memory
  auto keyA = [&](uint64_t gi) { return gi >= i0 && gi < i1 ? sa[gi - i0] : __ldg(a + gi); };
  auto keyB = [&](uint64_t gj) { return gj >= j0 && gj < j1 ? sb[gj - j0] : __ldg(b + gj); };
  const uint32_t cnt = merge_run<false>(dl, de, ia, ib, i0, j0, na, nb, keyA, keyB, nullptr, 0);
  uint32_t total;
  const uint32_t base = merge_block_scan(cnt, s_warp, &total);
  if (!WRITE) {
    if (tid == 0) tcount[t] = total;
    return;
  }
  merge_run<true>(dl, de, ia, ib, i0, j0, na, nb, keyA, keyB, rec, base);
  __syncthreads();
  const uint64_t o0 = toff[t];
  for (uint32_t x = tid; x < total; x += kMThreads) {
    const uint32_t r = rec[x], ty = r >> 30, xa = (r >> 15) & 0x7FFFu, xb = r & 0x7FFFu;
    uint64_t k;
    double v;
    if (ty == kRecB) {
      k = sb[xb];
      v = sign * sv[la + xb];
    } else {
      k = sa[xa];
      v = sv[xa];
      if (ty == kRecAB) v = v + sign * (xb < lb ? sv[la + xb] : __ldg(vb + j0 + xb));
    }
    kc[o0 + x] = k;
    vc[o0 + x] = v;
  }
}

// Exclusive scan of the tile counts into toff (uint64) and the total into *nnz_c; one CTA.
__global__ void __launch_bounds__(1024) k_merge_scan(const uint32_t* __restrict__ tcount,
                                                     uint64_t ntiles, uint64_t* __restrict__ toff,
                                                     uint64_t* __restrict__ nnz_c) {
  __shared__ unsigned long long s_warp[32];
  __shared__ unsigned long long s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (uint64_t c0 = 0; c0 < ntiles; c0 += 1024) {
    const uint64_t i = c0 + tid;
    const unsigned long long v = i < ntiles ? tcount[i] : 0ull;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const unsigned long long w = s_warp[lane];
      unsigned long long wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      s_warp[lane] = wi - w;
    }
    __syncthreads();
    const unsigned long long carry = s_carry;
    if (i < ntiles) toff[i] = carry + s_warp[warp] + incl - v;
    __syncthreads();
    if (tid == 1023) s_carry = carry + s_warp[warp] + incl;
    __syncthreads();
  }
  if (tid == 0) *nnz_c = s_carry;
}

cudaError_t run_count_scan(const uint32_t* counts, uint64_t n, uint64_t* offsets, uint64_t* total,
                           const Launch& L) {
  if (L.mark) L.mark(L.ctx, "k_merge_scan_counts");
  k_merge_scan<<<1, 1024, 0, L.stream>>>(counts, n, offsets, total);
  return cudaGetLastError();
}

uint64_t merge_tiles(uint64_t na, uint64_t nb) { return (na + nb + kMTile - 1) / kMTile; }

size_t merge_ctrl_bytes(uint64_t na, uint64_t nb) {
  const uint64_t nt = merge_tiles(na, nb);
  return ((nt + 1) * 8 + 255) / 256 * 256 + (nt * 4 + 255) / 256 * 256 + nt * 8 + 256;
}

cudaError_t run_merge(uint64_t na, const uint64_t* ka, const double* va, uint64_t nb,
                      const uint64_t* kb, const double* vb, double sign, uint64_t* kc,
                      double* vc, uint64_t* nnz_c, void* ctrl, const Launch& L) {
  const uint64_t nt = merge_tiles(na, nb);
  char* cb = static_cast<char*>(ctrl);
  uint64_t* split = reinterpret_cast<uint64_t*>(cb);
  cb += ((nt + 1) * 8 + 255) / 256 * 256;
  uint32_t* tcount = reinterpret_cast<uint32_t*>(cb);
  cb += (nt * 4 + 255) / 256 * 256;
  uint64_t* toff = reinterpret_cast<uint64_t*>(cb);
  if (nt == 0) return cudaMemsetAsync(nnz_c, 0, 8, L.stream);
  if (L.mark) L.mark(L.ctx, "k_merge_split");
  k_merge_split<<<(unsigned)((nt + 1 + 255) / 256), 256, 0, L.stream>>>(ka, na, kb, nb, nt, split);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if ((e = kernel_setup(reinterpret_cast<const void*>(k_merge<false>), merge_smem(false),
                        kMThreads)) != cudaSuccess ||
      (e = kernel_setup(reinterpret_cast<const void*>(k_merge<true>), merge_smem(true),
                        kMThreads)) != cudaSuccess)
    return e;
  if (L.mark) L.mark(L.ctx, "k_merge_count");
  k_merge<false><<<(unsigned)nt, kMThreads, merge_smem(false), L.stream>>>(
      ka, va, na, kb, vb, nb, sign, split, tcount, nullptr, nullptr, nullptr);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (L.mark) L.mark(L.ctx, "k_merge_scan");
  k_merge_scan<<<1, 1024, 0, L.stream>>>(tcount, nt, toff, nnz_c);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (L.mark) L.mark(L.ctx, "k_merge_write");
  k_merge<true><<<(unsigned)nt, kMThreads, merge_smem(true), L.stream>>>(
      ka, va, na, kb, vb, nb, sign, split, tcount, toff, kc, vc);
  return cudaGetLastError();
}

}  // namespace lco
