// block.cu — the block-transpose schedule: a permutation whose rearranged modes all lie
// in a small old-order prefix of the modes.
//
// Let k be the largest old position among the prefix + middle modes of the flat plan
// (§8(a) a1).  The old modes 0..k form a "block" id b = K div F (F = product of the
// later, free, modes).  The input is sorted by old key, so every block is one contiguous
// run; the free modes are suffix modes in unchanged relative order, so every block is
// also one contiguous run of the output, at the position its block coordinates take in
// the NEW order (PAPER.md:245: the resting trailing indices need no sorting; :183 the
// data is "already sorted").  The permutation is then a transpose of a ragged grid of
// runs, with no sorting at all:
//   k_block_bounds    run starts / ends of the blocks present (one read of the keys);
//   k_block_counts    counts moved to the blocks' NEW-order ids (a dense grid transpose);
//   k_scan_tiles x2   exclusive scan of the counts in new order -> output starts;
//   k_block_delta     delta[b] = output start - input start (mod 2^32);
//   k_block_scatter   out = i + delta[b]: K' (LIV shuffle), V, position, one coalesced
//                     read and one run-coalesced write per nonzero.
// Taken when the block grid is small (<= nnz / 4 blocks): BASELINE C4 (2048 x 2048 blocks
// of ~13 nonzeros), Table 2's {0,1,3,2}-type permutations.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "device_common.cuh"
#include "launch.h"
#include "lco_internal.h"

namespace lco {

constexpr int kBkTile = 4096;  // scan tile (counts)

__device__ __forceinline__ uint64_t block_of(uint64_t k, const FastDiv& f) { return fdiv(f, k); }

// One tile of kBkU x 256 consecutive nonzeros per CTA, lane-consecutive: the key loads of
// a thread are independent (8 in flight), the neighbours come from the same warp's loads
// or one extra load at the warp's edges.
constexpr int kBkU = 8;

__global__ void __launch_bounds__(256) k_block_bounds(uint64_t nnz, const uint64_t* __restrict__ keys,
                                                      FastDiv fF, uint32_t* __restrict__ bstart,
                                                      uint32_t* __restrict__ bend) {
  const uint64_t base = (uint64_t)blockIdx.x * 256 * kBkU + threadIdx.x;
  uint64_t b[kBkU];
#pragma unroll
  for (int u = 0; u < kBkU; ++u) {
    const uint64_t i = base + (uint64_t)u * 256;
    b[u] = i < nnz ? block_of(__ldcs(keys + i), fF) : ~0ull;
  }
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < kBkU; ++u) {
    const uint64_t i = base + (uint64_t)u * 256;
    uint64_t prev = __shfl_up_sync(0xffffffffu, b[u], 1);
    uint64_t next = __shfl_down_sync(0xffffffffu, b[u], 1);
    if (i < nnz) {
      if (lane == 0) prev = i > 0 ? block_of(__ldg(keys + i - 1), fF) : ~0ull;
      if (lane == 31 || i + 1 >= nnz) next = i + 1 < nnz ? block_of(__ldg(keys + i + 1), fF) : ~0ull;
      if (i == 0 || prev != b[u]) bstart[b[u]] = (uint32_t)i;
      if (i == nnz - 1 || next != b[u]) bend[b[u]] = (uint32_t)(i + 1);
    }
  }
}

__global__ void k_block_counts(uint64_t nblocks, const __grid_constant__ KeyPlan kb,
                               const uint32_t* __restrict__ bstart,
                               const uint32_t* __restrict__ bend, uint32_t* __restrict__ cnew) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += stride)
    cnew[reencode(kb, b)] = __ldg(bend + b) - __ldg(bstart + b);
}

// Tile sums (SUMS) / tile-local exclusive scan plus the tile's offset (!SUMS), in place.
template <bool SUMS>
__global__ void __launch_bounds__(256) k_scan_tiles(uint64_t n, uint32_t* __restrict__ a,
                                                    uint32_t* __restrict__ sums,
                                                    const uint64_t* __restrict__ toff) {
  __shared__ uint32_t s_warp[32];
  constexpr int PER = kBkTile / 256;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t base = (uint64_t)blockIdx.x * kBkTile + (uint64_t)tid * PER;
  uint32_t v[PER], sum = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    v[i] = base + i < n ? a[base + i] : 0u;
    sum += v[i];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < 8 ? s_warp[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < 8) s_warp[lane] = wi - w;
    if (SUMS && lane == 7) sums[blockIdx.x] = wi;
  }
  __syncthreads();
  if (SUMS) return;
  uint32_t run = (uint32_t)toff[blockIdx.x] + s_warp[warp] + incl - sum;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    if (base + i < n) a[base + i] = run;
    run += v[i];
  }
}

__global__ void k_block_delta(uint64_t nblocks, const __grid_constant__ KeyPlan kb,
                              const uint32_t* __restrict__ bstart,
                              const uint32_t* __restrict__ outstart, uint32_t* __restrict__ delta) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += stride)
    delta[b] = __ldg(outstart + reencode(kb, b)) - __ldg(bstart + b);
}

// kBkU nonzeros per thread, lane-consecutive (coalesced reads; a block's nonzeros are
// consecutive in the output too, so the writes come in runs); all loads issued first.
template <bool VALS>
__global__ void __launch_bounds__(256) k_block_scatter(uint64_t nnz, const __grid_constant__ KeyPlan kp,
                                                       FastDiv fF, const uint64_t* __restrict__ keys_in,
                                                       const double* __restrict__ vals_in,
                                                       const uint32_t* __restrict__ idx_in,
                                                       const uint32_t* __restrict__ delta,
                                                       uint64_t* __restrict__ keys_out,
                                                       double* __restrict__ vals_out,
                                                       uint32_t* __restrict__ perm_out) {
  // grid-stride over chunks in launch order with a small grid: the concurrently written
  // output window (one run per block per active chunk) stays small enough for L2 to
  // complete the partial lines before they are evicted
  for (uint64_t base = (uint64_t)blockIdx.x * 256 * kBkU + threadIdx.x; base < nnz;
       base += (uint64_t)gridDim.x * 256 * kBkU) {
  uint64_t k[kBkU];
  double v[kBkU];
  uint32_t o[kBkU];
#pragma unroll
  for (int u = 0; u < kBkU; ++u) {
    const uint64_t i = base + (uint64_t)u * 256;
    k[u] = i < nnz ? __ldcs(keys_in + i) : 0ull;
    if (VALS) v[u] = i < nnz ? __ldcs(vals_in + i) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kBkU; ++u) {
    const uint64_t i = base + (uint64_t)u * 256;
    o[u] = i < nnz ? (uint32_t)i + __ldg(delta + block_of(k[u], fF)) : 0u;
  }
  reencode_keys<kBkU>(kp, k);
#pragma unroll
  for (int u = 0; u < kBkU; ++u) {
    const uint64_t i = base + (uint64_t)u * 256;
    if (i < nnz) {
      keys_out[o[u]] = k[u];
      if (VALS) vals_out[o[u]] = v[u];
      if (perm_out) perm_out[o[u]] = idx_in ? __ldg(idx_in + i) : (uint32_t)i;
    }
  }
  }
}

size_t block_ctrl_bytes(uint64_t nblocks) {
  const uint64_t nt = (nblocks + kBkTile - 1) / kBkTile;
  return 3 * ((nblocks * 4 + 255) / 256 * 256) + (nt * 4 + 255) / 256 * 256 + nt * 8 + 512;
}

cudaError_t run_block(const KeyPlan& kp, const KeyPlan& kb, uint64_t nblocks, uint64_t F,
                      const PassIO& io, const Launch& L) {
  cudaError_t e;
  const uint64_t nnz = io.nnz;
  const size_t tb = (nblocks * 4 + 255) / 256 * 256;
  char* cb = reinterpret_cast<char*>(io.ctrl);
  uint32_t* bstart = reinterpret_cast<uint32_t*>(cb);
  uint32_t* bend = reinterpret_cast<uint32_t*>(cb + tb);  // later: delta
  uint32_t* cnew = reinterpret_cast<uint32_t*>(cb + 2 * tb);  // later: output starts
  const uint64_t nt = (nblocks + kBkTile - 1) / kBkTile;
  uint32_t* sums = reinterpret_cast<uint32_t*>(cb + 3 * tb);
  uint64_t* toff = reinterpret_cast<uint64_t*>(cb + 3 * tb + (nt * 4 + 255) / 256 * 256);
  uint64_t* total = toff + nt;
  const FastDiv fF = make_fastdiv(F);
  if ((e = cudaMemsetAsync(bstart, 0, 2 * tb, L.stream)) != cudaSuccess) return e;
  const unsigned gn = (unsigned)((nnz + 256 * kBkU - 1) / (256 * kBkU));
  const unsigned gb = (unsigned)umin64((nblocks + 255) / 256, 148 * 16);
  if (L.mark) L.mark(L.ctx, "k_block_bounds");
  k_block_bounds<<<gn, 256, 0, L.stream>>>(nnz, io.keys_in, fF, bstart, bend);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (L.mark) L.mark(L.ctx, "k_block_counts");
  k_block_counts<<<gb, 256, 0, L.stream>>>(nblocks, kb, bstart, bend, cnew);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (L.mark) L.mark(L.ctx, "k_block_scan");
  k_scan_tiles<true><<<(unsigned)nt, 256, 0, L.stream>>>(nblocks, cnew, sums, nullptr);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = run_count_scan(sums, nt, toff, total, Launch{L.stream, nullptr, nullptr})) != cudaSuccess)
    return e;
  k_scan_tiles<false><<<(unsigned)nt, 256, 0, L.stream>>>(nblocks, cnew, nullptr, toff);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (L.mark) L.mark(L.ctx, "k_block_delta");
  k_block_delta<<<gb, 256, 0, L.stream>>>(nblocks, kb, bstart, cnew, bend);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (L.mark) L.mark(L.ctx, "k_block_scatter");
  const unsigned gsc = (unsigned)umin64(gn, 148 * 32);
  if (io.vals_out)
    k_block_scatter<true><<<gsc, 256, 0, L.stream>>>(nnz, kp, fF, io.keys_in, io.vals_in, io.idx_in,
                                                   bend, io.keys_out, io.vals_out, io.perm_out);
  else
    k_block_scatter<false><<<gsc, 256, 0, L.stream>>>(nnz, kp, fF, io.keys_in, io.vals_in, io.idx_in,
                                                    bend, io.keys_out, io.vals_out, io.perm_out);
  return cudaGetLastError();
}

}  // namespace lco
