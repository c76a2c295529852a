// small.cu — the `single` schedule: an input of at most 8,192 nonzeros sorted on one digit
// of <= 10 bits by ONE stable counting pass (SURVEY.md §8(a) a4-a7 in a single launch).
//
// One thread-block cluster of kSmCtas CTAs (portable size 8, one SM each), two records
// per thread.  CTA r takes the r-th contiguous chunk of the input: LIV shuffle,
// digit, stable rank inside the warp (one ballot per digit bit), per-warp digit counts
// -> exclusive prefix over the warps and the CTA's digit counts in shared memory.  After a
// cluster barrier every CTA reads the other CTAs' counts through distributed shared
// memory: the records of digit d in lower CTAs and the digit totals (scanned -> digit
// starts).  A record's output position is then
//     start[d] + (d in lower CTAs) + (d in lower warps) + (d in lower lanes)
// -- input order within a digit, the stable order of PAPER.md:245 -- and it is written
// straight there (K', value bits, source position).  A C1-sized tensor was issue-bound on
// the single SM of the one-CTA pass (17 us); spread over 8 SMs the pass has no count /
// scan / offsets kernels and no grid-wide synchronization.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "device_common.cuh"
#include "launch.h"
#include "lco_internal.h"

namespace cg = cooperative_groups;

namespace lco {

constexpr int kSmCtas = 8;
constexpr int kSmThreads = 512;
constexpr int kSmItems = 2;  // records per thread (warp w owns 64 consecutive records)
constexpr uint32_t kSmCap = (uint32_t)kSmCtas * kSmThreads * kSmItems;  // 8,192 records

template <int RB>
constexpr size_t single_cluster_smem() {
  // per-warp counts (u16) | CTA counts | digit totals | digit starts
  return (size_t)(kSmThreads / 32) * (1 << RB) * 2 + (size_t)(1 << RB) * 4 * 3;
}

template <int RB, bool VALS>
__global__ void __cluster_dims__(kSmCtas, 1, 1) __launch_bounds__(kSmThreads, 1)
    k_single_cluster(const __grid_constant__ PassParams a, const __grid_constant__ ScatterIO io) {
  constexpr int BINS = 1 << RB;
  constexpr int W = kSmThreads / 32;
  constexpr int PB = BINS > kSmThreads ? BINS / kSmThreads : 1;  // digits per thread (scans)
  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(smem);                  // [W][BINS]
  uint32_t* cnt = reinterpret_cast<uint32_t*>(wcnt + (size_t)W * BINS);  // [BINS] read remotely
  uint32_t* tot = cnt + BINS;                                          // [BINS]
  uint32_t* off = tot + BINS;                                          // [BINS]
  __shared__ uint32_t s_warp[32];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rank = cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t n = (uint32_t)a.nnz;
  const uint32_t chunk = (n + kSmCtas - 1) / kSmCtas;
  const uint32_t base = umin64((uint64_t)rank * chunk, n);
  const uint32_t m = (uint32_t)umin64(chunk, n - base);
  for (int i = tid; i < W * BINS / 2; i += kSmThreads) reinterpret_cast<uint32_t*>(wcnt)[i] = 0u;
  uint64_t k2[kSmItems];
  bool ok[kSmItems];
#pragma unroll
  for (int it = 0; it < kSmItems; ++it) {
    const uint32_t pos = warp * 32 * kSmItems + it * 32 + lane;  // input order: (warp, it, lane)
    ok[it] = pos < m;
    k2[it] = ok[it] ? __ldcs(io.keys_in + base + pos) : 0ull;
  }
  reencode_keys<kSmItems>(a.kp, k2);  // LIV shuffle
  const DigitFn dg(a);
  uint32_t d[kSmItems], below[kSmItems];
  __syncthreads();  // counters zeroed
  uint16_t* wc = wcnt + warp * BINS;
  const uint32_t ltm = lanemask_lt();
#pragma unroll
  for (int it = 0; it < kSmItems; ++it) {  // stable rank: earlier items, earlier lanes
    d[it] = ok[it] ? dg(a, k2[it]) : 0u;
    uint32_t peers = __ballot_sync(0xffffffffu, ok[it]);
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const uint32_t bit = (d[it] >> b) & 1u;
      peers &= __ballot_sync(0xffffffffu, bit) ^ (bit - 1u);
    }
    peers = ok[it] ? peers : 0u;
    const uint32_t bl = __popc(peers & ltm);
    const uint32_t before = ok[it] ? (uint32_t)wc[d[it]] : 0u;
    __syncwarp();
    if (ok[it] && bl == 0) wc[d[it]] = (uint16_t)(before + __popc(peers));
    below[it] = before + bl;
    __syncwarp();
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PB; ++j) {  // exclusive prefix over the warps; the CTA's digit counts
    const int dd = tid + j * kSmThreads;
    if (dd < BINS) {
      uint32_t s = 0;
#pragma unroll 8
      for (int w = 0; w < W; ++w) {
        const uint32_t c = wcnt[w * BINS + dd];
        wcnt[w * BINS + dd] = (uint16_t)s;
        s += c;
      }
      cnt[dd] = s;
    }
  }
  cl.sync();  // every CTA's counts are visible cluster-wide
  uint32_t lower[PB];
#pragma unroll
  for (int j = 0; j < PB; ++j) {
    const int dd = tid + j * kSmThreads;
    lower[j] = 0;
    if (dd < BINS) {
      uint32_t t = 0;
#pragma unroll
      for (int r = 0; r < kSmCtas; ++r) {
        const uint32_t c = cl.map_shared_rank(cnt, r)[dd];
        t += c;
        lower[j] += (uint32_t)r < rank ? c : 0u;
      }
      tot[dd] = t;
    }
  }
  cl.sync();  // no CTA reads a peer's counts after this (they may exit)
  block_scan_bins<kSmThreads, BINS>(tot, off, s_warp);  // digit starts (ends with a barrier)
#pragma unroll
  for (int j = 0; j < PB; ++j) {  // ... plus the lower CTAs' records of the digit
    const int dd = tid + j * kSmThreads;
    if (dd < BINS) off[dd] += lower[j];
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kSmItems; ++it) {
    if (!ok[it]) continue;
    const uint32_t i = base + warp * 32 * kSmItems + it * 32 + lane;
    const uint32_t g = off[d[it]] + wcnt[warp * BINS + d[it]] + below[it];
    io.kout[g] = k2[it];
    if (VALS) io.vout[g] = __ldcs(io.vals_in + i);
    if (io.pout) io.pout[g] = io.idx_in ? __ldg(io.idx_in + i) : i;
  }
}

template <int RB, bool VALS>
static cudaError_t launch_single_cluster_t(const PassParams& a, const ScatterIO& io,
                                           cudaStream_t s) {
  constexpr size_t smem = single_cluster_smem<RB>();
  cudaError_t e = kernel_setup(reinterpret_cast<const void*>(k_single_cluster<RB, VALS>), smem, 0);
  if (e != cudaSuccess) return e;
  k_single_cluster<RB, VALS><<<kSmCtas, kSmThreads, smem, s>>>(a, io);
  return cudaGetLastError();
}

cudaError_t run_single_cluster(int rb, const KeyPlan& kp, const PassIO& io, const Launch& L) {
  if (io.nnz > kSmCap) return cudaErrorInvalidValue;
  PassParams a;
  memset(&a, 0, sizeof a);
  a.kp = kp;
  a.kp.passes = 1;
  a.qshift = kp.divT.kind == 1 ? (int)kp.divT.s : (kp.divT.kind == 0 ? 0 : -1);
  a.nnz = io.nnz;
  ScatterIO sio;
  memset(&sio, 0, sizeof sio);
  sio.keys_in = io.keys_in;
  sio.vals_in = io.vals_in;
  sio.idx_in = io.idx_in;
  sio.kout = io.keys_out;
  sio.vout = io.vals_out;
  sio.pout = io.perm_out;
  const bool vals = io.vals_out != nullptr;
  if (L.mark) L.mark(L.ctx, "k_single_cluster");
  switch (rb) {
    case 8: return vals ? launch_single_cluster_t<8, true>(a, sio, L.stream)
                        : launch_single_cluster_t<8, false>(a, sio, L.stream);
    case 10: return vals ? launch_single_cluster_t<10, true>(a, sio, L.stream)
                         : launch_single_cluster_t<10, false>(a, sio, L.stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lco
