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
//   k_block_counts    counts moved to the blocks' NEW-order ids (a tiled grid transpose)
//                     and the sums of the scan tiles;
//   k_scan_tiles      exclusive scan of the counts in new order -> output starts;
//   k_block_tiles     a tiled transpose of the runs: per tile of blocks, long input runs
//                     -> LIV shuffle -> shared memory in output order -> long output
//                     runs (K', V, position).
// Taken when the block grid is small (<= nnz / 4 blocks): BASELINE C4 (2048 x 2048 blocks
// of ~13 nonzeros).
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

// 256 consecutive nonzeros per warp (8 per lane, lane-consecutive): all key loads are
// issued before any block id is computed; block ids are 32-bit (nblocks < 2^31); each
// nonzero's neighbours come from one lane rotation per direction (lane 0's predecessor is
// the previous item's rotated value at lane 0), plus one key on each side of the warp.
constexpr int kBkU = 8;

__global__ void __launch_bounds__(256) k_block_bounds(uint64_t nnz, const uint64_t* __restrict__ keys,
                                                      FastDiv fF, uint32_t* __restrict__ bstart,
                                                      uint32_t* __restrict__ bend) {
  const int lane = threadIdx.x & 31;
  const uint64_t wbase = ((uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * (32 * kBkU);
  uint64_t k[kBkU];
#pragma unroll
  for (int u = 0; u < kBkU; ++u) {
    const uint64_t i = wbase + u * 32 + lane;
    k[u] = i < nnz ? __ldcs(keys + i) : 0ull;
  }
  const bool has_p = wbase > 0, has_n = wbase + 32 * kBkU < nnz;
  const uint64_t kp = (lane == 31 && has_p) ? __ldg(keys + wbase - 1) : 0ull;
  const uint64_t kn = (lane == 0 && has_n) ? __ldg(keys + wbase + 32 * kBkU) : 0ull;
  constexpr uint32_t kNone = 0xffffffffu;
  uint32_t b[kBkU];
#pragma unroll
  for (int u = 0; u < kBkU; ++u)
    b[u] = wbase + u * 32 + lane < nnz ? (uint32_t)block_of(k[u], fF) : kNone;
  // rotations: up[u] at lane l = b[u] at lane l-1 (lane 0: lane 31), dn[u] at lane l =
  // b[u] at lane l+1 (lane 31: lane 0)
  uint32_t up_prev = __shfl_sync(0xffffffffu, (lane == 31 && has_p) ? (uint32_t)block_of(kp, fF) : kNone,
                                 (lane + 31) & 31);
  uint32_t dn[kBkU + 1];
#pragma unroll
  for (int u = 0; u < kBkU; ++u) dn[u] = __shfl_sync(0xffffffffu, b[u], (lane + 1) & 31);
  dn[kBkU] = __shfl_sync(0xffffffffu, (lane == 0 && has_n) ? (uint32_t)block_of(kn, fF) : kNone,
                         (lane + 1) & 31);
#pragma unroll
  for (int u = 0; u < kBkU; ++u) {
    const uint64_t i = wbase + u * 32 + lane;
    const uint32_t up = __shfl_sync(0xffffffffu, b[u], (lane + 31) & 31);
    const uint32_t prev = lane == 0 ? up_prev : up;  // lane 0: item u-1 at lane 31
    const uint32_t next = lane == 31 ? dn[u + 1] : dn[u];  // lane 31: item u+1 at lane 0
    up_prev = up;
    if (i < nnz) {
      if (prev != b[u]) bstart[b[u]] = (uint32_t)i;
      if (next != b[u]) bend[b[u]] = (uint32_t)(i + 1);
    }
  }
}

// The same with 16-byte key loads (keys 16-byte aligned): item u of a lane is the pair
// (2 lane, 2 lane + 1) of the warp's 64-key chunk u; a pair's outer neighbours come from
// one lane rotation per direction.
template <int U2>
__global__ void __launch_bounds__(256) k_block_bounds(uint64_t nnz, const uint64_t* __restrict__ keys,
                                                       FastDiv fF, uint32_t* __restrict__ bstart,
                                                       uint32_t* __restrict__ bend) {
  const int lane = threadIdx.x & 31;
  constexpr int W = 64 * U2;  // keys per warp
  const uint64_t wbase = ((uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * W;
  const bool full = wbase + W <= nnz;
  ulonglong2 k[U2];
#pragma unroll
  for (int u = 0; u < U2; ++u) {
    const uint64_t i = wbase + u * 64 + 2 * lane;
    if (full) {
      k[u] = __ldcs(reinterpret_cast<const ulonglong2*>(keys + i));
    } else {
      k[u].x = i < nnz ? __ldcs(keys + i) : 0ull;
      k[u].y = i + 1 < nnz ? __ldcs(keys + i + 1) : 0ull;
    }
  }
  const bool has_p = wbase > 0, has_n = wbase + W < nnz;
  const uint64_t kp = (lane == 31 && has_p) ? __ldg(keys + wbase - 1) : 0ull;
  const uint64_t kn = (lane == 0 && has_n) ? __ldg(keys + wbase + W) : 0ull;
  constexpr uint32_t kNone = 0xffffffffu;
  uint32_t b0[U2], b1[U2];
#pragma unroll
  for (int u = 0; u < U2; ++u) {
    const uint64_t i = wbase + u * 64 + 2 * lane;
    b0[u] = i < nnz ? (uint32_t)block_of(k[u].x, fF) : kNone;
    b1[u] = i + 1 < nnz ? (uint32_t)block_of(k[u].y, fF) : kNone;
  }
  // up: b1 of lane l-1 (lane 0: previous chunk's lane 31); dn: b0 of lane l+1 (lane 31:
  // next chunk's lane 0)
  uint32_t up_prev = __shfl_sync(0xffffffffu, (lane == 31 && has_p) ? (uint32_t)block_of(kp, fF) : kNone,
                                 (lane + 31) & 31);
  uint32_t dn[U2 + 1];
#pragma unroll
  for (int u = 0; u < U2; ++u) dn[u] = __shfl_sync(0xffffffffu, b0[u], (lane + 1) & 31);
  dn[U2] = __shfl_sync(0xffffffffu, (lane == 0 && has_n) ? (uint32_t)block_of(kn, fF) : kNone,
                       (lane + 1) & 31);
#pragma unroll
  for (int u = 0; u < U2; ++u) {
    const uint64_t i = wbase + u * 64 + 2 * lane;
    const uint32_t up = __shfl_sync(0xffffffffu, b1[u], (lane + 31) & 31);
    const uint32_t prev = lane == 0 ? up_prev : up;
    const uint32_t next = lane == 31 ? dn[u + 1] : dn[u];
    up_prev = up;
    if (i < nnz) {
      if (prev != b0[u]) bstart[b0[u]] = (uint32_t)i;
      if (b1[u] != b0[u]) bend[b0[u]] = (uint32_t)(i + 1);
    }
    if (i + 1 < nnz) {
      if (b0[u] != b1[u]) bstart[b1[u]] = (uint32_t)(i + 1);
      if (next != b1[u]) bend[b1[u]] = (uint32_t)(i + 2);
    }
  }
}

// Exclusive scan of the new-order counts, in place, plus the tile's offset: one tile of
// kBkTile counts per CTA, 512 per warp read lane-consecutively (coalesced), warp scans
// with a running carry.
__global__ void __launch_bounds__(256) k_scan_tiles(uint64_t n, uint32_t* __restrict__ a,
                                                    const uint64_t* __restrict__ toff) {
  __shared__ uint32_t s_warp[8];
  constexpr int PER = kBkTile / 256;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t wbase = (uint64_t)blockIdx.x * kBkTile + (uint64_t)warp * 32 * PER;
  uint32_t v[PER], carry = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const uint64_t x = wbase + i * 32 + lane;
    v[i] = x < n ? a[x] : 0u;
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    uint32_t incl = v[i];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t ex = carry + incl - v[i];
    carry += __shfl_sync(0xffffffffu, incl, 31);
    v[i] = ex;
  }
  if (lane == 0) s_warp[warp] = carry;
  __syncthreads();
  uint32_t off = (uint32_t)toff[blockIdx.x];
  for (int w = 0; w < warp; ++w) off += s_warp[w];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const uint64_t x = wbase + i * 32 + lane;
    if (x < n) a[x] = off + v[i];
  }
}

// ---------------------------------------------------------------------------------
// k_block_tiles: one tile of TB x TA blocks per CTA (TB consecutive values of the new-
// innermost block mode B, TA of the old-innermost A, the other block coordinates fixed).
// Its TB input rows (fixed c_B, c_A in the tile) are contiguous runs of the input and its
// TA output runs (fixed c_A, c_B in the tile) contiguous runs of the output, so the CTA
// reads TB long runs, LIV-shuffles the keys and stages K', V and the
// source position in shared memory in OUTPUT order, then writes TA long runs: the
// output of a ~13-nonzero block is no longer written by itself (unaligned short runs cap
// a scatter at ~3 TB/s).  A tile larger than the stage (big blocks) is
// written straight from registers: its runs are long anyway.
// ---------------------------------------------------------------------------------
constexpr int kBtThreads = 256;
constexpr int kBtLgWarps = 3;
// measured on C4: 2,048-nonzero stages at 4 CTAs/SM beat 3,072-4,096 at
// 2-3 CTAs/SM and 1,024-1,800 at 5-6; 2 nonzeros per thread per round beat 4 and 8
constexpr int kBtCap = 2048;    // staged nonzeros per tile: 17 B each
constexpr int kBtMinBlocks = 4;
constexpr int kBtU = 2;         // nonzeros per thread per round (register path)
constexpr int kBtWU = 4;        // nonzeros per thread per round (stage -> output)
constexpr int kBtTarget = 1700;  // expected nonzeros per tile the host sizes tiles for

struct BlockTiling {
  uint64_t dA, dB;
  uint32_t mid, ntA, ntB;  // tile counts < 2^31: 32-bit index arithmetic
  int lgTA, lgTB;
};

__device__ __forceinline__ uint64_t tile_base(const BlockTiling& g, uint32_t t, uint64_t* b0,
                                              uint64_t* a0) {
  const uint32_t bT = t % g.ntB;
  t /= g.ntB;
  const uint32_t aT = t % g.ntA;
  t /= g.ntA;
  *b0 = (uint64_t)bT << g.lgTB;
  *a0 = (uint64_t)aT << g.lgTA;
  // old block id at c_B = c_A = 0
  return ((uint64_t)(t / g.mid) * g.dB * g.mid + t % g.mid) * g.dA;
}

// Block counts moved to NEW-order positions: a 32 x 32 (A x B) tile transpose through
// shared memory (reads along the old-innermost mode A, writes along the new-innermost
// mode B, both coalesced), plus each scan tile's sum (atomics per written run).
// T consecutive tiles per CTA, every tile's loads issued before any is transposed (the
// kernel is L2-latency bound: the bounds were just written).
constexpr int kBcT = 4;

template <int T>
__global__ void __launch_bounds__(256) k_block_counts(const __grid_constant__ BlockTiling g,
                                                      const __grid_constant__ KeyPlan kb, uint32_t ntiles,
                                                      const uint32_t* __restrict__ bstart,
                                                      const uint32_t* __restrict__ bend,
                                                      uint32_t* __restrict__ cnew,
                                                      uint32_t* __restrict__ sums) {
  __shared__ uint32_t t[T][32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
  const uint64_t strideB = (uint64_t)g.mid * g.dA;
  uint64_t b0[T], a0[T], base[T];
  uint32_t s[T][4], e[T][4];
#pragma unroll
  for (int j = 0; j < T; ++j) {
    const uint32_t tile = blockIdx.x * T + j;
    base[j] = tile_base(g, tile < ntiles ? tile : 0u, &b0[j], &a0[j]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // r = ty + 8 q: B offset, tx: A offset
      const int r = ty + 8 * q;
      s[j][q] = e[j][q] = 0;
      if (tile < ntiles && b0[j] + r < g.dB && a0[j] + tx < g.dA) {
        const uint64_t id = base[j] + (b0[j] + r) * strideB + a0[j] + tx;
        s[j][q] = __ldg(bstart + id);
        e[j][q] = __ldg(bend + id);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < T; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) t[j][ty + 8 * q][tx] = e[j][q] - s[j][q];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < T; ++j) {
    if (blockIdx.x * T + j >= ntiles) break;  // CTA-uniform
    // new id of (b0, a0 + r) = nid0 + r * sA (the new stride of mode A)
    const uint64_t nid0 = reencode(kb, base[j] + b0[j] * strideB + a0[j]);
    const uint64_t sA = a0[j] + 1 < g.dA ? reencode(kb, base[j] + b0[j] * strideB + a0[j] + 1) - nid0 : 0;
#pragma unroll
    for (int r = ty; r < 32; r += 8) {  // r: A offset, tx: B offset
      if (a0[j] + r >= g.dA) continue;  // warp-uniform
      const uint64_t nid = nid0 + r * sA;
      const bool ok = b0[j] + tx < g.dB;
      const uint32_t c = ok ? t[j][tx][r] : 0u;
      if (ok) cnew[nid + tx] = c;
      // scan-tile sums: the run [nid, nid + 32) meets at most two scan tiles
      const uint64_t tile0 = nid / kBkTile;
      const bool second = (nid + tx) / kBkTile != tile0;
      const uint32_t s0 = __reduce_add_sync(0xffffffffu, second ? 0u : c);
      const uint32_t s1 = __reduce_add_sync(0xffffffffu, second ? c : 0u);
      if (tx == 0 && s0) atomicAdd(sums + tile0, s0);
      if (tx == 0 && s1) atomicAdd(sums + tile0 + 1, s1);
    }
  }
}

template <bool VALS>
__global__ void __launch_bounds__(kBtThreads, kBtMinBlocks) k_block_tiles(
    const __grid_constant__ BlockTiling g, const __grid_constant__ KeyPlan kp,
    const __grid_constant__ KeyPlan kb, FastDiv fF, const uint64_t* __restrict__ keys_in,
    const double* __restrict__ vals_in, const uint32_t* __restrict__ idx_in,
    const uint32_t* __restrict__ bstart, const uint32_t* __restrict__ bend,
    const uint32_t* __restrict__ outstart, uint64_t* __restrict__ keys_out,
    double* __restrict__ vals_out, uint32_t* __restrict__ perm_out) {
  // input-ordered stage of the rows (K, V) and, per output slot, the row it comes from
  extern __shared__ __align__(16) unsigned char bt_smem[];
  uint64_t* sK = reinterpret_cast<uint64_t*>(bt_smem);
  double* sV = reinterpret_cast<double*>(sK + kBtCap);
  uint8_t* sB = reinterpret_cast<uint8_t*>(sV + kBtCap);
  __shared__ uint32_t s_cnt[kBtThreads], s_ipre[kBtThreads], s_opre[kBtThreads];  // TA * TB <= threads
  __shared__ uint32_t s_rowlen[32], s_runlen[32], s_runpre[33], s_rowoff[33], s_rs[32], s_ost[32];
  __shared__ uint64_t s_nid[32];  // new block id of (b0, a0 + a)
  // per block (a, b): stage index - slot, input index - stage index, K' - K
  __shared__ uint4 s_blk[kBtThreads];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lgTA = g.lgTA, lgTB = g.lgTB, TA = 1 << lgTA, TB = 1 << lgTB, nblk = TA * TB;
  // tile -> (hi, B tile, mid, A tile), B tiles fastest: consecutive CTAs extend the same
  // output runs, so partial sectors at run ends meet in L2
  uint64_t b0, a0;
  const uint64_t base = tile_base(g, blockIdx.x, &b0, &a0);
  const uint64_t strideB = (uint64_t)g.mid * g.dA;
  // 1. counts and starts of the tile's blocks; row-wise (over A) exclusive scan
  {
    const int b = tid >> lgTA, a = tid & (TA - 1);
    uint32_t c = 0, s = 0;
    if (tid < nblk && b0 + b < g.dB && a0 + a < g.dA) {
      const uint64_t id = base + (b0 + b) * strideB + a0 + a;
      s = __ldg(bstart + id);
      c = __ldg(bend + id) - s;
      // the output start of run a = the new-order start of its first block (b = 0)
      if (b == 0) {
        const uint64_t nid = reencode(kb, id);
        s_nid[a] = nid;
        s_ost[a] = __ldg(outstart + nid);
      }
    }
    uint32_t incl = c;
    for (int o = 1; o < TA; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o, TA);
      if (a >= o) incl += y;
    }
    if (tid < nblk) {
      s_cnt[tid] = c;
      s_ipre[tid] = incl - c;
      if (a == TA - 1) s_rowlen[b] = incl;
      if (c) s_rs[b] = s - (incl - c);  // every present block of a row agrees
    }
  }
  __syncthreads();
  // 2. column-wise (over B) exclusive scan: offsets of the blocks in their output run
  {
    const int a = tid >> lgTB, b = tid & (TB - 1);
    const uint32_t c = tid < nblk ? s_cnt[(b << lgTA) + a] : 0u;
    uint32_t incl = c;
    for (int o = 1; o < TB; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o, TB);
      if (b >= o) incl += y;
    }
    if (tid < nblk) {
      s_opre[(a << lgTB) + b] = incl - c;
      if (b == TB - 1) s_runlen[a] = incl;
    }
  }
  __syncthreads();
  // 3. run prefixes (output slots) and row offsets (input stage)
  if (warp < 2) {
    const int nr = warp == 0 ? TA : TB;
    const uint32_t v = lane < nr ? (warp == 0 ? s_runlen[lane] : s_rowlen[lane]) : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t* pre = warp == 0 ? s_runpre : s_rowoff;
    if (lane < nr) pre[lane] = incl - v;
    if (lane == nr - 1) pre[nr] = incl;
  }
  __syncthreads();
  const uint32_t E = s_runpre[TA];
  if (E <= (uint32_t)kBtCap) {
    // 4. rows -> input stage with cp.async (no registers held, every row in flight at
    //    once; measured faster than one TMA bulk copy per row, whose ~1 KB copies of
    //    16-byte aligned row interiors ran C4's tiles at 0.50 vs 0.45 ms)
    {
      const int lgW = lgTB >= kBtLgWarps ? 0 : kBtLgWarps - lgTB;
      const uint32_t gw = 32u << lgW, g0 = ((warp & ((1 << lgW) - 1)) << 5) + lane;
      for (int b = warp >> lgW; b < TB; b += (kBtThreads / 32) >> lgW) {
        const uint32_t len = s_rowlen[b], rs = s_rs[b], ro = s_rowoff[b];
        for (uint32_t r = g0; r < len; r += gw) {
          cp_async8(sK + ro + r, keys_in + rs + r);
          if (VALS) cp_async8(sV + ro + r, vals_in + rs + r);
        }
      }
      cp_async_commit();
    }
    // 5. while they fly: per block, stage offset of its slots; per slot, its row
    if (tid < nblk) {
      const int b = tid >> lgTA, a = tid & (TA - 1);
      const uint32_t c = s_cnt[tid], first = s_runpre[a] + s_opre[(a << lgTB) + b];
      for (uint32_t w = 0; w < c; ++w) sB[first + w] = (uint8_t)b;
      // the free modes follow the block modes unchanged in both orders, so the LIV
      // shuffle of a key of block (b, a) is K + (new id - old id) * F
      const uint64_t oid = base + (b0 + b) * strideB + a0 + a;
      const uint64_t kd = (s_nid[a] + b - oid) * fF.d;
      s_blk[(a << lgTB) + b] = make_uint4(s_rowoff[b] + s_ipre[tid] - first, s_rs[b] - s_rowoff[b],
                                          (uint32_t)kd, (uint32_t)(kd >> 32));
    }
    cp_async_wait<0>();
    __syncthreads();
    // 6. write the TA output runs (2^lgW warps per run): gather from the stage, LIV
    //    shuffle, long coalesced runs of K', V and the source position
    const int lgW = lgTA >= kBtLgWarps ? 0 : kBtLgWarps - lgTA;
    const uint32_t gw = 32u << lgW, g0 = ((warp & ((1 << lgW) - 1)) << 5) + lane;
    for (int a = warp >> lgW; a < TA; a += (kBtThreads / 32) >> lgW) {
      const uint32_t s0 = s_runpre[a], n = s_runpre[a + 1] - s0, o = s_ost[a];
      const uint4* blk = s_blk + (a << lgTB);
      for (uint32_t j0 = g0; j0 < n; j0 += gw * kBtWU) {
        uint32_t bb[kBtWU];
        uint4 r[kBtWU];
        uint64_t k[kBtWU];
        double v[kBtWU];
#pragma unroll
        for (int u = 0; u < kBtWU; ++u) {
          const uint32_t j = j0 + u * gw;
          bb[u] = j < n ? sB[s0 + j] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kBtWU; ++u) r[u] = blk[bb[u]];
#pragma unroll
        for (int u = 0; u < kBtWU; ++u) {
          const uint32_t src = s0 + j0 + u * gw + r[u].x;
          k[u] = sK[src] + (((uint64_t)r[u].w << 32) | r[u].z);
          if (VALS) v[u] = sV[src];
        }
#pragma unroll
        for (int u = 0; u < kBtWU; ++u) {
          const uint32_t j = j0 + u * gw;
          if (j >= n) continue;
          keys_out[o + j] = k[u];
          if (VALS) vals_out[o + j] = v[u];
          if (perm_out) {
            const uint32_t p = s0 + j + r[u].x + r[u].y;
            perm_out[o + j] = idx_in ? __ldg(idx_in + p) : p;
          }
        }
      }
    }
    return;
  }
  // Tile larger than the stage (blocks of thousands of nonzeros: long runs anyway): per
  // nonzero, destination = position in its row + delta, written from registers; a
  // nonzero's block within its row is its own old block id minus the row's.
  if (tid < nblk) {
    const int b = tid >> lgTA, a = tid & (TA - 1);
    s_cnt[tid] = s_ost[a] + s_opre[(a << lgTB) + b] - s_ipre[tid];
  }
  __syncthreads();
  const int lgW = lgTB >= kBtLgWarps ? 0 : kBtLgWarps - lgTB;
  const uint32_t gw = 32u << lgW, g0 = ((warp & ((1 << lgW) - 1)) << 5) + lane;
  for (int b = warp >> lgW; b < TB; b += (kBtThreads / 32) >> lgW) {
    const uint32_t len = s_rowlen[b];
    const uint32_t rs = s_rs[b];
    const uint64_t id0 = base + (b0 + b) * strideB + a0;
    const uint32_t* dl = s_cnt + (b << lgTA);
    for (uint32_t r0 = 0; r0 < len; r0 += gw * kBtU) {
      uint64_t k[kBtU];
      double v[kBtU];
      uint32_t blk[kBtU];
#pragma unroll
      for (int u = 0; u < kBtU; ++u) {
        const uint32_t r = r0 + g0 + u * gw;
        k[u] = r < len ? __ldcs(keys_in + rs + r) : 0ull;
        if (VALS) v[u] = r < len ? __ldcs(vals_in + rs + r) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kBtU; ++u) blk[u] = (uint32_t)(fdiv(fF, k[u]) - id0);
      reencode_keys<kBtU>(kp, k);
#pragma unroll
      for (int u = 0; u < kBtU; ++u) {
        const uint32_t r = r0 + g0 + u * gw;
        if (r >= len) continue;
        const uint32_t d = r + dl[blk[u]];
        keys_out[d] = k[u];
        if (VALS) vals_out[d] = v[u];
        if (perm_out) perm_out[d] = idx_in ? __ldg(idx_in + rs + r) : rs + r;
      }
    }
  }
}

size_t block_ctrl_bytes(uint64_t nblocks) {
  const uint64_t nt = (nblocks + kBkTile - 1) / kBkTile;
  return 3 * ((nblocks * 4 + 255) / 256 * 256) + (nt * 4 + 255) / 256 * 256 + nt * 8 + 512;
}

cudaError_t run_block(const KeyPlan& kp, const KeyPlan& kb, uint64_t nblocks, uint64_t F,
                      const BlockGrid& bg, const PassIO& io, const Launch& L) {
  cudaError_t e;
  const uint64_t nnz = io.nnz;
  const size_t tb = (nblocks * 4 + 255) / 256 * 256;
  char* cb = reinterpret_cast<char*>(io.ctrl);
  uint32_t* bstart = reinterpret_cast<uint32_t*>(cb);
  uint32_t* bend = reinterpret_cast<uint32_t*>(cb + tb);
  uint32_t* cnew = reinterpret_cast<uint32_t*>(cb + 2 * tb);  // later: output starts
  const uint64_t nt = (nblocks + kBkTile - 1) / kBkTile;
  uint32_t* sums = reinterpret_cast<uint32_t*>(cb + 3 * tb);
  uint64_t* toff = reinterpret_cast<uint64_t*>(cb + 3 * tb + (nt * 4 + 255) / 256 * 256);
  uint64_t* total = toff + nt;
  const FastDiv fF = make_fastdiv(F);
  if ((e = cudaMemsetAsync(bstart, 0, 2 * tb, L.stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(sums, 0, nt * 4, L.stream)) != cudaSuccess) return e;
  // 16-byte key loads when the keys are 16-byte aligned (C4 bounds 0.090 -> 0.080 ms)
  if (L.mark) L.mark(L.ctx, "k_block_bounds");
  if ((reinterpret_cast<uintptr_t>(io.keys_in) & 15) == 0) {
    k_block_bounds<4><<<(unsigned)((nnz + 2047) / 2048), 256, 0, L.stream>>>(nnz, io.keys_in, fF, bstart, bend);
  } else {
    const unsigned gn = (unsigned)((nnz + 256 * kBkU - 1) / (256 * kBkU));  // 8 warps x 256
    k_block_bounds<<<gn, 256, 0, L.stream>>>(nnz, io.keys_in, fF, bstart, bend);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // counts in new order (32 x 32 transpose tiles) and the scan-tile sums
  BlockTiling gc;
  gc.dA = bg.dA;
  gc.dB = bg.dB;
  gc.lgTA = gc.lgTB = 5;
  const uint64_t ncA = (bg.dA + 31) >> 5, ncB = (bg.dB + 31) >> 5;
  const uint64_t nct = ncA * ncB * bg.mid * bg.hi;
  if (nct >= (1ull << 31)) return cudaErrorInvalidValue;
  gc.ntA = (uint32_t)ncA;
  gc.ntB = (uint32_t)ncB;
  gc.mid = (uint32_t)bg.mid;
  if (L.mark) L.mark(L.ctx, "k_block_counts");
  // 4 transpose tiles per CTA (C4 0.035 -> 0.032 ms; 2 per CTA: no change)
  k_block_counts<kBcT><<<(unsigned)((nct + kBcT - 1) / kBcT), 256, 0, L.stream>>>(gc, kb, (uint32_t)nct, bstart,
                                                                               bend, cnew, sums);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = run_count_scan(sums, nt, toff, total, L)) != cudaSuccess) return e;
  if (L.mark) L.mark(L.ctx, "k_scan_tiles");
  k_scan_tiles<<<(unsigned)nt, 256, 0, L.stream>>>(nblocks, cnew, toff);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // tile shape: about kBtTarget expected nonzeros, at most 32 x 32 blocks and 256 in all,
  // the longer side along B (the output runs)
  BlockTiling g;
  g.dA = bg.dA;
  g.dB = bg.dB;
  int lg = 0;
  const double avg = (double)nnz / (double)nblocks;
  while (lg < 8 && avg * (double)(2ull << lg) <= kBtTarget) ++lg;
  const int capA = umin64(ceil_log2(bg.dA), 5), capB = umin64(ceil_log2(bg.dB), 5);
  int lgB = umin64((lg + 1) / 2, capB);
  int lgA = umin64(lg - lgB, capA);
  lgB = umin64(lg - lgA, capB);
  g.lgTA = lgA;
  g.lgTB = lgB;
  const uint64_t ntA = (bg.dA + (1ull << lgA) - 1) >> lgA, ntB = (bg.dB + (1ull << lgB) - 1) >> lgB;
  const uint64_t ntiles = ntA * ntB * bg.mid * bg.hi;
  if (ntiles >= (1ull << 31)) return cudaErrorInvalidValue;
  g.ntA = (uint32_t)ntA;
  g.ntB = (uint32_t)ntB;
  g.mid = (uint32_t)bg.mid;
  const size_t smem = (size_t)kBtCap * 17;
  if (L.mark) L.mark(L.ctx, "k_block_tiles");
  auto fn = io.vals_out ? k_block_tiles<true> : k_block_tiles<false>;
  if ((e = kernel_setup(reinterpret_cast<const void*>(fn), smem, kBtThreads)) != cudaSuccess) return e;
  fn<<<(unsigned)ntiles, kBtThreads, smem, L.stream>>>(g, kp, kb, fF, io.keys_in, io.vals_in,
                                                       io.idx_in, bstart, bend, cnew, io.keys_out,
                                                       io.vals_out, io.perm_out);
  return cudaGetLastError();
}

}  // namespace lco
