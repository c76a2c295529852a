// kernels.cu — sm_100a kernels of the LCO permutation hot path.
//
// One stable radix pass over a digit of the shaved key q = K' div T is a
// tile-granular reduce-then-scan:
//   k_count    per tile (4096 nonzeros): LIV shuffle on the first pass,
//              digit, tile histogram (row of thist) and, per chunk of tiles,
//              the chunk sums;
//   k_scan     per digit, exclusive scan of the chunk sums; the last CTA turns the digit
//              totals into bucket starts;
//   k_offsets  per chunk, per digit: running sum over the chunk's tile rows -> the global
//              position of each tile's first nonzero of each digit (toff);
//   k_scatter  per tile, in launch order: load -> (first pass) decode + re-encode ->
//              warp ranking with ballots -> shared-memory reorder -> coalesced scatter of
//              keys, values and source positions to toff + rank.  Tiles are ranked stably
//              and their offsets come from the exclusive scan, so the pass is stable
//              ("original relative ordering is used to break ties"); no
//              CTA waits on another.
// Other kernels:
//   k_copy     identity after normalization
//   k_keyhist  histogram of the top bits of K' (splitter selection, §8(e))
//   k_validate LCO_FLAG_VALIDATE precondition check
//
// No tensor cores: nothing here is a dense contraction (HBM bound).
// Measured alternatives that were replaced: a decoupled
// look-back (onesweep) pass, whose look-back chain over 1024-2048 bins advanced a few
// tiles per L2 round trip; static per-CTA chunks, whose 296 x bins write frontiers
// overflowed L2 write combining (1.8x DRAM write traffic); match_any ranking, which is
// MIO-bound on sm_100a.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "device_common.cuh"
#include "launch.h"
#include "lco_internal.h"

namespace lco {

// ---------------------------------------------------------------------------------
// k_copy
// ---------------------------------------------------------------------------------
__global__ void k_copy(uint64_t nnz, const uint64_t* __restrict__ keys_in,
                       const double* __restrict__ vals_in, const uint32_t* __restrict__ idx_in,
                       uint64_t* __restrict__ keys_out, double* __restrict__ vals_out,
                       uint32_t* __restrict__ perm_out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    keys_out[i] = keys_in[i];
    if (vals_out) vals_out[i] = vals_in[i];
    if (perm_out) perm_out[i] = idx_in ? idx_in[i] : (uint32_t)i;
  }
}

// ---------------------------------------------------------------------------------
// k_count: one tile per CTA: tile histogram -> thist[t][BINS] (uint16) and added into
// its chunk's sums csum[t / ctiles][BINS] (segmented mode: into its segment's
// totals csum[seg][BINS]); csum is zeroed by the launcher.
// ---------------------------------------------------------------------------------
template <int RB, bool FIRST, bool ADAPT = false, int ITEMS = kItems, bool PERSIST = false>
__global__ void __launch_bounds__(kThreads) k_count(const __grid_constant__ PassParams a,
                                                    const uint64_t* __restrict__ keys,
                                                    uint16_t* __restrict__ thist,
                                                    uint32_t* __restrict__ csum) {
  constexpr int BINS = 1 << RB;
  __shared__ uint32_t h[BINS];
  if (a.run_if && *a.run_if == 0u) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // one tile per CTA, or (a.persist: tile tables whose length only the device knows)
  // tiles blockIdx.x, + gridDim.x, ... of a persistent grid
  for (uint32_t t = blockIdx.x; !PERSIST || t < a.tiles; t += gridDim.x) {
  uint64_t base;
  uint32_t n, seg;
  if (!tile_range(a, t, &base, &n, &seg)) return;
  if (tid == 0 && a.pf_dist && !PERSIST) {
    // the keys of the tile pf_dist CTAs later into L2 (C5 first count 0.77 -> 0.66 ms)
    const uint32_t t2 = t + a.pf_dist;
    uint64_t b2 = 0;
    uint32_t m = 0;
    if (!a.ttab) {
      const uint32_t tl = a.tile ? a.tile : (uint32_t)kTile;
      b2 = (uint64_t)t2 * tl;
      m = b2 < a.nnz ? (uint32_t)umin64(tl, a.nnz - b2) : 0u;
    } else if (t2 < *a.ntiles) {
      const TileEntry e2 = a.ttab[t2];
      b2 = e2.start;
      m = e2.n;
    }
    if (m) prefetch_l2(keys + b2, (size_t)m * 8);
  }
  for (int i = tid; i < BINS; i += kThreads) h[i] = 0;
  const DigitFn dg(a);
  // pow2 first pass: the digit is a few bit fields of the OLD key, no full shuffle
  const bool direct = FIRST && !a.splitters && a.kp.ndmv[a.pass] >= 0;
  __syncthreads();
  // keys loaded per round: first passes (a few bit moves per key) run more CTAs per SM
  // with 2 (C5 count 0.97 -> 0.76 ms); later passes keep 8 (4: 0.71 -> 0.75 ms)
  constexpr int H = FIRST ? 2 : kItems / 2;
#pragma unroll
  for (int half = 0; half < ITEMS / H; ++half) {
    uint64_t k[H];
#pragma unroll
    for (int it = 0; it < H; ++it) {
      const uint32_t pos = warp * 32 * ITEMS + (half * H + it) * 32 + lane;
      k[it] = pos < n ? __ldcs(keys + base + pos) : 0ull;
    }
    if (direct) {
#pragma unroll
      for (int it = 0; it < H; ++it) {
        const uint32_t pos = warp * 32 * ITEMS + (half * H + it) * 32 + lane;
        if (pos < n) atomicAdd(&h[digit_from_old(a.kp, a.pass, k[it])], 1u);
      }
      continue;
    }
    if (FIRST) reencode_keys<H>(a.kp, k);  // LIV shuffle
#pragma unroll
    for (int it = 0; it < H; ++it) {
      const uint32_t pos = warp * 32 * ITEMS + (half * H + it) * 32 + lane;
      // plain shared atomics: a histogram needs no order (conflicting lanes of a warp
      // are serialized by the hardware, which only costs on long runs of equal digits)
      if (pos < n) atomicAdd(&h[dg(a, k[it])], 1u);
    }
  }
  __syncthreads();
  uint16_t* row = thist + (size_t)t * BINS;
  uint32_t* cs = csum + (size_t)seg * BINS;  // chunk sums, or segment totals (segmented)
  for (int d = tid; d < BINS; d += kThreads) {
    const uint32_t v = h[d];
    if (thist) row[d] = (uint16_t)v;  // (null: cursor-based scatter, totals only)
    if (v) atomicAdd(cs + d, v);
  }
  if (ADAPT && (t & 31u) == 0) {  // distinct digits of every 32nd tile
    uint32_t nz = 0;
    for (int d = tid; d < BINS; d += kThreads) nz += h[d] != 0u;
    nz = __reduce_add_sync(0xffffffffu, nz);
    if (lane == 0 && nz) atomicAdd(a.distinct, nz);
  }
  if (!PERSIST) return;
  __syncthreads();  // h is zeroed for the next tile
  }
}

// ---------------------------------------------------------------------------------
// k_scan: csum[c][d] <- sum_{c' < c} csum[c'][d] (in place); totals; the last CTA
// turns the totals into bucket starts (and an optional uint64 copy of the totals).
// ---------------------------------------------------------------------------------
template <int RB>
__global__ void __launch_bounds__(kScanThreads) k_scan(uint32_t* __restrict__ csum,
                                                       uint32_t nchunks,
                                                       uint32_t* __restrict__ totals,
                                                       uint32_t* __restrict__ bucket,
                                                       uint32_t* __restrict__ done,
                                                       uint64_t* __restrict__ counts64,
                                                       int ncounts, const uint32_t* run_if) {
  constexpr int BINS = 1 << RB;
  if (run_if && *run_if == 0u) return;
  constexpr int LANES = BINS >= 32 ? 32 : BINS;  // bins per CTA (one warp-wide row)
  constexpr int SPLIT = kScanThreads / LANES;    // chunk groups per bin
  __shared__ uint32_t part[kScanThreads];
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t sh[BINS];
  __shared__ bool s_last;
  const int tid = threadIdx.x;
  const int d = blockIdx.x * LANES + tid % LANES;
  const int g = tid / LANES;
  const uint32_t per = (nchunks + SPLIT - 1) / SPLIT;
  const uint32_t c0 = min(nchunks, g * per), c1 = min(nchunks, c0 + per);
  // the first RC chunk sums stay in registers for the write-back; the rest are re-read in
  // batches of 8 (a load-then-store loop over csum serializes one L2 round trip per
  // chunk: the store may alias the next load)
  constexpr int RC = 24;
  uint32_t cache[RC];
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < RC; ++i) {
    cache[i] = c0 + i < c1 ? __ldcg(csum + (size_t)(c0 + i) * BINS + d) : 0u;
    sum += cache[i];
  }
#pragma unroll 8
  for (uint32_t c = c0 + RC; c < c1; ++c) sum += __ldcg(csum + (size_t)c * BINS + d);
  part[tid] = sum;
  __syncthreads();
  uint32_t run = 0;
  for (int g2 = 0; g2 < g; ++g2) run += part[g2 * LANES + tid % LANES];
#pragma unroll
  for (int i = 0; i < RC; ++i) {
    if (c0 + i < c1) {
      csum[(size_t)(c0 + i) * BINS + d] = run;
      run += cache[i];
    }
  }
  for (uint32_t c = c0 + RC; c < c1; c += 8) {
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = c + u < c1 ? __ldcg(csum + (size_t)(c + u) * BINS + d) : 0u;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (c + u < c1) {
        csum[(size_t)(c + u) * BINS + d] = run;
        run += v[u];
      }
    }
  }
  if (g == SPLIT - 1) totals[d] = run;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int i = tid; i < BINS; i += kScanThreads) {
    sh[i] = __ldcg(totals + i);
    if (counts64 && i < ncounts) counts64[i] = sh[i];
  }
  __syncthreads();
  block_scan_bins<kScanThreads, BINS>(sh, bucket, s_warp);
}

// ---------------------------------------------------------------------------------
// k_offsets: toff[t][d] = bucket[d] + csum[c][d] + sum of thist rows before t in c.
// Thread = PER consecutive digits (vector loads of the u16 rows, vector stores of the
// offsets); rows are fetched four at a time so the loads overlap.
// ---------------------------------------------------------------------------------
template <int RB>
__global__ void __launch_bounds__(kThreads) k_offsets(const __grid_constant__ PassParams a,
                                                      const uint16_t* __restrict__ thist,
                                                      const uint32_t* __restrict__ csum,
                                                      const uint32_t* __restrict__ bucket,
                                                      uint32_t* __restrict__ toff) {
  if (a.run_if && *a.run_if == 0u) return;
  constexpr int BINS = 1 << RB;
  constexpr int PER = BINS / kThreads;
  static_assert(PER == 1 || PER == 4 || PER == 8, "digit widths 8, 10, 11");
  constexpr int U = 4;
  const uint32_t c = blockIdx.x;
  const uint32_t t0 = c * a.ctiles, t1 = min(a.tiles, t0 + a.ctiles);
  const int d0 = threadIdx.x * PER;
  uint32_t run[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i)
    run[i] = __ldg(bucket + d0 + i) + __ldcg(csum + (size_t)c * BINS + d0 + i);
  for (uint32_t t = t0; t < t1; t += U) {
    uint32_t h[U][PER];
#pragma unroll
    for (int r = 0; r < U; ++r) {
      if (t + r < t1) RowVec<PER>::load(thist + (size_t)(t + r) * BINS + d0, h[r]);
    }
#pragma unroll
    for (int r = 0; r < U; ++r) {
      if (t + r < t1) {
        RowVec<PER>::store(toff + (size_t)(t + r) * BINS + d0, run);
#pragma unroll
        for (int i = 0; i < PER; ++i) run[i] += h[r][i];
      }
    }
  }
}

// ---------------------------------------------------------------------------------
// k_scatter: one tile per CTA.
//   rank    every warp ranks its 512 nonzeros in input order: match.any finds the lanes
//           holding the same digit, per-warp u16 counters give the running count, so
//           rank = (earlier warps, earlier items, earlier lanes) = the stable order;
//   stage   keys go to shared memory at their tile-sorted slot; values and source
//           positions are gathered straight from global memory into their slots with
//           cp.async (no registers, the loads fly during the bookkeeping);
//   write   one loop writes K', V and the position of each slot to toff + rank:
//           consecutive threads write consecutive slots, i.e. runs of equal digit.
// Shared memory: sK [tile] u64 | sV [tile] f64 (holds the per-warp counters while
// ranking) | sP [tile] u32 | gbase [bins] u32 | loff [bins] u32 | (first unordered pass:
// counters [bins] u32, slot -> input position [tile] u16) | sdig [tile] u16, left out
// in passes after the first when the write loop shifts the digit out of the staged K'
// (power-of-two T; the L1 keeps the 16 KB: C5 level-2 pass 6.71 -> 6.28 ms, C3b middle
// pass -5 %; first passes measured slower with the dependent load).
// ---------------------------------------------------------------------------------
constexpr int scatter_nt(int rb, int tile = kTile) {
  return tile > kTile ? 1024 : (rb <= 10 ? 512 : 256);
}

// The write loop of a pass after the first takes a slot's digit from its staged K' (a
// shift: q = K' >> qshift) instead of a staged copy; the launch then leaves out the sdig
// array (more L1).
__host__ __device__ inline bool scatter_keydig(const PassParams& a) {
  return a.qshift >= 0 && !a.splitters;
}

template <int RB, int TILE = kTile, bool EARLY = false>
constexpr size_t scatter_smem_bytes() {
  // EARLY: + the digit counters [bins] u32 and the slot -> input position map [tile] u16
  // + 2 / 2 / 4 spare slots of sK / sV / sP: a tile staged in input order sits at an
  // offset that makes its shared and global addresses congruent mod 16 (stage_cg)
  return (size_t)TILE * (8 + 8 + 4 + 2) + 48 + (size_t)(1 << RB) * 8 +
         (EARLY ? (size_t)TILE * 2 + (size_t)(1 << RB) * 4 : 0);
}

// NT threads (IT = kTile / NT nonzeros each): 512 for digits of <= 10 bits (more warps
// in flight per SM, half the serial work per thread), 256 for 11-bit digits (whose
// per-warp counters would not fit in sV with 16 warps).
// UNST (MSD passes of lco_permute, unique keys): the order inside a tile's digit run is
// free, because every leaf sorts its records on (remaining bits of q, K') and K' is unique
// -- so a record takes its slot with one shared atomic (no per-warp counters, no ballots).
template <int RB, bool FIRST, bool LAST, bool VALS, int NT, bool ADAPT = false, bool UNST = false,
          int TILE = kTile>
__global__ void __launch_bounds__(NT, (NT >= 1024 ? 1 : 2))
    k_scatter(const __grid_constant__ PassParams a, const __grid_constant__ ScatterIO io) {
  constexpr int BINS = 1 << RB;
  constexpr int W = NT / 32;
  constexpr int IT = TILE / NT;
  constexpr int NB = BINS >= NT ? BINS / NT : 1;
  static_assert(UNST || W * BINS * 2 <= TILE * 8, "warp counters must fit in sV");
  // unordered passes: V (and P) in input order, loaded with the keys, gathered by slot in
  // the write loop -- first pass per-lane cp.async (C5 4.66 -> 4.24 ms), later passes
  // 16-byte L2-only copies that hold no L1 lines (C5 level 2 6.28 -> 5.90 ms; the same
  // with per-lane copies was slower, 7.44)
  constexpr bool EARLY = UNST;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* const sK0 = reinterpret_cast<uint64_t*>(smem);       // [TILE + 2]
  double* const sV0 = reinterpret_cast<double*>(sK0 + TILE + 2);  // [TILE + 2]
  uint16_t* whist = reinterpret_cast<uint16_t*>(sV0);             // [W][BINS] (ranking only)
  uint32_t* const sP0 = reinterpret_cast<uint32_t*>(sV0 + TILE + 2);  // [TILE + 4]
  uint32_t* gbase = reinterpret_cast<uint32_t*>(sP0 + TILE + 4);  // [BINS]
  uint32_t* loff = gbase + BINS;                                  // [BINS]
  // EARLY: V stays in input order (loaded at the start of the tile, in flight during the
  // ranking); sidx maps a slot to its input position
  uint32_t* ucnt = loff + BINS;                                   // [BINS] (EARLY)
  uint16_t* sidx = reinterpret_cast<uint16_t*>(ucnt + (EARLY ? BINS : 0));  // [TILE] (EARLY)
  // slot digits, last: absent (not allocated) when the write loop takes the digit from
  // the staged key (a shift of K', scatter_keydig)
  uint16_t* sdig = sidx + (EARLY ? TILE : 0);                     // [TILE]
  const bool kdig = !FIRST && scatter_keydig(a) && !io.direct && !io.keep_old_key;
  __shared__ uint32_t s_warp[32];
  __shared__ int s_ovf;
  if (a.run_if && *a.run_if == 0u) return;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // one tile per CTA, or (a.persist) tiles blockIdx.x, + gridDim.x, ... of a persistent grid
  for (uint32_t t = blockIdx.x; t < a.tiles; t += gridDim.x) {
  uint64_t base;
  uint32_t n, seg;
  if (!tile_range(a, t, &base, &n, &seg)) return;
  // tiles staged in input order with 16-byte copies sit at offsets congruent to their
  // global addresses mod 16 (else stage_cg falls back to one copy per element)
  uint64_t* sK = sK0;
  double* sV = sV0;
  uint32_t* sP = sP0;
  if (EARLY && !FIRST) {
    sK += (reinterpret_cast<uintptr_t>(io.kin + base) >> 3) & 1u;
    if (VALS) sV += (reinterpret_cast<uintptr_t>(io.vin + base) >> 3) & 1u;
    if (io.pout != nullptr) sP += (reinterpret_cast<uintptr_t>(io.pin + base) >> 2) & 3u;
  }
  if (tid == 0 && a.pf_dist) {
    // the tile the CTA launched pf_dist later will load: bring it into L2 now, so its
    // loads see L2 latency while HBM streams in the background
    const uint32_t t2 = t + a.pf_dist;
    uint64_t b2 = 0;
    uint32_t m = 0;
    if (!a.ttab) {
      b2 = (uint64_t)t2 * TILE;
      m = b2 < a.nnz ? (uint32_t)umin64(TILE, a.nnz - b2) : 0u;
    } else if (t2 < *a.ntiles) {
      const TileEntry e2 = a.ttab[t2];
      b2 = e2.start;
      m = e2.n;
    }
    if (m) {
      prefetch_l2((FIRST ? io.keys_in : io.kin) + b2, (size_t)m * 8);
      if (VALS) prefetch_l2((FIRST ? io.vals_in : io.vin) + b2, (size_t)m * 8);
      if (!FIRST && io.pout) prefetch_l2(io.pin + b2, (size_t)m * 4);
      if (io.toff) prefetch_l2(io.toff + (size_t)t2 * BINS, (size_t)BINS * 4);
    }
  }
  // global offsets of this tile's digit runs (from the exclusive scan): issued first, so
  // their latency hides behind the tile's loads (C5 level 2: 7.7 % of stall samples)
  uint32_t tv[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int d = tid + b * NT;
    tv[b] = (d < BINS && !a.single && !a.cursor) ? __ldcs(io.toff + (size_t)t * BINS + d) : 0u;
  }
  if (FIRST && UNST && tid == 0) s_ovf = 0;
  // UNST digit counters: their own array when V is staged early, else inside sV
  uint32_t* cnt = EARLY ? ucnt : reinterpret_cast<uint32_t*>(whist);
  if (UNST) {
    for (int i = tid; i < BINS; i += NT) cnt[i] = 0u;
  } else {
    for (int i = tid; i < W * BINS / 2; i += NT) reinterpret_cast<uint32_t*>(whist)[i] = 0u;
  }
  // ---- load keys; warp w owns a contiguous slice, lanes consecutive ----
  uint64_t key[IT];
  uint32_t meta[IT];
  if (EARLY && !FIRST) {
    // 16-byte L2-only copies in input order: the keys (one group, read back into
    // registers below), then V and P (still in flight while the keys are ranked)
    stage_cg<8>(sK, io.kin + base, n, tid, NT);
    cp_async_commit();
    if (VALS) stage_cg<8>(sV, io.vin + base, n, tid, NT);
    if (io.pout != nullptr) stage_cg<4>(sP, io.pin + base, n, tid, NT);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t pos = warp * 32 * IT + it * 32 + lane;
      key[it] = pos < n ? sK[pos] : 0ull;  // slots overwrite sK only after the ranking barrier
    }
  } else {
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t pos = warp * 32 * IT + it * 32 + lane;
      key[it] = pos < n ? __ldcs((FIRST ? io.keys_in : io.kin) + base + pos) : 0ull;
    }
  }
  if (EARLY && !FIRST) {
  } else if (EARLY) {  // values in input order, in flight while the keys are ranked
    const bool want_p0 = !FIRST && io.pout != nullptr;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t pos = warp * 32 * IT + it * 32 + lane;
      if (pos < n) {
        if (VALS) cp_async8(sV + pos, (FIRST ? io.vals_in : io.vin) + base + pos);
        if (want_p0) cp_async4(sP + pos, io.pin + base + pos);
      }
    }
    cp_async_commit();
  }
  // global offsets of this tile's digit runs (loaded at the top of the tile)
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int d = tid + b * NT;
    if (d < BINS) gbase[d] = tv[b];
  }
  {
    const DigitFn dg(a);
    if (FIRST && io.keep_old_key) {  // partition: route by K', move the old key
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const uint32_t pos = warp * 32 * IT + it * 32 + lane;
        meta[it] = pos < n ? dg(a, reencode(a.kp, key[it])) : kInvalid;
      }
    } else {
      if (FIRST) {  // LIV shuffle, in place, two rounds
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint64_t kk[IT / 2];
#pragma unroll
          for (int i = 0; i < IT / 2; ++i) kk[i] = key[half * (IT / 2) + i];
          reencode_keys<IT / 2>(a.kp, kk);
#pragma unroll
          for (int i = 0; i < IT / 2; ++i) key[half * (IT / 2) + i] = kk[i];
        }
      }
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const uint32_t pos = warp * 32 * IT + it * 32 + lane;
        meta[it] = pos < n ? dg(a, key[it]) : kInvalid;
      }
    }
  }
  __syncthreads();
  if (UNST) {
    // ---- unordered slots: one shared atomic per record on the tile's digit counter;
    // tiles with few distinct digits aggregate a warp's equal digits first (match.any)
    const bool few = ADAPT && *a.distinct < (uint64_t)((a.tiles + 31) / 32) *
                                                ((1u << a.kp.dbits[a.pass]) / 8);
    if (few) {
      const uint32_t ltm = lanemask_lt();
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const uint32_t d = meta[it];
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t base = 0;
        if (d != kInvalid && (peers & ltm) == 0) base = atomicAdd(&cnt[d], (uint32_t)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, __ffs(peers) - 1);
        if (d != kInvalid) meta[it] = d | ((base + __popc(peers & ltm)) << 16);
      }
    } else {
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const uint32_t d = meta[it];
        if (d != kInvalid) meta[it] = d | (atomicAdd(&cnt[d], 1u) << 16);
      }
    }
    __syncthreads();
    block_scan_bins<NT, BINS>(cnt, loff, s_warp);
    if (a.cursor) {
      // this tile's run of digit d from the digit's cursor: sampled level 1 (one row;
      // a run past its bucket's capacity raises the overflow), or the segmented level 2
      // (one row per level-1 bucket, exact totals: no per-tile offsets)
      uint32_t* crow = a.cursor + (FIRST ? 0u : (size_t)seg * BINS);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int d = tid + b * NT;
        if (d < BINS) {
          const uint32_t c = cnt[d];
          uint32_t g0 = 0;
          if (c) {
            g0 = atomicAdd(crow + d, c);
            if (FIRST && (g0 + c > a.cap_end[d] || g0 + c < g0)) s_ovf = 1;
          }
          gbase[d] = g0;
        }
      }
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t d = meta[it] & 0xFFFFu;
      if (d != kInvalid) {
        const uint32_t lp = loff[d] + (meta[it] >> 16);
        sK[lp] = key[it];
        if (!kdig) sdig[lp] = (uint16_t)d;
        if (EARLY) sidx[lp] = (uint16_t)(warp * 32 * IT + it * 32 + lane);
        meta[it] = d | (lp << 16);
      }
    }
  } else {
  // ---- warp-level stable ranking into per-warp digit counters ----
  uint16_t* wh = whist + warp * BINS;
  const uint32_t ltm = lanemask_lt();
  // few distinct digits per tile (structured keys): match.any, whose cost grows with the
  // distinct values per warp, beats one ballot per digit bit
  const bool few = ADAPT && *a.distinct < (uint64_t)((a.tiles + 31) / 32) *
                                              ((1u << a.kp.dbits[a.pass]) / 8);  // < 1/8 used
  // lanes holding the same digit: for <= 10-bit digits one ballot per digit bit (ALU
  // pipe; match.any goes through the MIO queue and its latency dominated the 8-bit
  // ranking loop on random keys, ncu: +25 % on C5); for 11-bit digits, or tiles with few
  // distinct digits, match.any (12 ballots cost more: -6 % on C4).  One loop per method,
  // chosen once per tile, so each keeps its own register allocation.
  auto rank_item = [&](int it, uint32_t peers) {
    const uint32_t d = meta[it];
    const bool ok = d != kInvalid;
    peers &= ok ? 0xffffffffu : 0u;
    const uint32_t below = __popc(peers & ltm);
    const uint32_t before = ok ? (uint32_t)wh[d] : 0u;  // every peer reads the same counter
    __syncwarp();
    if (ok && below == 0) wh[d] = (uint16_t)(before + __popc(peers));
    meta[it] = d | ((before + below) << 16);
    __syncwarp();
  };
  if (RB >= 11 || (ADAPT && few)) {
#pragma unroll
    for (int it = 0; it < IT; ++it) rank_item(it, __match_any_sync(0xffffffffu, meta[it]));
  } else {
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t d = meta[it];
      uint32_t peers = __ballot_sync(0xffffffffu, d != kInvalid);
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        const uint32_t bit = (d >> b) & 1u;
        peers &= __ballot_sync(0xffffffffu, bit) ^ (bit - 1u);
      }
      rank_item(it, peers);
    }
  }
  __syncthreads();
  // ---- per digit: exclusive prefix across warps, tile count ----
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int d = tid + b * NT;
    if (d < BINS) {
      uint32_t s = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const uint32_t cw = whist[w * BINS + d];
        whist[w * BINS + d] = (uint16_t)s;
        s += cw;
      }
      loff[d] = s;
    }
  }
  __syncthreads();
  block_scan_bins<NT, BINS>(loff, loff, s_warp);
  // ---- local (tile-sorted) slots; stage keys and digits ----
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const uint32_t d = meta[it] & 0xFFFFu;
    if (d != kInvalid) {
      const uint32_t lp = loff[d] + whist[warp * BINS + d] + (meta[it] >> 16);
      sK[lp] = key[it];
      if (!kdig) sdig[lp] = (uint16_t)d;
      meta[it] = d | (lp << 16);
    }
  }
  }  // stable ranking
  __syncthreads();  // the warp counters (in sV) are dead from here on
  // ---- gather values / positions into their slots (cp.async, global -> shared) ----
  const bool want_p = io.pout != nullptr || io.direct;
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    if (EARLY) break;  // loaded in input order above
    if ((meta[it] & 0xFFFFu) == kInvalid) continue;
    const uint32_t pos = warp * 32 * IT + it * 32 + lane;
    const uint32_t lp = meta[it] >> 16;
    if (VALS) cp_async8(sV + lp, (FIRST ? io.vals_in : io.vin) + base + pos);
    if (want_p) {
      if (FIRST) {
        if (LAST && io.idx_in) cp_async4(sP + lp, io.idx_in + base + pos);
        else sP[lp] = (uint32_t)(base + pos) + (LAST ? io.idx_base : 0u);
      } else {
        cp_async4(sP + lp, io.pin + base + pos);
      }
    }
  }
  cp_async_commit();
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int d = tid + b * NT;
    if (d < BINS) {
      // global position of local slot 0 of digit d (single tile: the tile order is final)
      gbase[d] = a.single ? 0u : gbase[d] - loff[d];
      if (io.direct) gbase[d] -= io.bucket[d];  // ... within its destination's chunk
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  if (FIRST && UNST && a.cursor && s_ovf) {  // a bucket overflowed: the exact path redoes it
    if (tid == 0) atomicOr(a.overflow, 1u);
    return;
  }
  // ---- one write loop: K', V, position of each slot ----
  const bool remap = !FIRST && LAST && io.idx_in != nullptr;
  if (io.direct) {  // partition: the scatter IS the exchange (stores to peer memory)
    for (uint32_t p = tid; p < n; p += NT) {
      const uint32_t d = sdig[p];
      const uint64_t w = io.doff[d] + (uint32_t)(gbase[d] + p);  // gbase wraps mod 2^32
      io.dk[d][w] = sK[p];
      if (VALS) io.dv[d][w] = sV[p];
      io.dp[d][w] = sP[p];
    }
  } else {
    const DigitFn dgw(a);
    if (EARLY) {
      for (uint32_t p = tid; p < n; p += NT) {
        const uint64_t k = sK[p];
        const uint32_t g = gbase[kdig ? dgw(a, k) : (uint32_t)sdig[p]] + p;
        const uint32_t src = sidx[p];
        io.kout[g] = k;
        if (VALS) io.vout[g] = sV[src];
        if (io.pout) io.pout[g] = FIRST ? (uint32_t)(base + src) : sP[src];
      }
    } else
    for (uint32_t p = tid; p < n; p += NT) {
      const uint64_t k = sK[p];
      const uint32_t g = gbase[kdig ? dgw(a, k) : (uint32_t)sdig[p]] + p;
      io.kout[g] = k;
      if (VALS) io.vout[g] = sV[p];
      if (want_p) {
        const uint32_t v = sP[p];
        io.pout[g] = remap ? __ldg(io.idx_in + v) : v;
      }
    }
  }
  if (!a.persist) return;
  __syncthreads();  // the stage is reused by the next tile
  }
}

// ---------------------------------------------------------------------------------
// k_validate: flag[0] |= 1 if keys not strictly increasing, 2 if a key >= total.
// ---------------------------------------------------------------------------------
__global__ void k_validate(uint64_t nnz, const uint64_t* __restrict__ keys, uint64_t total,
                           int need_sorted, uint32_t* flag) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t f = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const uint64_t k = keys[i];
    if (k >= total) f |= 2u;
    if (need_sorted && i > 0 && keys[i - 1] >= k) f |= 1u;
  }
  if (f) atomicOr(flag, f);
}

// ---------------------------------------------------------------------------------
// k_keyhist: counts[K' >> shift] += 1 (splitter selection for the sharded path).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_keyhist(const __grid_constant__ KeyPlan kp,
                                                 const uint64_t* __restrict__ keys,
                                                 uint64_t nnz, int shift, int bins,
                                                 unsigned long long* counts) {
  extern __shared__ uint32_t hk[];
  for (int i = threadIdx.x; i < bins; i += blockDim.x) hk[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const uint64_t b = reencode(kp, __ldcs(keys + i)) >> shift;
    atomicAdd(&hk[b < (uint64_t)bins ? b : bins - 1], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bins; i += blockDim.x)
    if (hk[i]) atomicAdd(counts + i, (unsigned long long)hk[i]);
}

// ---------------------------------------------------------------------------------
// Launchers (called from api.cu)
// ---------------------------------------------------------------------------------
uint64_t pass_tiles(uint64_t nnz, uint32_t tile) { return (nnz + tile - 1) / tile; }

// L2 prefetch distance of the pass kernels: one wave of resident CTAs (2 per SM), so a
// CTA brings the tile its successor on the same SM will load into L2 (measured: -3 to
// -6 % on the C4 / C5 / C3a passes).
uint32_t prefetch_distance() {
  int sms = 148;
  if (device_sms(&sms) != cudaSuccess) sms = 148;
  return (uint32_t)sms;
}
int pass_tile() { return kTile; }
int pass_rb(int bits) { return bits <= 8 ? 8 : (bits <= 10 ? 10 : 11); }

// control block: thist (uint16 [tiles][bins]) | toff ([tiles][bins]) | csum ([chunks][bins])
//                | totals | bucket | counter
size_t pass_ctrl_bytes(int rb, uint64_t nnz, uint32_t tile) {
  const uint64_t tiles = pass_tiles(nnz, tile);
  const uint64_t chunks = (tiles + chunk_tiles((uint32_t)tiles) - 1) / chunk_tiles((uint32_t)tiles);
  const size_t bins = (size_t)1 << rb;
  return (tiles * bins * 2 + 255) / 256 * 256 + tiles * bins * 4 + (chunks + 2) * bins * 4 + 512;
}

PassCtrl pass_ctrl_layout(int rb, uint64_t nnz, uint32_t* ctrl, uint32_t tile) {
  PassCtrl c;
  const uint32_t tiles = (uint32_t)pass_tiles(nnz, tile);
  const uint32_t nchunks = (tiles + chunk_tiles(tiles) - 1) / chunk_tiles(tiles);
  const size_t bins = (size_t)1 << rb;
  char* cb = reinterpret_cast<char*>(ctrl);
  c.thist = reinterpret_cast<uint16_t*>(cb);
  cb += ((size_t)tiles * bins * 2 + 255) / 256 * 256;
  c.toff = reinterpret_cast<uint32_t*>(cb);
  cb += (size_t)tiles * bins * 4;
  c.csum = reinterpret_cast<uint32_t*>(cb);
  c.totals = c.csum + (size_t)nchunks * bins;
  c.bucket = c.totals + bins;
  c.done = c.bucket + bins;
  c.tiles = tiles;
  c.nchunks = nchunks;
  return c;
}

template <int RB, int ITEMS>
static cudaError_t launch_count_t(bool first, const PassParams& a, const uint64_t* keys,
                                  uint16_t* thist, uint32_t* csum, uint32_t grid, cudaStream_t s) {
  if (a.persist) {  // table-driven later passes (MSD level 3), sampled level 1's fallback
    if (first) k_count<RB, true, false, ITEMS, true><<<grid, kThreads, 0, s>>>(a, keys, thist, csum);
    else k_count<RB, false, false, ITEMS, true><<<grid, kThreads, 0, s>>>(a, keys, thist, csum);
    return cudaGetLastError();
  }
  if (a.distinct) {
    if (first) k_count<RB, true, true, ITEMS><<<grid, kThreads, 0, s>>>(a, keys, thist, csum);
    else k_count<RB, false, true, ITEMS><<<grid, kThreads, 0, s>>>(a, keys, thist, csum);
  } else if (first) {
    k_count<RB, true, false, ITEMS><<<grid, kThreads, 0, s>>>(a, keys, thist, csum);
  } else {
    k_count<RB, false, false, ITEMS><<<grid, kThreads, 0, s>>>(a, keys, thist, csum);
  }
  return cudaGetLastError();
}

template <int RB>
static cudaError_t launch_count_rb(bool first, const PassParams& a, const uint64_t* keys,
                                   uint16_t* thist, uint32_t* csum, uint32_t grid, cudaStream_t s) {
  if (a.tile == (uint32_t)kTileL)
    return launch_count_t<RB, kTileL / kThreads>(first, a, keys, thist, csum, grid, s);
  return launch_count_t<RB, kItems>(first, a, keys, thist, csum, grid, s);
}

cudaError_t launch_count(int rb, bool first, const PassParams& a, const uint64_t* keys,
                         uint16_t* thist, uint32_t* csum, uint32_t grid, cudaStream_t s) {
  switch (rb) {
    case 8: return launch_count_rb<8>(first, a, keys, thist, csum, grid, s);
    case 10: return launch_count_rb<10>(first, a, keys, thist, csum, grid, s);
    case 11: return launch_count_rb<11>(first, a, keys, thist, csum, grid, s);
  }
  return cudaErrorInvalidValue;
}

template <int RB, bool F, bool LST>
static cudaError_t launch_scatter_t(bool vals, const PassParams& a, const ScatterIO& io,
                                   uint32_t grid, cudaStream_t s) {
  constexpr int NT = scatter_nt(RB);
  // no sdig array (the last one) when the write loop takes digits from the keys
  const bool kdig = !F && scatter_keydig(a) && !io.direct && !io.keep_old_key;
  size_t smem = scatter_smem_bytes<RB>() - (kdig ? (size_t)kTile * 2 : 0);
  void (*fn)(const PassParams, const ScatterIO);
  if (a.unstable && !LST && a.tile == (uint32_t)kTileL) {  // large tiles, one CTA per SM
    constexpr int NL = scatter_nt(RB, kTileL);
    smem = scatter_smem_bytes<RB, kTileL, true>() - (kdig ? (size_t)kTileL * 2 : 0);
    fn = vals ? k_scatter<RB, F, false, true, NL, false, true, kTileL>
              : k_scatter<RB, F, false, false, NL, false, true, kTileL>;
    cudaError_t e = kernel_setup(reinterpret_cast<const void*>(fn), smem, NL);
    if (e != cudaSuccess) return e;
    fn<<<grid, NL, smem, s>>>(a, io);
    return cudaGetLastError();
  }
  if (a.unstable && !LST) {  // MSD passes of lco_permute (the last pass is never one)
    smem = scatter_smem_bytes<RB, kTile, true>() - (kdig ? (size_t)kTile * 2 : 0);
    if (a.distinct) fn = vals ? k_scatter<RB, F, false, true, NT, true, true> : k_scatter<RB, F, false, false, NT, true, true>;
    else fn = vals ? k_scatter<RB, F, false, true, NT, false, true> : k_scatter<RB, F, false, false, NT, false, true>;
  } else if (a.distinct) {
    fn = vals ? k_scatter<RB, F, LST, true, NT, true> : k_scatter<RB, F, LST, false, NT, true>;
  } else {
    fn = vals ? k_scatter<RB, F, LST, true, NT> : k_scatter<RB, F, LST, false, NT>;
  }
  cudaError_t e = kernel_setup(reinterpret_cast<const void*>(fn), smem, NT);
  if (e != cudaSuccess) return e;
  fn<<<grid, NT, smem, s>>>(a, io);
  return cudaGetLastError();
}

template <int RB>
static cudaError_t launch_scatter_rb(bool first, bool last, bool vals, const PassParams& a,
                                     const ScatterIO& io, uint32_t grid, cudaStream_t s) {
  if (first && last) return launch_scatter_t<RB, true, true>(vals, a, io, grid, s);
  if (first) return launch_scatter_t<RB, true, false>(vals, a, io, grid, s);
  if (!last) return launch_scatter_t<RB, false, false>(vals, a, io, grid, s);
  return launch_scatter_t<RB, false, true>(vals, a, io, grid, s);
}

// The whole input as one tile of up to kTileL records sorted on a digit of <= 10 bits:
// one stable pass of one 1,024-thread CTA whose tile order is the final order (no
// count / scan / offsets kernels: C1-sized tensors are launch-latency bound).
template <int RB>
static cudaError_t launch_single_t(bool vals, const PassParams& a, const ScatterIO& io,
                                   cudaStream_t s) {
  constexpr int NL = scatter_nt(RB, kTileL);
  constexpr size_t smem = scatter_smem_bytes<RB, kTileL>();
  auto fn = vals ? k_scatter<RB, true, true, true, NL, false, false, kTileL>
                 : k_scatter<RB, true, true, false, NL, false, false, kTileL>;
  cudaError_t e = kernel_setup(reinterpret_cast<const void*>(fn), smem, NL);
  if (e != cudaSuccess) return e;
  fn<<<1, NL, smem, s>>>(a, io);
  return cudaGetLastError();
}

cudaError_t run_single_tile(int rb, const KeyPlan& kp, const PassIO& io, const Launch& L) {
  PassParams a;
  memset(&a, 0, sizeof a);
  a.kp = kp;
  a.kp.passes = 1;
  a.qshift = kp.divT.kind == 1 ? (int)kp.divT.s : (kp.divT.kind == 0 ? 0 : -1);
  a.nnz = io.nnz;
  a.tile = kTileL;
  a.tiles = 1;
  a.single = 1;
  ScatterIO sio = pass_buffers(io, 0, true, nullptr);
  if (L.mark) L.mark(L.ctx, "k_scatter_single_tile");
  switch (rb) {
    case 8: return launch_single_t<8>(io.vals_out != nullptr, a, sio, L.stream);
    case 10: return launch_single_t<10>(io.vals_out != nullptr, a, sio, L.stream);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_scatter(int rb, bool first, bool last, bool vals, const PassParams& a,
                           const ScatterIO& io, uint32_t grid, cudaStream_t s) {
  switch (rb) {
    case 8: return launch_scatter_rb<8>(first, last, vals, a, io, grid, s);
    case 10: return launch_scatter_rb<10>(first, last, vals, a, io, grid, s);
    case 11: return launch_scatter_rb<11>(first, last, vals, a, io, grid, s);
  }
  return cudaErrorInvalidValue;
}

// Buffers of pass j: read set (j-1)%2, write set j%2 (A = 0, B = 1); the first pass reads
// the inputs, the last writes the outputs.
ScatterIO pass_buffers(const PassIO& io, int j, bool last, const uint32_t* toff) {
  ScatterIO s;
  memset(&s, 0, sizeof s);
  s.keys_in = io.keys_in;
  s.vals_in = io.vals_in;
  s.idx_in = io.idx_in;
  s.kin = (j % 2 == 1) ? io.kA : io.kB;
  s.vin = (j % 2 == 1) ? io.vA : io.vB;
  s.pin = (j % 2 == 1) ? io.pA : io.pB;
  s.kout = last ? io.keys_out : ((j % 2 == 0) ? io.kA : io.kB);
  s.vout = last ? io.vals_out : ((j % 2 == 0) ? io.vA : io.vB);
  s.pout = last ? io.perm_out : ((j % 2 == 0) ? io.pA : io.pB);
  s.toff = toff;
  s.keep_old_key = io.splitters ? 1 : 0;
  s.idx_base = io.idx_base;
  return s;
}

// One unsegmented pass: count -> scan -> offsets -> scatter (count_only: stop after the
// scan, leaving digit totals and bucket starts in the control block).
cudaError_t run_pass(int rb, const PassParams& a0, const PassIO& io, int j, bool first,
                     bool last, const Launch& L, bool count_only) {
  const int BINS = 1 << rb;
  const uint32_t tile = a0.tile ? a0.tile : (uint32_t)kTile;
  const PassCtrl c = pass_ctrl_layout(rb, io.nnz, io.ctrl, tile);
  PassParams a = a0;
  a.tile = tile;
  a.pass = j;
  a.tiles = c.tiles;
  a.nchunks = c.nchunks;
  a.ctiles = chunk_tiles(c.tiles);
  cudaError_t e;
  const bool part = io.splitters != nullptr;
  if ((e = cudaMemsetAsync(c.csum, 0, ((size_t)c.nchunks * BINS + 2 * BINS) * 4 + 8, L.stream)) !=
      cudaSuccess)
    return e;  // chunk sums, totals, bucket starts, k_scan's completion counter, distinct
  if (a0.adapt) a.distinct = c.done + 1;  // LSD passes (run_passes) only
  const uint64_t* in_keys = first ? io.keys_in : ((j % 2 == 1) ? io.kA : io.kB);
  // a persistent pass (the predicated fallback of a sampled level 1, usually a no-op):
  // grids of a few CTAs per SM loop over the tiles
  uint32_t gcount = c.tiles, gscat = c.tiles;
  if (a.persist) {
    int sms = 148;
    if ((e = device_sms(&sms)) != cudaSuccess) return e;
    gcount = c.tiles < (uint32_t)sms * 8u ? c.tiles : (uint32_t)sms * 8u;
    gscat = c.tiles < (uint32_t)sms * 2u ? c.tiles : (uint32_t)sms * 2u;
  }
  if (L.mark) L.mark(L.ctx, first ? "k_count_first" : "k_count");
  if ((e = launch_count(rb, first, a, in_keys, c.thist, c.csum, gcount, L.stream)) != cudaSuccess)
    return e;
  if (L.mark) L.mark(L.ctx, "k_scan");
  const int scan_grid = BINS >= 32 ? BINS / 32 : 1;
  switch (rb) {
    case 8:
      k_scan<8><<<scan_grid, kScanThreads, 0, L.stream>>>(c.csum, c.nchunks, c.totals, c.bucket,
                                                          c.done, part ? io.counts64 : nullptr,
                                                          io.world, a.run_if);
      break;
    case 10:
      k_scan<10><<<scan_grid, kScanThreads, 0, L.stream>>>(c.csum, c.nchunks, c.totals, c.bucket,
                                                           c.done, part ? io.counts64 : nullptr,
                                                           io.world, a.run_if);
      break;
    case 11:
      k_scan<11><<<scan_grid, kScanThreads, 0, L.stream>>>(c.csum, c.nchunks, c.totals, c.bucket,
                                                           c.done, part ? io.counts64 : nullptr,
                                                           io.world, a.run_if);
      break;
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (count_only) return cudaSuccess;
  if (L.mark) L.mark(L.ctx, "k_offsets");
  switch (rb) {
    case 8: k_offsets<8><<<c.nchunks, kThreads, 0, L.stream>>>(a, c.thist, c.csum, c.bucket, c.toff); break;
    case 10: k_offsets<10><<<c.nchunks, kThreads, 0, L.stream>>>(a, c.thist, c.csum, c.bucket, c.toff); break;
    case 11: k_offsets<11><<<c.nchunks, kThreads, 0, L.stream>>>(a, c.thist, c.csum, c.bucket, c.toff); break;
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ScatterIO s = pass_buffers(io, j, last, c.toff);
  if (io.direct) {
    s.direct = 1;
    s.bucket = c.bucket;
    for (int d = 0; d < kMaxDirect && d < BINS; ++d) {
      s.dk[d] = io.direct->k[d];
      s.dv[d] = io.direct->v[d];
      s.dp[d] = io.direct->p[d];
      s.doff[d] = io.direct->off[d];
    }
  }
  if (L.mark)
    L.mark(L.ctx, part ? "k_partition"
                       : (first && last ? "k_scatter_single"
                                        : (first ? "k_scatter_first"
                                                 : (last ? "k_scatter_last" : "k_scatter_mid"))));
  return launch_scatter(rb, first, last, io.vals_out != nullptr, a, s, gscat, L.stream);
}

// Stable LSD radix sort over all passes of the key plan (or one partition pass).
cudaError_t run_passes(int rb, const KeyPlan& kp, const PassIO& io, const Launch& L) {
  const bool part = io.splitters != nullptr;
  const int P = part ? 1 : kp.passes;
  PassParams a;
  memset(&a, 0, sizeof a);
  a.kp = kp;
  a.pf_dist = prefetch_distance();
  if (part) a.kp.passes = 1;
  a.qshift = kp.divT.kind == 1 ? (int)kp.divT.s : (kp.divT.kind == 0 ? 0 : -1);
  a.nnz = io.nnz;
  a.splitters = io.splitters;
  a.world = io.world;
  // LSD passes choose their ranking from the distinct digits per tile (k_count samples)
  a.adapt = !part && !(io.tune && io.tune->no_match);
  for (int j = 0; j < P; ++j) {
    cudaError_t e = run_pass(rb, a, io, j, j == 0, j == P - 1, L);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t run_partition(int rb, const KeyPlan& kp, const PassIO& io, const Launch& L,
                          bool count_only) {
  PassParams a;
  memset(&a, 0, sizeof a);
  a.kp = kp;
  a.kp.passes = 1;
  a.pf_dist = prefetch_distance();
  a.qshift = kp.divT.kind == 1 ? (int)kp.divT.s : (kp.divT.kind == 0 ? 0 : -1);
  a.nnz = io.nnz;
  a.splitters = io.splitters;
  a.world = io.world;
  return run_pass(rb, a, io, 0, true, true, L, count_only);
}

cudaError_t run_copy(uint64_t nnz, const uint64_t* keys_in, const double* vals_in,
                     const uint32_t* idx_in, uint64_t* keys_out, double* vals_out,
                     uint32_t* perm_out, const Launch& L) {
  if (L.mark) L.mark(L.ctx, "k_copy");
  const int grid = (int)umin64((nnz + 255) / 256, 148 * 16);
  k_copy<<<grid, 256, 0, L.stream>>>(nnz, keys_in, vals_in, idx_in, keys_out, vals_out,
                                     perm_out);
  return cudaGetLastError();
}

cudaError_t run_validate(uint64_t nnz, const uint64_t* keys, uint64_t total, int need_sorted,
                         uint32_t* flag, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(flag, 0, 4, s);
  if (e != cudaSuccess) return e;
  const int grid = (int)umin64((nnz + 255) / 256, 148 * 8);
  k_validate<<<grid > 0 ? grid : 1, 256, 0, s>>>(nnz, keys, total, need_sorted, flag);
  return cudaGetLastError();
}

cudaError_t run_keyhist(const KeyPlan& kp, uint64_t nnz, const uint64_t* keys, int shift,
                        int bins, uint64_t* counts, cudaStream_t s) {
  cudaError_t e = kernel_setup(reinterpret_cast<const void*>(k_keyhist), 16384 * 4, 0);
  if (e != cudaSuccess) return e;
  const int grid = (int)umin64((nnz + 511) / 512, 148 * 2);
  k_keyhist<<<grid > 0 ? grid : 1, 512, (size_t)bins * 4, s>>>(
      kp, keys, nnz, shift, bins, reinterpret_cast<unsigned long long*>(counts));
  return cudaGetLastError();
}

}  // namespace lco
