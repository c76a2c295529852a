// device_common.cuh — device helpers shared by kernels.cu and msd.cu (internal).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lco_internal.h"

namespace lco {

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) {
  return a < b ? a : b;
}

constexpr int kThreads = 256;  // k_scatter / k_count CTA size (8 warps)
constexpr int kItems = 16;     // nonzeros per thread per tile
constexpr int kTile = kThreads * kItems;
// Large tiles of the unordered MSD passes (k_scatter UNST, one 1,024-thread CTA per SM):
// twice the records per digit run of a 4,096-record tile.
constexpr int kTileL = 8192;
constexpr int kChunkTiles = 64;  // max tiles per scan chunk

// Tiles per scan chunk: up to 64, fewer for small inputs so that k_offsets' running
// sums stay short and there are enough chunks to fill the GPU.
__host__ __device__ __forceinline__ uint32_t chunk_tiles(uint32_t tiles) {
  uint32_t c = tiles / 512;
  return c < 4 ? 4u : (c > (uint32_t)kChunkTiles ? (uint32_t)kChunkTiles : c);
}
constexpr int kScanThreads = 1024;  // k_scan: 32 bins x 32 chunk groups per CTA
constexpr uint32_t kInvalid = 0xFFFFu;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Lanes of the warp holding the same BITS-bit digit (0 for invalid lanes): one ballot
// per digit bit (ALU pipe), instead of MATCH.ANY (MIO pipe).
template <int BITS>
__device__ __forceinline__ uint32_t peers_of(uint32_t d, bool valid) {
  uint32_t m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const bool bit = (d >> b) & 1u;
    const uint32_t v = __ballot_sync(0xffffffffu, bit);
    m &= bit ? v : ~v;
  }
  return valid ? m : 0u;
}

// ---------------------------------------------------------------------------------
// Block-wide exclusive scan of BINS counters from `in` into `out`, NT threads.
// ---------------------------------------------------------------------------------
template <int NT, int BINS>
__device__ __forceinline__ void block_scan_bins(const uint32_t* in, uint32_t* out,
                                                uint32_t* s_warp) {
  constexpr int PER = BINS >= NT ? BINS / NT : 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t v[PER];
  uint32_t sum = 0;
  const bool active = tid * PER < BINS;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    v[i] = active ? in[tid * PER + i] : 0u;
    sum += v[i];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < NT / 32 ? s_warp[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < NT / 32) s_warp[lane] = wi - w;
  }
  __syncthreads();
  uint32_t run = s_warp[warp] + incl - sum;
  if (active) {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      out[tid * PER + i] = run;
      run += v[i];
    }
  }
  __syncthreads();
}

// Destination rank of a new key: number of splitters <= k2 (splitters ascending).
__device__ __forceinline__ uint32_t rank_of(const uint64_t* __restrict__ spl, int world,
                                            uint64_t k2) {
  int lo = 0, hi = world - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(spl + mid) <= k2) lo = mid + 1;
    else hi = mid;
  }
  return (uint32_t)lo;
}

// ---------------------------------------------------------------------------------
// Per-pass parameters shared by the pass kernels.
// ---------------------------------------------------------------------------------
// Segmented passes (MSD level 2): tiles never straddle a segment; the tile table lists
// every tile's element range and segment.
struct TileEntry {
  uint32_t start;
  uint32_t n;
  uint32_t seg;
  uint32_t pad;
};

struct PassParams {
  KeyPlan kp;
  int pass;
  int qshift;               // >= 0: q = K' >> qshift (T a power of two); -1: fast division
  uint64_t nnz;
  uint32_t tiles;
  uint32_t nchunks;
  uint32_t ctiles;            // tiles per scan chunk
  const uint64_t* splitters;  // partition mode: digit = destination rank
  int world;
  const TileEntry* ttab;      // segmented mode: tile table (else tiles are t * kTile)
  const uint32_t* ntiles;     // segmented mode: number of valid table entries
  uint32_t pf_dist;           // L2 prefetch distance in tiles (resident CTAs), 0 = off
  // LSD passes: k_count adds every tile's number of distinct digits here; k_scatter ranks
  // with match.any instead of one ballot per digit bit when tiles hold few distinct digits
  uint32_t* distinct;
  int adapt;  // host side: run_pass points `distinct` into its control block
  // MSD passes of lco_permute: slots inside a tile's digit run in any order (k_scatter
  // UNST); the leaves order records by (remaining q bits, K'), unique for unique keys
  int unstable;
  uint32_t tile;  // records per tile of unsegmented passes (0: kTile)
  int persist;    // persistent grid: each CTA loops over tiles (tile table length on device)
  int single;     // the whole input is one tile: its sorted order is the output order
  // sampled level 1 (msd.cu): the unordered first pass takes each tile's run bases from
  // per-digit cursors into capacity-padded buckets (no count / scan / offsets kernels);
  // a tile whose run would pass its bucket's end writes nothing and raises *overflow
  uint32_t* cursor;
  const uint32_t* cap_end;
  uint32_t* overflow;
  // the exact fallback of a sampled level 1: its kernels return at once unless *run_if
  const uint32_t* run_if;
};

// PER consecutive uint16 tile-histogram entries in, PER uint32 offsets out (vector
// loads / stores of one row slice; used by the offset kernels).
template <int PER>
struct RowVec;
template <>
struct RowVec<8> {
  __device__ static void load(const uint16_t* p, uint32_t (&h)[8]) {
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      h[2 * i] = w[i] & 0xFFFFu;
      h[2 * i + 1] = w[i] >> 16;
    }
  }
  __device__ static void store(uint32_t* p, const uint32_t (&r)[8]) {
    reinterpret_cast<uint4*>(p)[0] = make_uint4(r[0], r[1], r[2], r[3]);
    reinterpret_cast<uint4*>(p)[1] = make_uint4(r[4], r[5], r[6], r[7]);
  }
};
template <>
struct RowVec<4> {
  __device__ static void load(const uint16_t* p, uint32_t (&h)[4]) {
    const uint2 v = __ldcg(reinterpret_cast<const uint2*>(p));
    h[0] = v.x & 0xFFFFu;
    h[1] = v.x >> 16;
    h[2] = v.y & 0xFFFFu;
    h[3] = v.y >> 16;
  }
  __device__ static void store(uint32_t* p, const uint32_t (&r)[4]) {
    reinterpret_cast<uint4*>(p)[0] = make_uint4(r[0], r[1], r[2], r[3]);
  }
};
template <>
struct RowVec<1> {
  __device__ static void load(const uint16_t* p, uint32_t (&h)[1]) { h[0] = __ldcg(p); }
  __device__ static void store(uint32_t* p, const uint32_t (&r)[1]) { p[0] = r[0]; }
};

// Shaved key q = K' div T.
__device__ __forceinline__ uint64_t q_of(const PassParams& a, uint64_t k2) {
  return a.qshift >= 0 ? (k2 >> a.qshift) : fdiv(a.kp.divT, k2);
}

__device__ __forceinline__ uint32_t digit_new(const PassParams& a, uint64_t k2) {
  if (a.splitters) return rank_of(a.splitters, a.world, k2);
  return digit_of(a.kp, q_of(a, k2), a.pass);
}

// Digit extraction with the per-pass shift hoisted: for T a power of two the digit is a
// single shift-and-mask of K'.
struct DigitFn {
  int sh;         // >= 0: digit = (K' >> sh) & mask
  uint32_t mask;
  __device__ __forceinline__ DigitFn(const PassParams& a) {
    mask = (1u << a.kp.dbits[a.pass]) - 1u;
    sh = (a.qshift >= 0 && !a.splitters) ? a.qshift + a.kp.dshift[a.pass] : -1;
  }
  __device__ __forceinline__ uint32_t operator()(const PassParams& a, uint64_t k2) const {
    if (sh >= 0) return bm_window((uint32_t)k2, (uint32_t)(k2 >> 32), sh) & mask;
    return digit_new(a, k2);
  }
};

// LIV shuffle of N keys in registers: bit moves for power-of-two plans, fast division
// otherwise.
template <int N>
__device__ __forceinline__ void reencode_keys(const KeyPlan& p, uint64_t (&k)[N]) {
  if (p.pow2 && p.nmv > 0) reencode_moves<N>(p, k);
  else reencode_n<N>(p, k);
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// 16 bytes, cached in L2 only: no L1 line is held while the data is in flight
__device__ __forceinline__ void cp_async16_cg(uint32_t smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_dst), "l"(gsrc) : "memory");
}

__device__ __forceinline__ uint32_t smem_addr16(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// Stage n elements of E (4 or 8) bytes g[0..n) into s[0..n) with CTA threads tid / nt:
// where s and g are congruent mod 16, 16-byte L2-only copies for the aligned body and
// one-element copies for the head and tail (else one-element copies throughout).
template <int E>
__device__ __forceinline__ void stage_cg(void* s, const void* g, uint32_t n, int tid, int nt) {
  constexpr uint32_t PER = 16 / E;
  const uint32_t sa = smem_addr16(s);
  const char* gb = static_cast<const char*>(g);
  const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(gb) & 15u);
  const bool cong = ((reinterpret_cast<uintptr_t>(gb) ^ sa) & 15u) == 0;
  const uint32_t h = cong ? (uint32_t)umin64(n, mis ? (16u - mis) / E : 0u) : n;
  const uint32_t m = (n - h) / PER;  // 16-byte chunks
  {
    const uint32_t s0 = sa + h * E;
    const char* g0 = gb + (size_t)h * E;
    for (uint32_t c = tid; c < m; c += nt) cp_async16_cg(s0 + c * 16u, g0 + (size_t)c * 16u);
  }
  const uint32_t t0 = h + m * PER;
  char* sb = static_cast<char*>(s);
  for (uint32_t i = tid; i < h + (n - t0); i += nt) {  // head [0, h) and tail [t0, n)
    const uint32_t e = i < h ? i : t0 + (i - h);
    if (E == 8) cp_async8(sb + (size_t)e * 8, gb + (size_t)e * 8);
    else cp_async4(sb + (size_t)e * 4, gb + (size_t)e * 4);
  }
}
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on a shared-memory mbarrier.
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// orders this thread's (and, after a barrier, the CTA's) generic-proxy accesses of shared
// memory before later async-proxy (bulk copy) writes to it
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
// global [src, src + bytes) -> shared [dst, ...); 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
}

// One array of a staged range: n elements of E bytes at g go to shared memory at s0 + off
// elements (off makes shared and global addresses congruent mod 16; s0 has 16 / E spare
// slots): a 16-byte aligned body [h, t0) for one bulk copy, a head [0, h) and a tail
// [t0, n) of fewer than 16 / E elements each.
template <int E>
struct BulkPart {
  uint32_t off, h, t0;
  __device__ __forceinline__ BulkPart(const void* g, uint32_t n) {
    const uint32_t ga = (uint32_t)reinterpret_cast<uintptr_t>(g);
    off = (ga / E) & (16u / E - 1u);
    const uint32_t head = ((16u - (ga & 15u)) & 15u) / E;
    h = head < n ? head : n;
    t0 = h + ((n - h) * E / 16u) * (16u / E);
  }
  __device__ __forceinline__ uint32_t body_bytes() const { return (t0 - h) * E; }
  __device__ __forceinline__ uint32_t edge(uint32_t n) const { return h + (n - t0); }
  // i-th head / tail element (i < edge(n)) with a per-element cp.async
  __device__ __forceinline__ void copy_edge(uint32_t i, void* s0, const void* g) const {
    const uint32_t e = i < h ? i : t0 + (i - h);
    char* sd = static_cast<char*>(s0) + (size_t)(off + e) * E;
    const char* gs = static_cast<const char*>(g) + (size_t)e * E;
    if (E == 8) cp_async8(sd, gs);
    else cp_async4(sd, gs);
  }
};

// Bulk prefetch of [p, p + bytes) into L2 (no registers, no completion tracking).
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~(uintptr_t)15;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a))
               : "memory");
}

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Element range of tile t; false if t is past the end of a segmented table.
__device__ __forceinline__ bool tile_range(const PassParams& a, uint32_t t, uint64_t* base,
                                           uint32_t* n, uint32_t* seg) {
  if (a.ttab) {
    if (t >= *a.ntiles) return false;
    const TileEntry e = a.ttab[t];
    *base = e.start;
    *n = e.n;
    *seg = e.seg;
    return true;
  }
  const uint32_t tl = a.tile ? a.tile : (uint32_t)kTile;
  *base = (uint64_t)t * tl;
  *n = (uint32_t)umin64(tl, a.nnz - *base);
  *seg = t / a.ctiles;
  return true;
}

// Inputs / outputs of one k_scatter launch.
struct ScatterIO {
  const uint64_t* keys_in;  // FIRST pass inputs
  const double* vals_in;
  const uint32_t* idx_in;
  const uint64_t* kin;      // later-pass inputs (carried K', V, source position)
  const double* vin;
  const uint32_t* pin;
  uint64_t* kout;           // outputs (final arrays on the last pass)
  double* vout;
  uint32_t* pout;
  const uint32_t* toff;     // [tiles][BINS] from k_offsets
  int keep_old_key;         // partition: scatter the old key
  uint32_t idx_base;        // partition: added to single-pass source positions
  // partition straight into the receivers (lco_partition_direct): record w of digit d
  // (= destination rank) goes to dk[d][doff[d] + w], w = position - bucket[d]
  int direct;
  const uint32_t* bucket;
  uint64_t* dk[16];
  double* dv[16];
  uint32_t* dp[16];
  uint64_t doff[16];
};

}  // namespace lco
