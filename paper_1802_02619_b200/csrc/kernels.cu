// kernels.cu — sm_100a kernels of the LCO permutation hot path.
//
//   k_copy        identity after normalization: copy keys/values, perm = idx or iota
//                 ("no data movement" case)
//   k_hist        one read of the input keys: LIV shuffle + shaved key
//                 q = K' div T + digit histograms of all radix passes;
//                 the last CTA scans them into bucket starts
//   k_pass        one stable LSD radix pass over a digit of q ("stably
//                 sorted ... original relative ordering is used to break ties"):
//                 tile load -> (first pass) decode + re-encode -> warp match_any
//                 ranking -> decoupled look-back across tiles -> shared-memory reorder
//                 -> coalesced scatter; the last pass writes keys/perm and moves the
//                 values
//   k_partition   stable multisplit by new-key range for the sharded path (§8(e))
//   k_keyhist     histogram of the top bits of K' (splitter selection, §8(e))
//   k_validate    LCO_FLAG_VALIDATE precondition check
//
// No tensor cores: nothing here is a dense contraction (SURVEY.md §8(d) roofline is
// HBM bandwidth).
#include <cuda_runtime.h>

#include <cstdint>

#include "launch.h"
#include "lco_internal.h"

namespace lco {

static inline uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

constexpr int kThreads = 256;  // k_pass CTA size (8 warps)
constexpr int kItems = 16;     // nonzeros per thread per tile
constexpr int kTile = kThreads * kItems;
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 1u << 31;
constexpr uint32_t kValueMask = (1u << 30) - 1;
constexpr uint32_t kInvalid = 0xFFFFu;

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------------------------
// Block-wide exclusive scan of `bins` counters (in place into `out`), NT threads.
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
// k_hist: digit histograms of q = K' div T for every pass.
// ---------------------------------------------------------------------------------
struct HistArgs {
  KeyPlan kp;
  const uint64_t* keys;
  uint64_t nnz;
  uint32_t* ghist;     // [passes][bins], zeroed by the caller
  uint32_t* bucket;    // [passes][bins] exclusive scan (written by the last CTA)
  uint32_t* done;      // CTA completion counter, zeroed by the caller
  uint32_t* zero;      // region zeroed here (status of the first pass)
  uint64_t zero_words; // in uint32
  const uint64_t* splitters;  // partition mode: digit = destination rank (else null)
  int world;
  uint64_t* counts64;  // partition mode: per-rank counts (uint64), or null
};

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

constexpr int kHistThreads = 512;

template <int RB>
__global__ void __launch_bounds__(kHistThreads) k_hist(const __grid_constant__ HistArgs a) {
  constexpr int BINS = 1 << RB;
  extern __shared__ __align__(16) uint32_t sh[];  // [passes][BINS]
  __shared__ uint32_t s_warp[32];
  __shared__ bool s_last;
  const int P = a.kp.passes;
  const int tid = threadIdx.x;
  for (int i = tid; i < P * BINS; i += kHistThreads) sh[i] = 0;
  {  // zero the first pass's look-back status (overlaps with the histogram)
    const uint64_t stride = (uint64_t)gridDim.x * kHistThreads;
    for (uint64_t i = (uint64_t)blockIdx.x * kHistThreads + tid; i < a.zero_words; i += stride)
      a.zero[i] = 0;
  }
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * kHistThreads;
  constexpr int U = 4;
  for (uint64_t i0 = (uint64_t)blockIdx.x * kHistThreads * U + tid; i0 < a.nnz;
       i0 += stride * U) {
    uint64_t k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t i = i0 + (uint64_t)u * kHistThreads;
      k[u] = i < a.nnz ? __ldcs(a.keys + i) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t i = i0 + (uint64_t)u * kHistThreads;
      if (i < a.nnz) {
        const uint64_t k2 = reencode(a.kp, k[u]);
        if (a.splitters) {
          atomicAdd(&sh[rank_of(a.splitters, a.world, k2)], 1u);
        } else {
          const uint64_t q = fdiv(a.kp.divT, k2);
          for (int j = 0; j < P; ++j) atomicAdd(&sh[j * BINS + digit_of(a.kp, q, j)], 1u);
        }
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < P * BINS; i += kHistThreads) {
    uint32_t v = sh[i];
    if (v) atomicAdd(&a.ghist[i], v);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int j = 0; j < P; ++j) {
    for (int i = tid; i < BINS; i += kHistThreads) {
      sh[i] = __ldcg(a.ghist + j * BINS + i);
      if (a.counts64 && i < a.world) a.counts64[i] = sh[i];
    }
    __syncthreads();
    block_scan_bins<kHistThreads, BINS>(sh, a.bucket + j * BINS, s_warp);
  }
}

// ---------------------------------------------------------------------------------
// k_pass: one stable LSD pass (onesweep-style decoupled look-back).
// VMODE: 0 no values, 1 carry values through shared memory (single pass),
//        2 gather vals_in[position] in the last pass (multi-pass).
// ---------------------------------------------------------------------------------
struct PassArgs {
  KeyPlan kp;
  int pass;
  uint64_t nnz;
  // FIRST-pass inputs
  const uint64_t* keys_in;
  const double* vals_in;
  const uint32_t* idx_in;
  // later-pass inputs (carried new keys and source positions)
  const uint64_t* kin;
  const uint32_t* pin;
  // outputs: intermediate (kout, pout) or final (keys_out, perm_out, vals_out)
  uint64_t* kout;
  uint32_t* pout;
  double* vals_out;
  const uint32_t* bucket;  // [bins] exclusive digit starts of this pass
  uint32_t* status;        // [tiles][bins] look-back words of this pass (zeroed)
  uint32_t* status_next;   // [tiles][bins] to zero for the next pass, or null
  uint32_t* tile_counter;  // dynamic tile id (zeroed)
  const uint64_t* splitters;  // partition mode (single pass): digit = destination rank
  int world;
  int keep_old_key;        // partition mode: scatter the old key, not K'
  uint32_t idx_base;       // added to the source position in single-pass payloads
};

template <int RB>
constexpr size_t pass_smem_bytes() {
  return (size_t)kTile * 8 + (size_t)(kThreads / 32) * (1 << RB) * 2 + (size_t)(1 << RB) * 8 +
         (size_t)kTile * 2;
}

template <int RB, bool FIRST, bool LAST, int VMODE>
__global__ void __launch_bounds__(kThreads) k_pass(const __grid_constant__ PassArgs a) {
  constexpr int BINS = 1 << RB;
  constexpr int W = kThreads / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* stage = reinterpret_cast<uint64_t*>(smem);              // [kTile]
  uint16_t* whist = reinterpret_cast<uint16_t*>(stage + kTile);     // [W][BINS]
  uint32_t* tcount = reinterpret_cast<uint32_t*>(whist + W * BINS); // [BINS] -> global base
  uint32_t* toff = tcount + BINS;                                   // [BINS]
  uint16_t* sdig = reinterpret_cast<uint16_t*>(toff + BINS);        // [kTile]
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(a.tile_counter, 1u);
  for (int i = tid; i < W * BINS / 2; i += kThreads) reinterpret_cast<uint32_t*>(whist)[i] = 0u;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = (uint64_t)tile * kTile;
  const uint32_t n = (uint32_t)min((uint64_t)kTile, a.nnz - base);
  if (a.status_next)
    for (int i = tid; i < BINS; i += kThreads) a.status_next[(size_t)tile * BINS + i] = 0u;

  // ---- load the tile (warp w owns a contiguous slice; lane-consecutive elements) ----
  uint64_t key[kItems];
  uint32_t pay[kItems];  // payload: source position, or idx_in value (single pass)
  double val[VMODE == 1 ? kItems : 1];
  uint32_t meta[kItems];
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint32_t pos = warp * 32 * kItems + it * 32 + lane;
    const uint64_t i = base + pos;
    key[it] = 0;
    pay[it] = 0;
    if (pos < n) {
      if (FIRST) {
        key[it] = __ldcs(a.keys_in + i);
        if constexpr (VMODE == 1) val[it] = __ldcs(a.vals_in + i);
        if (LAST && a.idx_in) pay[it] = __ldcs(a.idx_in + i);
        else pay[it] = (uint32_t)i + (LAST ? a.idx_base : 0u);
      } else {
        key[it] = __ldcs(a.kin + i);
        pay[it] = __ldcs(a.pin + i);
      }
    }
  }
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint32_t pos = warp * 32 * kItems + it * 32 + lane;
    if (pos < n) {
      if (FIRST) {
        const uint64_t k2 = reencode(a.kp, key[it]);  // LIV shuffle
        if (a.splitters) {
          meta[it] = rank_of(a.splitters, a.world, k2);
          if (!a.keep_old_key) key[it] = k2;
        } else {
          key[it] = k2;
          meta[it] = digit_of(a.kp, fdiv(a.kp.divT, k2), a.pass);
        }
      } else {
        meta[it] = digit_of(a.kp, fdiv(a.kp.divT, key[it]), a.pass);
      }
    } else {
      meta[it] = kInvalid;
    }
  }
  // ---- warp-level stable ranking (match_any) into per-warp digit counters ----
  uint16_t* wh = whist + warp * BINS;
  const uint32_t ltm = lanemask_lt();
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint32_t d = meta[it];
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(peers) - 1;
    uint32_t before = 0;
    if (lane == leader && d != kInvalid) {
      before = wh[d];
      wh[d] = (uint16_t)(before + __popc(peers));
    }
    before = __shfl_sync(0xffffffffu, before, leader);
    meta[it] = d | ((before + __popc(peers & ltm)) << 16);
    __syncwarp();
  }
  __syncthreads();
  // ---- per-digit: exclusive prefix across warps, tile count ----
  for (int d = tid; d < BINS; d += kThreads) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t c = whist[w * BINS + d];
      whist[w * BINS + d] = (uint16_t)s;
      s += c;
    }
    tcount[d] = s;
    st_relaxed(a.status + (size_t)tile * BINS + d, (tile ? kFlagAgg : kFlagInc) | s);
  }
  __syncthreads();
  block_scan_bins<kThreads, BINS>(tcount, toff, s_warp);
  // ---- local (tile-sorted) positions; stage keys ----
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint32_t d = meta[it] & 0xFFFFu;
    if (d != kInvalid) {
      const uint32_t lp = toff[d] + whist[warp * BINS + d] + (meta[it] >> 16);
      stage[lp] = key[it];
      sdig[lp] = (uint16_t)d;
      meta[it] = d | (lp << 16);
    }
  }
  // ---- decoupled look-back per digit ----
  for (int d = tid; d < BINS; d += kThreads) {
    const uint32_t cnt = tcount[d];
    uint32_t excl = 0;
    if (tile > 0) {
      int64_t j = (int64_t)tile - 1;
      while (true) {
        const uint32_t s = ld_relaxed(a.status + (size_t)j * BINS + d);
        if ((s & (kFlagAgg | kFlagInc)) == 0) continue;
        excl += s & kValueMask;
        if (s & kFlagInc) break;
        --j;
      }
      st_relaxed(a.status + (size_t)tile * BINS + d, kFlagInc | (excl + cnt));
    }
    tcount[d] = a.bucket[d] + excl - toff[d];  // global position of local position 0 of d
  }
  __syncthreads();
  // ---- scatter keys (runs of equal digit are contiguous in stage) ----
  for (uint32_t p = tid; p < n; p += kThreads) a.kout[tcount[sdig[p]] + p] = stage[p];
  __syncthreads();
  uint32_t* stage32 = reinterpret_cast<uint32_t*>(stage);
#pragma unroll
  for (int it = 0; it < kItems; ++it)
    if ((meta[it] & 0xFFFFu) != kInvalid) stage32[meta[it] >> 16] = pay[it];
  __syncthreads();
  for (uint32_t p = tid; p < n; p += kThreads) {
    const uint32_t dst = tcount[sdig[p]] + p;
    const uint32_t v = stage32[p];
    if (!LAST) {
      a.pout[dst] = v;
    } else if (FIRST) {
      if (a.pout) a.pout[dst] = v;
    } else {
      if (a.pout) a.pout[dst] = a.idx_in ? __ldg(a.idx_in + v) : v;
      if constexpr (VMODE == 2) a.vals_out[dst] = __ldg(a.vals_in + v);
    }
  }
  if constexpr (VMODE == 1) {
    __syncthreads();
    double* stage64 = reinterpret_cast<double*>(stage);
#pragma unroll
    for (int it = 0; it < kItems; ++it)
      if ((meta[it] & 0xFFFFu) != kInvalid) stage64[meta[it] >> 16] = val[it];
    __syncthreads();
    for (uint32_t p = tid; p < n; p += kThreads) a.vals_out[tcount[sdig[p]] + p] = stage64[p];
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
template <int RB>
static cudaError_t set_smem_attrs() {
  static bool done = false;
  if (done) return cudaSuccess;
  const int bytes = (int)pass_smem_bytes<RB>();
  cudaError_t e = cudaSuccess;
#define LCO_ATTR(F, L, V)                                                                  \
  e = cudaFuncSetAttribute(k_pass<RB, F, L, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           bytes);                                                         \
  if (e != cudaSuccess) return e;
  LCO_ATTR(true, true, 0)
  LCO_ATTR(true, true, 1)
  LCO_ATTR(true, false, 0)
  LCO_ATTR(false, false, 0)
  LCO_ATTR(false, true, 0)
  LCO_ATTR(false, true, 2)
#undef LCO_ATTR
  e = cudaFuncSetAttribute(k_hist<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kMaxPasses * (1 << RB) * 4);
  if (e != cudaSuccess) return e;
  done = true;
  return cudaSuccess;
}

template <int RB>
static cudaError_t run_onesweep_rb(const KeyPlan& kp, const OnesweepIO& io, const Launch& L) {
  constexpr int BINS = 1 << RB;
  cudaError_t e = set_smem_attrs<RB>();
  if (e != cudaSuccess) return e;
  const bool part = io.splitters != nullptr;
  const int P = part ? 1 : kp.passes;
  const uint64_t nnz = io.nnz;
  const uint64_t tiles = (nnz + kTile - 1) / kTile;
  uint32_t* ghist = io.ctrl;
  uint32_t* bucket = io.ctrl + kMaxPasses * BINS;
  uint32_t* counters = bucket + kMaxPasses * BINS;  // [kMaxPasses] tile counters, [done]
  uint32_t* done = counters + kMaxPasses;
  const size_t ctrl_bytes = (size_t)(2 * kMaxPasses * BINS + kMaxPasses + 1) * 4;
  if (L.mark) L.mark(L.ctx, "memset_ctrl");
  e = cudaMemsetAsync(io.ctrl, 0, ctrl_bytes, L.stream);
  if (e != cudaSuccess) return e;
  KeyPlan kpp = kp;
  if (part) kpp.passes = 1;
  {
    HistArgs h;
    h.kp = kpp;
    h.keys = io.keys_in;
    h.nnz = nnz;
    h.ghist = ghist;
    h.bucket = bucket;
    h.done = done;
    h.zero = io.statusA;
    h.zero_words = tiles * BINS;
    h.splitters = io.splitters;
    h.world = io.world;
    h.counts64 = io.counts64;
    int grid = (int)umin64((nnz + kHistThreads * 4 - 1) / (kHistThreads * 4), 148 * 2);
    if (grid < 1) grid = 1;
    if (L.mark) L.mark(L.ctx, "k_hist");
    k_hist<RB><<<grid, kHistThreads, P * BINS * 4, L.stream>>>(h);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const size_t smem = pass_smem_bytes<RB>();
  for (int j = 0; j < P; ++j) {
    PassArgs p;
    p.kp = kpp;
    p.pass = j;
    p.nnz = nnz;
    p.keys_in = io.keys_in;
    p.vals_in = io.vals_in;
    p.idx_in = io.idx_in;
    p.kin = (j % 2 == 1) ? io.kA : io.kB;
    p.pin = (j % 2 == 1) ? io.pA : io.pB;
    const bool last = j == P - 1;
    p.kout = last ? io.keys_out : ((j % 2 == 0) ? io.kA : io.kB);
    p.pout = last ? io.perm_out : ((j % 2 == 0) ? io.pA : io.pB);
    p.vals_out = io.vals_out;
    p.bucket = bucket + j * BINS;
    p.status = (j % 2 == 0) ? io.statusA : io.statusB;
    p.status_next = last ? nullptr : ((j % 2 == 0) ? io.statusB : io.statusA);
    p.tile_counter = counters + j;
    p.splitters = io.splitters;
    p.world = io.world;
    p.keep_old_key = part ? 1 : 0;
    p.idx_base = io.idx_base;
    if (L.mark)
      L.mark(L.ctx, part ? "k_partition" : (P == 1 ? "k_pass_single" : (j == 0 ? "k_pass_first" : (last ? "k_pass_last" : "k_pass_mid"))));
    const dim3 grid((unsigned)tiles);
    if (P == 1) {
      if (io.vals_out) k_pass<RB, true, true, 1><<<grid, kThreads, smem, L.stream>>>(p);
      else k_pass<RB, true, true, 0><<<grid, kThreads, smem, L.stream>>>(p);
    } else if (j == 0) {
      k_pass<RB, true, false, 0><<<grid, kThreads, smem, L.stream>>>(p);
    } else if (!last) {
      k_pass<RB, false, false, 0><<<grid, kThreads, smem, L.stream>>>(p);
    } else {
      if (io.vals_out) k_pass<RB, false, true, 2><<<grid, kThreads, smem, L.stream>>>(p);
      else k_pass<RB, false, true, 0><<<grid, kThreads, smem, L.stream>>>(p);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

size_t onesweep_ctrl_bytes(int rb) {
  return (size_t)(2 * kMaxPasses * (1 << rb) + kMaxPasses + 1) * 4;
}
uint64_t onesweep_tiles(uint64_t nnz) { return (nnz + kTile - 1) / kTile; }
int onesweep_tile() { return kTile; }

cudaError_t run_onesweep(int rb, const KeyPlan& kp, const OnesweepIO& io, const Launch& L) {
  switch (rb) {
    case 8: return run_onesweep_rb<8>(kp, io, L);
    case 10: return run_onesweep_rb<10>(kp, io, L);
    case 11: return run_onesweep_rb<11>(kp, io, L);
  }
  return cudaErrorInvalidValue;
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
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_keyhist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         16384 * 4);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = (int)umin64((nnz + 511) / 512, 148 * 2);
  k_keyhist<<<grid > 0 ? grid : 1, 512, (size_t)bins * 4, s>>>(
      kp, keys, nnz, shift, bins, reinterpret_cast<unsigned long long*>(counts));
  return cudaGetLastError();
}

}  // namespace lco
