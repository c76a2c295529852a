// lco_internal.h — plan structures shared by the host planner (plan.cpp), the C ABI
// (api.cu) and the kernels (kernels.cu).  Not part of the public ABI.
#pragma once

#include <cstddef>
#include <cstdint>

#include "../../include/lco.h"

#if defined(__CUDACC__)
#define LCO_HD __host__ __device__ __forceinline__
#else
#define LCO_HD inline
#endif

namespace lco {

// ---------------------------------------------------------------------------------
// FastDiv: exact unsigned 64-bit division by a runtime-invariant divisor, the role
// libdivide plays in the paper ("we use a fast division library",
// PAPER.md:249).  Written from the Granlund-Montgomery round-up method: for d not a
// power of two, l = ceil(log2 d), m = floor(2^64 (2^l - d) / d) + 1, and
//   q = (t + ((x - t) >> 1)) >> (l - 1),  t = mulhi(m, x),
// exact for every x < 2^64.  Powers of two use a shift.
// ---------------------------------------------------------------------------------
struct FastDiv {
  uint64_t d;
  uint64_t m;
  uint32_t s;
  uint32_t kind;  // 0: d == 1, 1: power of two (x >> s), 2: magic with add
};

LCO_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

LCO_HD uint64_t fdiv(const FastDiv& f, uint64_t x) {
  if (f.kind == 1) return x >> f.s;
  if (f.kind == 0) return x;
  uint64_t t = mulhi64(f.m, x);
  return (t + ((x - t) >> 1)) >> f.s;
}

FastDiv make_fastdiv(uint64_t d);  // host (plan.cpp); d >= 1

// ---------------------------------------------------------------------------------
// Device-side plan: everything a kernel needs to turn an old key K into the new key
// K' and the sort key q = K' div T (the shaved key), and to cut q into radix digits.
// ---------------------------------------------------------------------------------
constexpr int kMaxModes = LCO_MAX_ORDER;
constexpr int kMaxPasses = 8;
constexpr int kMaxMoves = 40;       // bit moves of a power-of-two LIV shuffle
constexpr int kMaxDigitMoves = 12;  // bit moves that build one radix digit of q

// One bit-field move of a power-of-two LIV shuffle, in 32-bit words: take the 32-bit
// window of the old key starting at bit `a`, keep the low bits under `mask`, and add
// them at bit `b` of output word `hi` (0: bits 0-31, 1: bits 32-63).  Fields never
// overlap, so add == or.  The host splits every mode's field so that no move crosses
// an output word (build_moves, plan.cpp).
struct BitMove {
  uint32_t mask;
  uint8_t a;
  uint8_t hi;
  uint8_t b;
  uint8_t pad;
};

struct KeyPlan {
  int n;                          // normalized order (>= 2 on the radix path)
  FastDiv div[kMaxModes];         // div[m] divides by n_m (old normalized mode m)
  uint64_t dim[kMaxModes];        // n_m
  uint64_t nstride[kMaxModes];    // new-key stride of old mode m
  FastDiv divT;                   // q = K' div T
  int pow2;                       // 1: every normalized dim is a power of two
  uint8_t oshift[kMaxModes];      // pow2: bit offset of mode m in the old key
  uint8_t nshift[kMaxModes];      // pow2: bit offset of mode m in the new key
  uint8_t width[kMaxModes];       // pow2: log2 n_m
  uint64_t omask[kMaxModes];      // pow2: n_m - 1
  int passes;                     // P
  int dshift[kMaxPasses];         // digit j = (q >> dshift[j]) & ((1 << dbits[j]) - 1)
  int dbits[kMaxPasses];
  // pow2 plans: the shuffle as word-local bit moves, and every digit of q straight from
  // the OLD key (so a histogram of the first pass never builds K'); ndmv[j] < 0: the
  // digit needs the full shuffle.  Filled by build_moves / build_digit_moves.
  int nmv;
  BitMove mv[kMaxMoves];
  int ndmv[kMaxPasses];
  BitMove dmv[kMaxPasses][kMaxDigitMoves];
};

#if defined(__CUDACC__)
// 32-bit window of the key (hi:lo) starting at bit a (0..63).
__device__ __forceinline__ uint32_t bm_window(uint32_t lo, uint32_t hi, int a) {
  return a < 32 ? __funnelshift_r(lo, hi, a) : (hi >> (a - 32));
}

// LIV shuffle of N keys by bit moves (pow2 plans): two 32-bit output words per key.
template <int N>
__device__ __forceinline__ void reencode_moves(const KeyPlan& p, uint64_t (&k)[N]) {
  uint32_t olo[N], ohi[N];
#pragma unroll
  for (int i = 0; i < N; ++i) olo[i] = ohi[i] = 0u;
#pragma unroll 1
  for (int j = 0; j < p.nmv; ++j) {
    const BitMove m = p.mv[j];
    const uint32_t mul = 1u << m.b;
    // one 64-bit funnel shift per key (a = 0..63), mask, multiply-add into its word
    if (m.hi) {
#pragma unroll
      for (int i = 0; i < N; ++i) ohi[i] += ((uint32_t)(k[i] >> m.a) & m.mask) * mul;
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) olo[i] += ((uint32_t)(k[i] >> m.a) & m.mask) * mul;
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) k[i] = ((uint64_t)ohi[i] << 32) | olo[i];
}

// Digit `pass` of q straight from an OLD key (pow2 plans, p.ndmv[pass] >= 0).
__device__ __forceinline__ uint32_t digit_from_old(const KeyPlan& p, int pass, uint64_t k) {
  const uint32_t lo = (uint32_t)k, hi = (uint32_t)(k >> 32);
  uint32_t d = 0;
#pragma unroll 1
  for (int j = 0; j < p.ndmv[pass]; ++j) {
    const BitMove m = p.dmv[pass][j];
    d += (bm_window(lo, hi, m.a) & m.mask) << m.b;
  }
  return d;
}
#endif

// LIV shuffle of one key: decode old coordinates from the last mode
// with fast division, accumulate the new key with the new strides.
LCO_HD uint64_t reencode(const KeyPlan& p, uint64_t k) {
  if (p.pow2) {  // every mode is a bit field: the shuffle is a bit permutation
    uint64_t out = 0;
#pragma unroll 1
    for (int m = 0; m < p.n; ++m)
      out |= ((k >> p.oshift[m]) & ((1ull << p.width[m]) - 1ull)) << p.nshift[m];
    return out;
  }
  uint64_t out = 0;
#pragma unroll 1
  for (int m = p.n - 1; m > 0; --m) {
    uint64_t q = fdiv(p.div[m], k);
    out += (k - q * p.dim[m]) * p.nstride[m];
    k = q;
  }
  return out + k * p.nstride[0];
}

// LIV shuffle of N keys at once: the loop over modes is outermost so each mode's
// constants are read once per thread and applied to every item.
template <int N>
LCO_HD void reencode_n(const KeyPlan& p, uint64_t (&k)[N]) {
  if (p.pow2) {
    uint64_t out[N];
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = 0;
#pragma unroll 1
    for (int m = 0; m < p.n; ++m) {
      const int os = p.oshift[m], ns = p.nshift[m];
      const uint64_t mk = p.omask[m];
#pragma unroll
      for (int i = 0; i < N; ++i) out[i] |= ((k[i] >> os) & mk) << ns;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) k[i] = out[i];
    return;
  }
  uint64_t out[N];
#pragma unroll
  for (int i = 0; i < N; ++i) out[i] = 0;
#pragma unroll 1
  for (int m = p.n - 1; m > 0; --m) {
    const FastDiv f = p.div[m];
    const uint64_t dm = p.dim[m], st = p.nstride[m];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const uint64_t q = fdiv(f, k[i]);
      out[i] += (k[i] - q * dm) * st;
      k[i] = q;
    }
  }
  const uint64_t s0 = p.nstride[0];
#pragma unroll
  for (int i = 0; i < N; ++i) k[i] = out[i] + k[i] * s0;
}

LCO_HD uint32_t digit_of(const KeyPlan& p, uint64_t q, int pass) {
  return (uint32_t)(q >> p.dshift[pass]) & ((1u << p.dbits[pass]) - 1u);
}

enum Path { kPathCopy = 0, kPathOnesweep = 1, kPathLocal = 2, kPathMsd = 3, kPathTile = 4,
            kPathSeg = 5, kPathBlock = 7, kPathSingle = 8 };

// Host plan for one operation (permute or sort) of a handle.
struct OpPlan {
  int path;
  int sort_bits;
  int passes;
  int radix_bits;   // kernel instantiation: bins per pass = 2^radix_bits
  int tile;         // nonzeros per tile
  KeyPlan kp;
  uint64_t trailing, middle, segments, segdiv;
  // block-transpose schedule: old modes 0..k (k = last old position of a prefix / middle
  // mode) form the block id K div bfree; kb maps a block id to its new-order id.  The
  // block grid as (hi, B, mid, A): A = old mode k (innermost old), B = the innermost
  // block mode of the new order, hi / mid = products of the block modes before B and
  // between B and A (the tile decomposition of k_block_tiles)
  uint64_t nblocks, bfree;
  uint64_t bdA, bdB, bmid, bhi;
  KeyPlan kb;
};

// One stage of a hierarchical plan: the flat plan of a relative permutation.
constexpr int kMaxStages = 8;
struct StagePlan {
  int order;
  uint64_t dims[LCO_MAX_ORDER];  // stage input order
  int32_t perm[LCO_MAX_ORDER];   // relative permutation
  OpPlan op;
};

// Schedule overrides for tests and A/B measurements.  lco_create reads them ONCE from the
// environment into the handle (read_tuning, api.cu); no call ever reads the environment.
// All zero = the default schedule (DESIGN.md §2 lists the variables).
struct Tuning {
  int no_tile;      // LCO_NO_TILE: no segment-local tile schedule
  int no_block;     // LCO_NO_BLOCK: no block transpose
  int no_seg;       // LCO_NO_SEG: no segmented single pass
  int msd_force;    // LCO_MSD: MSD schedule whenever it applies
  int msd_b1;       // LCO_MSD_B1 (0: default), clamped to 4..11
  int msd_b2;       // LCO_MSD_B2 (0: default), clamped to 4..11
  int msd_cta;      // LCO_MSD_CTA: -1 default, 0 warp leaves, 1 CTA leaves
  int leafs_force;  // LCO_LEAFS: fully staged CTA leaves whenever they fit
  int no_leafs;     // LCO_NO_LEAFS
  int no_leafr;     // LCO_NO_LEAFR
  int no_sampled;   // LCO_NO_SAMPLED: level 1 of the MSD schedule counted exactly
  int no_cursor2;   // LCO_NO_CURSOR2: unordered level 2 with per-tile offsets (A/B)
  int sampled_test; // LCO_SAMPLED_TEST: sampled capacities halved (forces the exact fallback)
  int no_match;     // LCO_NO_MATCH: LSD passes never rank with match.any
  int lsd_maxbits;  // LCO_LSD_MAXBITS (0: default), clamped to 1..11
  int stable_msd;   // LCO_STABLE_MSD: MSD passes of lco_permute ranked stably
  int no_single;    // LCO_NO_SINGLE: no single-tile pass for tiny inputs
  int no_l3;        // LCO_NO_L3: no MSD level-3 re-split (oversize leaves stream)
  int l3_flat;      // LCO_L3_FLAT: level-3 count / scatter one CTA per tile (debug)
  int l3_bits;      // LCO_L3_BITS: level-3 digit bits (0: default 8; -1: 0 bits)
  int single_cta;   // LCO_SINGLE_CTA: the single-tile pass on one CTA, not a cluster
  int no_prefix_msd;  // LCO_NO_PREFIX_MSD: identity-prefix plans never switch to the full-key MSD
};

}  // namespace lco

struct lco_plan_s {
  int order;
  uint64_t dims[LCO_MAX_ORDER];
  int32_t perm[LCO_MAX_ORDER];
  uint64_t total;      // prod dims
  int key_bits;        // ceil(log2(total))
  int32_t rearr[LCO_MAX_ORDER];
  int norm_n;
  uint64_t norm_dims[LCO_MAX_ORDER];
  int32_t norm_perm[LCO_MAX_ORDER];
  int prefix_len, suffix_start;
  uint64_t max_nnz;
  uint32_t flags;
  lco::Tuning tune;        // read once at lco_create
  lco::OpPlan op_permute;  // nnz-independent parts; path refined per call
  lco::OpPlan op_sort;
  lco::KeyPlan kp_full;    // re-encode only (partition, histogram)
  int nstages;             // hierarchical plan: stages (>= 2 when it differs from flat)
  lco::StagePlan stages[lco::kMaxStages];
  // profiling
  int prof_calls_max;
  int prof_calls;
  int prof_stages;
  void** prof_events;      // cudaEvent_t[prof_calls_max * (kProfStages + 1)]
  int prof_nstages[64];
  char prof_names[1024];
};

namespace lco {
constexpr int kProfStages = 48;
// Host planning (plan.cpp)
lco_status build_plan(lco_plan_s* h, int order, const uint64_t* dims, const int32_t* perm);
void choose_passes(OpPlan* op, int sort_bits, int max_digit);  // max_digit 0: default
void build_digit_moves(KeyPlan* kp);  // after dshift / dbits are final (pow2 plans)
int ceil_log2(uint64_t x);  // smallest b with 2^b >= x
void set_error(const char* fmt, ...);
}  // namespace lco
