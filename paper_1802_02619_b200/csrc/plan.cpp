// plan.cpp — host planning for the LCO permutation (no CUDA calls).
//
// Implements RP step 1 (classify indices, §4.1) and the key shaving
// of step 2 ("(LIV mod 30) div 3") as a normalized plan:
//   1. drop size-1 modes (their coordinate is always 0);
//   2. fuse modes that are adjacent in both the old and the new order (they move as
//      one mixed-radix digit);
//   3. prefix a = identity run (those modes keep their significance: segments of
//      constant prefix are the paper's "regions where k is constant", and they occupy
//      the same positions before and after), suffix b = longest strictly increasing
//      tail of the perm (already in new relative order inside every run of equal
//      prefix+middle, hence "ignored", "the final index j can be
//      ignored"); the radix passes sort on q = K' div T, T = prod of suffix dims.
// DESIGN.md §"Plan" proves that a stable sort of the (sorted) input by q yields the
// new order; tests/test_plan.py checks it against the oracle on every permutation of
// orders 1-6.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "lco_internal.h"

namespace lco {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

const char* last_error() { return g_last_error.c_str(); }

int ceil_log2(uint64_t x) {
  int b = 0;
  while (b < 64 && (1ull << b) < x) ++b;
  return b;
}

FastDiv make_fastdiv(uint64_t d) {
  FastDiv f{d, 0, 0, 0};
  if (d <= 1) return f;  // kind 0: identity (d == 1)
  if ((d & (d - 1)) == 0) {
    f.kind = 1;
    f.s = (uint32_t)__builtin_ctzll(d);
    return f;
  }
  int l = ceil_log2(d);  // 2^(l-1) < d < 2^l, l <= 63 because d <= 2^63-1
  unsigned __int128 num = ((unsigned __int128)((1ull << l) - d)) << 64;
  f.m = (uint64_t)(num / d) + 1;
  f.s = (uint32_t)(l - 1);
  f.kind = 2;
  return f;
}

// Digit schedule: P = ceil(bits / 11) passes of <= 11 bits, as even as possible
// (results do not depend on the digit size).
void choose_passes(OpPlan* op, int bits, int max_digit) {
  op->sort_bits = bits;
  if (bits <= 0) {
    op->passes = 0;
    op->radix_bits = 0;
    return;
  }
  // digits of <= 10 bits unless one 11-bit pass does it all: an 11-bit digit writes runs
  // of ~2 nonzeros per bucket per 4,096-nonzero tile and ran at half the speed of a 7-bit
  // one (C3a: 11 + 10 bits 0.66 ms, 7 + 7 + 7 bits 0.60 ms; 10-bit digits as fast as 8)
  int kMaxDigit = max_digit > 0 ? (max_digit > 11 ? 11 : max_digit) : (bits <= 11 ? 11 : 10);
  // at most kMaxPasses passes (64-bit keys need digits of >= 8 bits)
  if ((bits + kMaxDigit - 1) / kMaxDigit > kMaxPasses) kMaxDigit = (bits + kMaxPasses - 1) / kMaxPasses;
  int P = (bits + kMaxDigit - 1) / kMaxDigit;
  int b = (bits + P - 1) / P;
  op->passes = P;
  op->radix_bits = b <= 8 ? 8 : (b <= 10 ? 10 : 11);
  op->kp.passes = P;
  for (int j = 0; j < P; ++j) {
    op->kp.dshift[j] = j * b;
    op->kp.dbits[j] = (j < P - 1) ? b : bits - (P - 1) * b;
  }
  op->tile = 4096;
  build_digit_moves(&op->kp);
}

// Power-of-two plans: every mode is a bit field of the key, so the LIV shuffle
// is a set of bit-field moves.  Split each mode's field at bit 32 of the
// NEW key so that every move lands inside one 32-bit output word.
static void build_moves(KeyPlan* kp) {
  kp->nmv = 0;
  for (int m = 0; m < kp->n; ++m) {
    int o = kp->oshift[m], nn = kp->nshift[m], w = kp->width[m];
    while (w > 0) {
      const int room = nn < 32 ? 32 - nn : 64 - nn;  // bits left in the output word
      const int take = w < room ? w : room;
      BitMove& mv = kp->mv[kp->nmv++];
      mv.a = (uint8_t)o;
      mv.hi = (uint8_t)(nn >= 32);
      mv.b = (uint8_t)(nn >= 32 ? nn - 32 : nn);
      mv.mask = take >= 32 ? 0xffffffffu : ((1u << take) - 1u);
      mv.pad = 0;
      o += take;
      nn += take;
      w -= take;
    }
  }
}

// Digit j of q = K' div T covers bits [log2 T + dshift[j], + dbits[j]) of K'; collect the
// pieces of the mode fields that land there, as moves from the OLD key.
void build_digit_moves(KeyPlan* kp) {
  for (int j = 0; j < kMaxPasses; ++j) kp->ndmv[j] = -1;
  if (!kp->pow2) return;
  const int tbits = kp->divT.kind == 1 ? (int)kp->divT.s : 0;
  if (kp->divT.kind == 2) return;
  for (int j = 0; j < kp->passes && j < kMaxPasses; ++j) {
    const int D = tbits + kp->dshift[j], E = D + kp->dbits[j];
    int cnt = 0;
    bool ok = true;
    for (int m = 0; m < kp->n && ok; ++m) {
      const int n0 = kp->nshift[m], n1 = n0 + kp->width[m];
      const int x0 = n0 > D ? n0 : D, x1 = n1 < E ? n1 : E;
      if (x0 >= x1) continue;
      if (cnt >= kMaxDigitMoves) {
        ok = false;
        break;
      }
      BitMove& mv = kp->dmv[j][cnt++];
      const int w = x1 - x0;
      mv.a = (uint8_t)(kp->oshift[m] + (x0 - n0));
      mv.hi = 0;
      mv.b = (uint8_t)(x0 - D);
      mv.mask = w >= 32 ? 0xffffffffu : ((1u << w) - 1u);
      mv.pad = 0;
    }
    kp->ndmv[j] = ok ? cnt : -1;
  }
}

struct FlatInfo {
  int n;
  uint64_t nd[LCO_MAX_ORDER];
  int32_t np[LCO_MAX_ORDER];
  int a, b;
};

static KeyPlan make_keyplan(int n, const uint64_t* nd, const int32_t* np, uint64_t T) {
  KeyPlan kp;
  memset(&kp, 0, sizeof kp);
  kp.n = n;
  uint64_t stride_at[kMaxModes];
  uint64_t acc = 1;
  for (int t = n - 1; t >= 0; --t) {
    stride_at[t] = acc;
    acc *= nd[np[t]];
  }
  for (int t = 0; t < n; ++t) kp.nstride[np[t]] = stride_at[t];
  for (int m = 0; m < n; ++m) {
    kp.dim[m] = nd[m];
    kp.div[m] = make_fastdiv(nd[m]);
  }
  if (n == 0) kp.nstride[0] = 1;
  kp.divT = make_fastdiv(T);
  for (int j = 0; j < kMaxPasses; ++j) kp.ndmv[j] = -1;
  kp.pow2 = n >= 1;
  for (int m = 0; m < n; ++m)
    if (nd[m] & (nd[m] - 1)) kp.pow2 = 0;
  if (kp.pow2) {
    int acc_old = 0;
    for (int m = n - 1; m >= 0; --m) {
      kp.width[m] = (uint8_t)__builtin_ctzll(nd[m]);
      kp.omask[m] = nd[m] - 1;
      kp.oshift[m] = (uint8_t)acc_old;
      acc_old += kp.width[m];
    }
    for (int m = 0; m < n; ++m) kp.nshift[m] = (uint8_t)__builtin_ctzll(kp.nstride[m]);
    build_moves(&kp);
  }
  return kp;
}

// Normalization (RP preprocessing): drop size-1 modes (their
// coordinate is always 0), then fuse runs of modes that are consecutive in both orders
// (they move as one mixed-radix digit); a = identity-prefix length, b = start of the
// longest strictly increasing suffix.
static void normalize(int order, const uint64_t* dims, const int32_t* perm, FlatInfo* fi) {
  int keep[LCO_MAX_ORDER];
  uint64_t d1[LCO_MAX_ORDER];
  int n1 = 0;
  for (int m = 0; m < order; ++m) {
    keep[m] = dims[m] > 1 ? n1 : -1;
    if (dims[m] > 1) d1[n1++] = dims[m];
  }
  int p1[LCO_MAX_ORDER];
  int k = 0;
  for (int t = 0; t < order; ++t)
    if (keep[perm[t]] >= 0) p1[k++] = keep[perm[t]];
  int gfirst[LCO_MAX_ORDER], glen[LCO_MAX_ORDER], ng = 0;
  for (int t = 0; t < n1; ++t) {
    if (t > 0 && p1[t] == p1[t - 1] + 1) {
      glen[ng - 1]++;
    } else {
      gfirst[ng] = p1[t];
      glen[ng] = 1;
      ng++;
    }
  }
  fi->n = ng;
  for (int g = 0; g < ng; ++g) {
    int rank = 0;
    for (int g2 = 0; g2 < ng; ++g2)
      if (gfirst[g2] < gfirst[g]) rank++;
    uint64_t d = 1;
    for (int i = 0; i < glen[g]; ++i) d *= d1[gfirst[g] + i];
    fi->nd[rank] = d;
    fi->np[g] = rank;
  }
  int a = 0;
  while (a < ng && fi->np[a] == a) ++a;
  int b = ng > 0 ? ng - 1 : 0;
  while (b > 0 && fi->np[b - 1] < fi->np[b]) --b;
  fi->a = a;
  fi->b = b;
}

// The flat plan: sort on q = K' div T (prefix + middle digits), T = prod of suffix dims.
static void flat_permute(const FlatInfo& fi, OpPlan* op, int max_digit) {
  const int n = fi.n, a = fi.a, b = fi.b;
  const uint64_t* nd = fi.nd;
  const int32_t* np = fi.np;
  uint64_t T = 1, S = 1, G = 1, D = 1;
  for (int t = b; t < n; ++t) T *= nd[np[t]];
  for (int t = a; t < b; ++t) S *= nd[np[t]];
  for (int m = 0; m < a && m < n; ++m) G *= nd[m];
  for (int m = a; m < n; ++m) D *= nd[m];
  memset(op, 0, sizeof *op);
  op->kp = make_keyplan(n, nd, np, n >= 2 ? T : 1);
  op->trailing = T;
  op->middle = S;
  op->segments = G;
  op->segdiv = D;
  if (n <= 1) {
    op->path = kPathCopy;
    choose_passes(op, 0, max_digit);
  } else {
    op->path = kPathOnesweep;
    choose_passes(op, ceil_log2(G * S), max_digit);
  }
  // block-transpose schedule (block.cu): blocks = old modes 0..k
  op->nblocks = 0;
  if (n >= 2 && b > 0) {
    int k = 0;
    for (int t = 0; t < b; ++t) k = np[t] > k ? np[t] : k;
    uint64_t nb = 1, F = 1;
    for (int m = 0; m <= k; ++m) nb *= nd[m];
    for (int m = k + 1; m < n; ++m) F *= nd[m];
    int32_t bp[LCO_MAX_ORDER];
    int j = 0;
    for (int t = 0; t < n; ++t)
      if (np[t] <= k) bp[j++] = np[t];
    op->nblocks = nb;
    op->bfree = F;
    op->kb = make_keyplan(k + 1, nd, bp, 1);
    const int B = bp[k];  // != k: the old-innermost block mode never stays innermost
    op->bdA = nd[k];
    op->bdB = nd[B];
    op->bmid = 1;
    op->bhi = 1;
    for (int m = B + 1; m < k; ++m) op->bmid *= nd[m];
    for (int m = 0; m < B; ++m) op->bhi *= nd[m];
  }
}

// Hierarchical plan ("the rearrangement procedure is recursively applied
// to each of these sub-regions"): walking the new order from the most
// significant mode, a resting mode refines the current regions (it is the old-most-
// significant of the remaining modes, already in place), and each maximal run of
// rearrangement modes is one stable sort inside the current regions.  Stage j permutes
// the order O_{j-1} (the modes fixed so far, then the rest in old order) into O_j; its
// own flat plan has the fixed modes as identity prefix and only that run as middle, so
// interior resting modes are never sorted.  One stage = the flat plan.
static void build_stages(lco_plan_s* h, const FlatInfo& fi) {
  const int n = fi.n;
  const int32_t* np = fi.np;
  h->nstages = 0;
  int O[LCO_MAX_ORDER];
  for (int m = 0; m < n; ++m) O[m] = m;
  auto resting = [&](int t) {
    for (int u = t + 1; u < n; ++u)
      if (np[u] < np[t]) return false;
    return true;
  };
  int t = 0;
  while (t < n && h->nstages < kMaxStages) {
    if (resting(t)) {
      ++t;
      continue;
    }
    int u = t;
    while (u < n && !resting(u)) ++u;
    int On[LCO_MAX_ORDER], k = 0;
    bool used[LCO_MAX_ORDER] = {false};
    for (int i = 0; i < u; ++i) {
      On[k++] = np[i];
      used[np[i]] = true;
    }
    for (int m = 0; m < n; ++m)
      if (!used[m]) On[k++] = m;
    StagePlan& S = h->stages[h->nstages++];
    S.order = n;
    for (int i = 0; i < n; ++i) S.dims[i] = fi.nd[O[i]];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        if (O[j] == On[i]) S.perm[i] = j;
    FlatInfo sfi;
    normalize(n, S.dims, S.perm, &sfi);
    flat_permute(sfi, &S.op, h->tune.lsd_maxbits);
    for (int i = 0; i < n; ++i) O[i] = On[i];
    t = u;
  }
}

lco_status build_plan(lco_plan_s* h, int order, const uint64_t* dims, const int32_t* perm) {
  h->order = order;
  uint64_t total = 1;
  for (int m = 0; m < order; ++m) {
    h->dims[m] = dims[m];
    h->perm[m] = perm ? perm[m] : m;
    if (dims[m] == 0) {
      set_error("dims[%d] == 0", m);
      return LCO_ERR_DIM;
    }
  }
  int seen[LCO_MAX_ORDER] = {0};
  for (int t = 0; t < order; ++t) {
    int p = h->perm[t];
    if (p < 0 || p >= order || seen[p]) {
      set_error("perm is not a bijection on 0..%d (perm[%d] = %d)", order - 1, t, p);
      return LCO_ERR_PERM;
    }
    seen[p] = 1;
  }
  for (int m = 0; m < order; ++m) {
    if (total > 0x7fffffffffffffffull / dims[m]) {
      set_error("product of dims exceeds 2^63-1 (PAPER.md:173)");
      return LCO_ERR_OVERFLOW;
    }
    total *= dims[m];
  }
  h->total = total;
  h->key_bits = ceil_log2(total);

  // RP step 1: perm[t] is a rearrangement index iff it crosses a mode
  // that was more significant before, i.e. iff it is not the minimum of perm[t..].
  for (int t = 0; t < order; ++t) {
    int mn = h->perm[t];
    for (int u = t + 1; u < order; ++u)
      if (h->perm[u] < mn) mn = h->perm[u];
    h->rearr[t] = h->perm[t] != mn;
  }

  FlatInfo fi;
  normalize(order, dims, h->perm, &fi);
  const int n = fi.n;
  const uint64_t* nd = fi.nd;
  h->norm_n = n;
  for (int m = 0; m < n; ++m) {
    h->norm_dims[m] = fi.nd[m];
    h->norm_perm[m] = fi.np[m];
  }
  h->prefix_len = fi.a;
  h->suffix_start = fi.b;
  flat_permute(fi, &h->op_permute, h->tune.lsd_maxbits);
  build_stages(h, fi);
  // sort: q = K' (all key digits)
  OpPlan& os = h->op_sort;
  memset(&os, 0, sizeof os);
  os.kp = make_keyplan(n, nd, fi.np, 1);
  os.trailing = 1;
  os.middle = total;
  os.segments = 1;
  os.segdiv = total;
  if (total <= 1) {
    os.path = kPathCopy;
    choose_passes(&os, 0, h->tune.lsd_maxbits);
  } else {
    os.path = kPathOnesweep;
    choose_passes(&os, h->key_bits, h->tune.lsd_maxbits);
  }
  h->kp_full = make_keyplan(n, nd, fi.np, 1);
  return LCO_OK;
}

}  // namespace lco
