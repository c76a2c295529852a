// api.cu — the C ABI declared in include/lco.h: argument checking, workspace layout,
// launch sequencing, error reporting and the measurement hook.  Every device step of
// the path runs in kernels.cu; nothing here computes on the data.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "launch.h"
#include "lco_internal.h"

namespace lco {
const char* last_error();
}

using namespace lco;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct WsLayout {
  size_t ctrl, kA, vA, pA, kB, vB, pB, flag, total;
};

// Per-call schedule.  The host plan fixes the sort key q = K' div T and its width B; the
// call picks how to sort it for this nnz (results are identical, only the cost differs):
//   copy     B == 0 (identity after normalization);
//   leaf     nnz fits one on-chip leaf: one kernel, one read + one write;
//   lsd      P = ceil(B / 11) stable LSD passes (the north_star's LSD over the disturbed
//            digits), each a tile-granular reduce-then-scan pass;
//   msd      1-2 stable MSD passes of 8 (+ up to 11) bits, then on-chip leaf sorts of
//            the remaining bits (the paper's RP recursion into regions).
// Model: HBM bytes per nonzero (count read 8 + pass r/w ~40, leaf r/w 40).
struct CallPlan {
  int path;     // kPathCopy, kPathOnesweep (LSD), kPathLocal (leaf only), kPathMsd
  int passes;   // global passes
  int rb;       // LSD radix instantiation
  MsdPlan msd;
  KeyPlan kp;
  double cost;  // modelled bytes per nonzero
  uint64_t segdiv, segments;  // tile path: identity-prefix segments
  uint64_t nblocks, bfree;    // block path
  BlockGrid bg;
  KeyPlan kb;
};

// Environment overrides of the schedule (tests and A/B measurements only), read once by
// lco_create; clamped so that no value can break a kernel's limits.
Tuning read_tuning() {
  Tuning t;
  memset(&t, 0, sizeof t);
  auto flag = [](const char* n) { return getenv(n) != nullptr ? 1 : 0; };
  auto num = [](const char* n, int lo, int hi, int dflt) {
    const char* v = getenv(n);
    if (!v) return dflt;
    int x = atoi(v);
    return x < lo ? lo : (x > hi ? hi : x);
  };
  t.no_tile = flag("LCO_NO_TILE");
  t.no_block = flag("LCO_NO_BLOCK");
  t.no_seg = flag("LCO_NO_SEG");
  t.msd_force = flag("LCO_MSD");
  t.msd_b1 = num("LCO_MSD_B1", 4, 11, 0);
  t.msd_b2 = num("LCO_MSD_B2", 4, 11, 0);
  t.msd_cta = num("LCO_MSD_CTA", 0, 1, -1);
  t.leafs_force = flag("LCO_LEAFS");
  t.no_leafs = flag("LCO_NO_LEAFS");
  t.no_leafr = flag("LCO_NO_LEAFR");
  t.no_sampled = flag("LCO_NO_SAMPLED");
  t.no_cursor2 = flag("LCO_NO_CURSOR2");
  t.sampled_test = flag("LCO_SAMPLED_TEST");
  t.no_match = flag("LCO_NO_MATCH");
  t.lsd_maxbits = num("LCO_LSD_MAXBITS", 1, 11, 0);
  t.stable_msd = flag("LCO_STABLE_MSD");
  t.no_single = flag("LCO_NO_SINGLE");
  t.no_l3 = flag("LCO_NO_L3");
  t.l3_flat = flag("LCO_L3_FLAT");
  t.l3_bits = num("LCO_L3_BITS", -1, 8, 0);
  t.single_cta = flag("LCO_SINGLE_CTA");
  t.no_prefix_msd = flag("LCO_NO_PREFIX_MSD");
  return t;
}

CallPlan choose_plan(const OpPlan& op, uint64_t nnz, const Tuning& tu) {
  CallPlan c;
  memset(&c, 0, sizeof c);
  c.kp = op.kp;
  const int B = op.sort_bits;
  if (op.path == kPathCopy || B == 0) {
    c.path = kPathCopy;
    c.cost = 36;
    return c;
  }
  // one tile, one digit: a single stable pass of one CTA (no count / scan kernels)
  if (nnz <= 8192 && B <= 10 && !tu.no_single) {
    c.path = kPathSingle;
    c.rb = B <= 8 ? 8 : 10;
    c.cost = 36;
    c.passes = 1;
    c.kp.passes = 1;  // the one digit: all B bits of q
    c.kp.dshift[0] = 0;
    c.kp.dbits[0] = B;
    build_digit_moves(&c.kp);
    return c;
  }
  if (nnz <= leaf_cap()) {
    c.path = kPathLocal;
    c.msd.levels = 0;
    c.msd.rb = B;
    c.cost = 36;
    return c;
  }
  // Identity prefix with small segments: every segment stays in place, so one on-chip
  // sort per tile of whole segments finishes the permutation (one read, one write).
  if (op.segments > 1 && nnz / op.segments <= 3072 && !tu.no_tile) {
    c.path = kPathTile;
    c.segdiv = op.segdiv;
    c.segments = op.segments;
    c.msd.rb = B;
    // one read + one write; when many nonzeros share a q value (more per segment than
    // middle values) the tile sort needs stable radix passes on chip, measured at about
    // twice the cost (C3b stage 2, Table 2 2%-fill stage 2)
    c.cost = nnz / op.segments > op.middle ? 80 : 40;
    return c;
  }
  c.path = kPathOnesweep;
  c.passes = op.passes;
  c.rb = op.radix_bits;
  c.cost = 4 + 48.0 * op.passes;
  // All rearranged modes in a small old-order prefix: a transpose of runs, no sorting
  // (block.cu): one read of the keys for the run bounds, O(blocks) tables, one tiled
  // copy that reads and writes long runs.
  if (op.nblocks && op.nblocks * 4 <= nnz && op.nblocks < (1ull << 31) && !tu.no_block) {
    const double bcost = 8 + 36 + 24.0 * (double)op.nblocks / (double)nnz;
    if (bcost < c.cost) {
      c.path = kPathBlock;
      c.nblocks = op.nblocks;
      c.bfree = op.bfree;
      c.bg = BlockGrid{op.bdA, op.bdB, op.bmid, op.bhi};
      c.kb = op.kb;
      c.passes = 0;
      c.cost = bcost;
      return c;
    }
  }
  // Identity prefix with large segments and a power-of-two middle of <= 11 bits: one
  // stable pass of the middle digit inside every segment (segment starts from a count of
  // the prefix digit), straight from the input to the outputs.
  {
    const int gb = ceil_log2(op.segments), mb = ceil_log2(op.middle);
    const bool pow2_mid = (op.middle & (op.middle - 1)) == 0;
    if (op.segments > 1 && gb <= 10 && mb >= 1 && mb <= 11 && pow2_mid && op.passes >= 2 &&
        !tu.no_seg) {
      c.path = kPathSeg;
      c.passes = 1;
      c.msd.b1 = gb;
      c.msd.b2 = mb;
      c.cost = 52;
      c.kp.passes = 2;
      c.kp.dshift[0] = mb;
      c.kp.dbits[0] = gb;
      c.kp.dshift[1] = 0;
      c.kp.dbits[1] = mb;
      build_digit_moves(&c.kp);
      return c;
    }
  }
  if (B <= 11) return c;
  // MSD levels of 8-bit digits (a 4,096-nonzero tile then writes runs of ~16 nonzeros
  // per digit, which the HBM write path sustains; 10-11-bit digits write runs of 2-4 and
  // ran at half the bandwidth, benchmarks/micro/scatter_bw.cu), then one on-chip sort per
  // leaf: by a warp when the expected leaf is <= leaf_target(), else by a CTA (<= 8K).
  // Two-level plans size the second digit for the fully staged CTA leaves (k_leafs,
  // ~1.9K nonzeros, three CTAs per SM): measured on C5 8+10 bits + k_leafs 22.5 ms vs
  // 8+8 + k_leafr (7.6K-nonzero leaves, L2 gathers) 23.3 ms.
  MsdPlan m;
  memset(&m, 0, sizeof m);
  const uint64_t wt = leaf_target();
  const uint64_t ct = cta_leaf_cap() * 15 / 16;  // expected size, ~4 sigma below the cap
  const uint64_t st = staged_leaf_target();
  double mcost;
  if ((nnz >> 8) <= ct) {
    m.levels = 1;
    m.b1 = B < 8 ? B : 8;
    m.b2 = 0;
    m.cta = (nnz >> m.b1) > wt;
    m.staged = m.cta && (nnz >> m.b1) <= st;
    mcost = 8 + 36 + 40;
  } else {
    m.levels = 2;
    m.b1 = 8;
    m.b2 = 8;
    while (m.b2 < 11 && (nnz >> (m.b1 + m.b2)) > st) ++m.b2;
    if (m.b1 + m.b2 > B) m.b2 = B - m.b1;  // B >= 12 here, so b2 >= 4
    m.cta = (nnz >> (m.b1 + m.b2)) > wt;
    m.staged = m.cta && (nnz >> (m.b1 + m.b2)) <= st;
    mcost = 8 + 36 + 8 + 40 + 40;
  }
  if (tu.leafs_force) m.staged = 1;
  // sampled level 1 for large two-level plans with an 8-bit first digit (set below, once
  // b1 is final): C5 saves the 0.66 ms count pass
  // schedule overrides for tests and A/B measurements (the defaults above otherwise),
  // kept inside the key: b1 + b2 < B
  if (tu.msd_b1) m.b1 = tu.msd_b1 < B - 1 ? tu.msd_b1 : B - 1;
  if (tu.msd_b2 && m.levels == 2) m.b2 = tu.msd_b2 < B - m.b1 ? tu.msd_b2 : B - m.b1 - 1;
  if (m.levels == 2 && m.b2 < 1) m.levels = 1, m.b2 = 0;
  if (tu.msd_cta >= 0) m.cta = tu.msd_cta;
  m.rb = B - m.b1 - m.b2;
  m.sampled = m.levels == 2 && m.b1 == 8 && nnz >= (1ull << 24) && !tu.no_sampled &&
              sampled_capacity(nnz) < (1ull << 32);
  // MSD leaves are sized for uniformly spread keys; structured keys (stencil operators,
  // identity-prefix segments) make them uneven, so MSD is taken only without a prefix
  // and with a clear modelled win.
  // (one level: below 0.9 of the LSD model, C2a 0.105 vs 0.127 ms; two levels: below
  // 0.75 -- structured tensors (Table 2's Laplacian) fill two-level buckets unevenly)
  if ((op.segments == 1 && mcost < (m.levels == 1 ? 0.9 : 0.75) * c.cost) || tu.msd_force) {
    c.path = kPathMsd;
    c.msd = m;
    c.cost = mcost;
    c.passes = m.levels;
    c.kp.passes = m.levels;
    c.kp.dshift[0] = B - m.b1;
    c.kp.dbits[0] = m.b1;
    if (m.levels == 2) {
      c.kp.dshift[1] = B - m.b1 - m.b2;
      c.kp.dbits[1] = m.b2;
    }
    build_digit_moves(&c.kp);
  }
  return c;
}

// Ping-pong buffers carry (K', V, position); V only when values are moved and the
// position only when a permutation vector is requested (sizes assume both).
WsLayout layout_for(const CallPlan& c, uint64_t nnz) {
  WsLayout w;
  memset(&w, 0, sizeof w);
  size_t off = 0;
  const bool lsd = c.path == kPathOnesweep, msd = c.path == kPathMsd, tile = c.path == kPathTile;
  const bool seg = c.path == kPathSeg, blk = c.path == kPathBlock;
  if ((lsd || msd || tile || seg || blk) && nnz > 0) {
    w.ctrl = off;
    off += align_up(lsd ? pass_ctrl_bytes(c.rb, nnz)
                        : ((msd || seg) ? msd_ctrl_bytes(c.msd.b1, c.msd.b2, nnz)
                                        : (blk ? block_ctrl_bytes(c.nblocks)
                                               : tile_ctrl_bytes(nnz, c.segments))));
    // the tile path needs both buffers only as scratch of the rare streaming fallback
    if (msd || tile || c.passes >= 2) {
      const uint64_t na = msd && c.msd.sampled ? sampled_capacity(nnz) : nnz;
      w.kA = off;
      off += align_up(na * 8);
      w.vA = off;
      off += align_up(na * 8);
      w.pA = off;
      off += align_up(na * 4);
    }
    if (msd || tile || c.passes >= 3) {
      w.kB = off;
      off += align_up(nnz * 8);
      w.vB = off;
      off += align_up(nnz * 8);
      w.pB = off;
      off += align_up(nnz * 4);
    }
  }
  w.flag = off;
  off += kAlign;
  w.total = off;
  return w;
}

int partition_rb(int world) { return world <= 256 ? 8 : (world <= 1024 ? 10 : 11); }

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  if (!a || !b || !na || !nb) return false;
  const char* x = static_cast<const char*>(a);
  const char* y = static_cast<const char*>(b);
  return x < y + nb && y < x + na;
}

lco_status cuda_fail(cudaError_t e, const char* where) {
  set_error("%s: %s", where, cudaGetErrorString(e));
  return LCO_ERR_CUDA;
}

// ---- measurement hook: one CUDA event before each launch, one after the last ----
struct ProfCtx {
  lco_plan_s* h;
  cudaStream_t s;
  int call;
  int stage;
};

void prof_mark(void* ctx, const char* name) {
  ProfCtx* c = static_cast<ProfCtx*>(ctx);
  lco_plan_s* h = c->h;
  if (c->stage >= kProfStages) return;
  cudaEvent_t ev = static_cast<cudaEvent_t>(h->prof_events[c->call * (kProfStages + 1) + c->stage]);
  cudaEventRecord(ev, c->s);
  if (c->call == 0) {
    size_t len = strlen(h->prof_names);
    snprintf(h->prof_names + len, sizeof(h->prof_names) - len, "%s%s", len ? ";" : "", name);
  }
  c->stage++;
}

bool prof_begin(lco_plan_s* h, cudaStream_t s, ProfCtx* c, Launch* L) {
  if (!h->prof_events || h->prof_calls >= h->prof_calls_max) return false;
  c->h = h;
  c->s = s;
  c->call = h->prof_calls;
  c->stage = 0;
  if (c->call == 0) h->prof_names[0] = 0;
  L->mark = prof_mark;
  L->ctx = c;
  return true;
}

void prof_end(ProfCtx* c) {
  lco_plan_s* h = c->h;
  int st = c->stage < kProfStages ? c->stage : kProfStages;
  cudaEventRecord(static_cast<cudaEvent_t>(h->prof_events[c->call * (kProfStages + 1) + st]), c->s);
  h->prof_nstages[c->call < 64 ? c->call : 63] = st;
  h->prof_calls++;
}

lco_status check_handle(lco_handle h) {
  if (!h) {
    set_error("NULL handle");
    return LCO_ERR_NULL;
  }
  return LCO_OK;
}

// Run one flat plan on device buffers with the workspace `ws` (layout_for of its call
// plan); launches only, no checks.
cudaError_t execute(lco_plan_s* h, const OpPlan& op, bool unique, uint64_t nnz,
                    const uint64_t* keys_in, const double* vals_in, const uint32_t* idx_in,
                    uint64_t* keys_out, double* vals_out, uint32_t* perm_out, char* ws,
                    const Launch& L) {
  const CallPlan cp = choose_plan(op, nnz, h->tune);
  const WsLayout w = layout_for(cp, nnz);
  if (cp.path == kPathCopy)
    return run_copy(nnz, keys_in, vals_in, idx_in, keys_out, vals_out, perm_out, L);
  PassIO io;
  memset(&io, 0, sizeof io);
  io.nnz = nnz;
  io.keys_in = keys_in;
  io.vals_in = vals_in;
  io.idx_in = idx_in;
  io.keys_out = keys_out;
  io.vals_out = vals_out;
  io.perm_out = perm_out;
  io.tune = &h->tune;
  io.unique = unique && !h->tune.stable_msd;
  io.ctrl = reinterpret_cast<uint32_t*>(ws + w.ctrl);
  const bool mv = vals_out != nullptr, mp = perm_out != nullptr;
  const bool hasA = cp.path == kPathMsd || cp.path == kPathTile || cp.passes >= 2;
  const bool hasB = cp.path == kPathMsd || cp.path == kPathTile || cp.passes >= 3;
  io.kA = hasA ? reinterpret_cast<uint64_t*>(ws + w.kA) : nullptr;
  io.vA = hasA && mv ? reinterpret_cast<double*>(ws + w.vA) : nullptr;
  io.pA = hasA && mp ? reinterpret_cast<uint32_t*>(ws + w.pA) : nullptr;
  io.kB = hasB ? reinterpret_cast<uint64_t*>(ws + w.kB) : nullptr;
  io.vB = hasB && mv ? reinterpret_cast<double*>(ws + w.vB) : nullptr;
  io.pB = hasB && mp ? reinterpret_cast<uint32_t*>(ws + w.pB) : nullptr;
  if (cp.path == kPathSingle)
    return h->tune.single_cta ? run_single_tile(cp.rb, cp.kp, io, L)
                              : run_single_cluster(cp.rb, cp.kp, io, L);
  if (cp.path == kPathOnesweep) return run_passes(cp.rb, cp.kp, io, L);
  if (cp.path == kPathTile) return run_tiles(cp.kp, cp.segdiv, cp.segments, h->key_bits, io, L);
  if (cp.path == kPathSeg) return run_seg(cp.msd.b1, cp.msd.b2, cp.kp, io, L);
  if (cp.path == kPathBlock) return run_block(cp.kp, cp.kb, cp.nblocks, cp.bfree, cp.bg, io, L);
  return run_msd(cp.msd, cp.kp, io, L);
}

// Hierarchical execution of a permute call: taken when the handle was created with
// LCO_FLAG_HIERARCHICAL and the plan has >= 2 stages.  (Measured on B200: the stages win
// on the paper's addition permutation {1,0,3,2} and Table 2's median {2,1,3,0} of the
// combinatorial Laplacian, by 14-18%, and lose where a stage's tile sort meets many
// nonzeros per q value, which the host cannot see; hence opt-in.)
struct Hier {
  bool use;
  double cost, flat_cost;
  size_t buf_off[2], inner_off, total;
};

Hier hier_for(const lco_plan_s* h, bool sort, uint64_t nnz) {
  Hier r;
  memset(&r, 0, sizeof r);
  r.flat_cost = choose_plan(sort ? h->op_sort : h->op_permute, nnz, h->tune).cost;
  if (sort || h->nstages < 2 || nnz == 0) return r;
  size_t inner = 0;
  for (int j = 0; j < h->nstages; ++j) {
    const CallPlan cp = choose_plan(h->stages[j].op, nnz, h->tune);
    r.cost += cp.cost;
    const size_t t = layout_for(cp, nnz).total;
    inner = t > inner ? t : inner;
  }
  const size_t set = 2 * align_up(nnz * 8) + align_up(nnz * 4);
  r.buf_off[0] = 0;
  r.buf_off[1] = h->nstages >= 3 ? set : 0;
  r.inner_off = (h->nstages >= 3 ? 2 : 1) * set;
  r.total = r.inner_off + inner;
  r.use = (h->flags & LCO_FLAG_HIERARCHICAL) != 0;
  return r;
}

lco_status run_op(lco_handle h, const OpPlan& op, bool sort, uint64_t nnz, const uint64_t* keys_in,
                  const double* vals_in, const uint32_t* idx_in, uint64_t* keys_out,
                  double* vals_out, uint32_t* perm_out, void* workspace, size_t ws_bytes,
                  void* stream) {
  lco_status st = check_handle(h);
  if (st) return st;
  if (nnz > h->max_nnz || nnz >= (1ull << 32)) {
    set_error("nnz %llu exceeds max_nnz %llu (or 2^32-1)", (unsigned long long)nnz,
              (unsigned long long)h->max_nnz);
    return LCO_ERR_CAPACITY;
  }
  if (nnz == 0) return LCO_OK;
  if (!keys_in || !keys_out) {
    set_error("keys_in and keys_out are required");
    return LCO_ERR_NULL;
  }
  if ((vals_in == nullptr) != (vals_out == nullptr)) {
    set_error("vals_in and vals_out must both be given or both be NULL");
    return LCO_ERR_ARG;
  }
  const size_t n8 = nnz * 8, n4 = nnz * 4;
  const void* ins[3] = {keys_in, vals_in, idx_in};
  const size_t insz[3] = {n8, n8, n4};
  const void* outs[3] = {keys_out, vals_out, perm_out};
  const size_t outsz[3] = {n8, n8, n4};
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j)
      if (overlaps(outs[i], outsz[i], ins[j], insz[j])) {
        set_error("output %d overlaps input %d", i, j);
        return LCO_ERR_ALIAS;
      }
    for (int j = i + 1; j < 3; ++j)
      if (overlaps(outs[i], outsz[i], outs[j], outsz[j])) {
        set_error("outputs %d and %d overlap", i, j);
        return LCO_ERR_ALIAS;
      }
  }
  const Hier hp = hier_for(h, sort, nnz);
  const size_t need = hp.use ? hp.total : layout_for(choose_plan(op, nnz, h->tune), nnz).total;
  if (!workspace || ws_bytes < need || (reinterpret_cast<uintptr_t>(workspace) % kAlign)) {
    set_error("workspace needs %zu bytes, 256-byte aligned (got %zu at %p)", need, ws_bytes,
              workspace);
    return LCO_ERR_WORKSPACE;
  }
  for (int i = 0; i < 3; ++i)
    if (overlaps(outs[i], outsz[i], workspace, need) ||
        overlaps(ins[i], insz[i], workspace, need)) {
      set_error("workspace overlaps an input or output");
      return LCO_ERR_ALIAS;
    }
  char* ws = static_cast<char*>(workspace);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (h->flags & LCO_FLAG_VALIDATE) {
    uint32_t* flag = reinterpret_cast<uint32_t*>(ws);
    cudaError_t e = run_validate(nnz, keys_in, h->total, sort ? 0 : 1, flag, s);
    if (e != cudaSuccess) return cuda_fail(e, "validate");
    uint32_t hf = 0;
    e = cudaMemcpyAsync(&hf, flag, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "validate");
    if (hf & 2u) {
      set_error("a key is >= prod(dims)");
      return LCO_ERR_KEY_RANGE;
    }
    if (hf & 1u) {
      set_error("keys_in is not strictly increasing");
      return LCO_ERR_UNSORTED;
    }
  }
  Launch L{s, nullptr, nullptr};
  ProfCtx pc;
  const bool prof = prof_begin(h, s, &pc, &L);
  cudaError_t e = cudaSuccess;
  if (!hp.use) {
    e = execute(h, op, !sort, nnz, keys_in, vals_in, idx_in, keys_out, vals_out, perm_out, ws, L);
  } else {
    // stage j reads stage j-1's (K', V, position) from one of two intermediate buffer
    // sets and the last stage writes the outputs; positions compose through idx_in.
    char* inner = ws + hp.inner_off;
    const bool mp = perm_out != nullptr;
    const uint64_t* k_in = keys_in;
    const double* v_in = vals_in;
    const uint32_t* i_in = idx_in;
    for (int j = 0; j < h->nstages && e == cudaSuccess; ++j) {
      const bool last = j == h->nstages - 1;
      char* buf = ws + hp.buf_off[j % 2];
      uint64_t* k_out = last ? keys_out : reinterpret_cast<uint64_t*>(buf);
      double* v_out = last ? vals_out
                           : (vals_in ? reinterpret_cast<double*>(buf + align_up(nnz * 8)) : nullptr);
      uint32_t* p_out = last ? perm_out
                             : (mp ? reinterpret_cast<uint32_t*>(buf + 2 * align_up(nnz * 8)) : nullptr);
      e = execute(h, h->stages[j].op, true, nnz, k_in, v_in, i_in, k_out, v_out, p_out, inner, L);
      k_in = k_out;
      v_in = v_out;
      i_in = p_out;
    }
  }
  if (prof) prof_end(&pc);
  if (e != cudaSuccess) return cuda_fail(e, sort ? "lco_sort" : "lco_permute");
  return LCO_OK;
}

}  // namespace

extern "C" {

lco_status lco_create(lco_handle* out, int order, const uint64_t* dims, const int32_t* perm,
                      uint64_t max_nnz, uint32_t flags) {
  if (!out || !dims) {
    set_error("out and dims are required");
    return LCO_ERR_NULL;
  }
  *out = nullptr;
  if (order < 1 || order > LCO_MAX_ORDER) {
    set_error("order %d outside 1..%d", order, LCO_MAX_ORDER);
    return LCO_ERR_ORDER;
  }
  if (max_nnz >= (1ull << 32)) {
    set_error("max_nnz must be < 2^32 (uint32 permutation vector)");
    return LCO_ERR_CAPACITY;
  }
  if (flags & ~(LCO_FLAG_VALIDATE | LCO_FLAG_HIERARCHICAL)) {
    set_error("unknown flags 0x%x", flags);
    return LCO_ERR_ARG;
  }
  lco_plan_s* h = new (std::nothrow) lco_plan_s;
  if (!h) {
    set_error("out of host memory");
    return LCO_ERR_ARG;
  }
  memset(h, 0, sizeof *h);
  h->tune = read_tuning();
  lco_status st = build_plan(h, order, dims, perm);
  if (st != LCO_OK) {
    delete h;
    return st;
  }
  h->max_nnz = max_nnz;
  h->flags = flags;
  *out = h;
  return LCO_OK;
}

lco_status lco_destroy(lco_handle h) {
  if (!h) return LCO_OK;
  if (h->prof_events) {
    for (int i = 0; i < h->prof_calls_max * (kProfStages + 1); ++i)
      if (h->prof_events[i]) cudaEventDestroy(static_cast<cudaEvent_t>(h->prof_events[i]));
    delete[] h->prof_events;
  }
  delete h;
  return LCO_OK;
}

// The plan lco_permute runs for this nnz.  An identity prefix (segments > 1) keeps the
// flat plan on LSD passes over the shaved key q (choose_plan takes MSD for one segment
// only).  When q still needs so many passes that the MSD schedule of the FULL new key
// models below it by choose_plan's own margins, the full key is sorted instead: the
// prefix digits of K' are already non-decreasing in the input, so a
// stable sort on K' and the segment-wise stable sort on q give the same output.
// (Table 2 Laplacian (0,3,2,1), 35-bit q in 4 passes: 2.73 ms vs 1.98 ms by lco_sort.)
static const OpPlan& permute_op(const lco_plan_s* h, uint64_t nnz) {
  const OpPlan& a = h->op_permute;
  if (a.segments <= 1 || nnz == 0 || a.path == kPathCopy || h->tune.no_prefix_msd) return a;
  const CallPlan ca = choose_plan(a, nnz, h->tune);
  if (ca.path != kPathOnesweep || ca.passes < 4) return a;
  const CallPlan cb = choose_plan(h->op_sort, nnz, h->tune);
  // two-level plans only: level 3 re-splits oversize buckets when the prefix
  // digits are unevenly filled; a one-level plan would defer them to the streaming leaf
  // (300K nonzeros sharing one prefix digit: 0.62 vs 0.15 ms by LSD)
  if (cb.path != kPathMsd || cb.msd.levels != 2) return a;
  return cb.cost < 0.75 * ca.cost ? h->op_sort : a;
}

lco_status lco_workspace_size(lco_handle h, uint64_t nnz, size_t* bytes) {
  lco_status st = check_handle(h);
  if (st) return st;
  if (!bytes) {
    set_error("bytes is NULL");
    return LCO_ERR_NULL;
  }
  const OpPlan& a = h->op_permute;
  const OpPlan& b = h->op_sort;
  size_t x = layout_for(choose_plan(a, nnz, h->tune), nnz).total;
  const Hier hp = hier_for(h, false, nnz);
  if (hp.use && hp.total > x) x = hp.total;
  size_t y = layout_for(choose_plan(b, nnz, h->tune), nnz).total;
  // partition (up to 2048 ranks) uses at most a single 11-bit pass
  CallPlan part;
  memset(&part, 0, sizeof part);
  part.path = kPathOnesweep;
  part.passes = 1;
  part.rb = 11;
  size_t z = layout_for(part, nnz).total;
  size_t m = x > y ? x : y;
  *bytes = m > z ? m : z;
  return LCO_OK;
}

lco_status lco_permute(lco_handle h, uint64_t nnz, const uint64_t* keys_in,
                       const double* vals_in, const uint32_t* idx_in, uint64_t* keys_out,
                       double* vals_out, uint32_t* perm_out, void* workspace,
                       size_t workspace_bytes, void* stream) {
  if (!h) return check_handle(h);
  return run_op(h, permute_op(h, nnz), false, nnz, keys_in, vals_in, idx_in, keys_out, vals_out,
                perm_out, workspace, workspace_bytes, stream);
}

lco_status lco_sort(lco_handle h, uint64_t nnz, const uint64_t* keys_in, const double* vals_in,
                    const uint32_t* idx_in, uint64_t* keys_out, double* vals_out,
                    uint32_t* perm_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!h) return check_handle(h);
  return run_op(h, h->op_sort, true, nnz, keys_in, vals_in, idx_in, keys_out, vals_out,
                perm_out, workspace, workspace_bytes, stream);
}

lco_status lco_host_workspace_size(lco_handle h, uint64_t nnz, size_t* bytes) {
  size_t inner = 0;
  lco_status st = lco_workspace_size(h, nnz, &inner);
  if (st) return st;
  *bytes = 4 * align_up(nnz * 8) + align_up(nnz * 4) + inner;
  return LCO_OK;
}

lco_status lco_permute_host(lco_handle h, uint64_t nnz, const uint64_t* keys_in,
                            const double* vals_in, uint64_t* keys_out, double* vals_out,
                            uint32_t* perm_out, void* workspace, size_t workspace_bytes,
                            void* stream) {
  lco_status st = check_handle(h);
  if (st) return st;
  if (nnz == 0) return LCO_OK;
  if (!keys_in || !keys_out) {
    set_error("keys_in and keys_out are required");
    return LCO_ERR_NULL;
  }
  if ((vals_in == nullptr) != (vals_out == nullptr)) {
    set_error("vals_in and vals_out must both be given or both be NULL");
    return LCO_ERR_ARG;
  }
  size_t need = 0;
  lco_host_workspace_size(h, nnz, &need);
  if (!workspace || workspace_bytes < need || reinterpret_cast<uintptr_t>(workspace) % kAlign) {
    set_error("host-path workspace needs %zu bytes, 256-byte aligned", need);
    return LCO_ERR_WORKSPACE;
  }
  char* ws = static_cast<char*>(workspace);
  const size_t a8 = align_up(nnz * 8), a4 = align_up(nnz * 4);
  uint64_t* dk = reinterpret_cast<uint64_t*>(ws);
  double* dv = reinterpret_cast<double*>(ws + a8);
  uint64_t* ok = reinterpret_cast<uint64_t*>(ws + 2 * a8);
  double* ov = reinterpret_cast<double*>(ws + 3 * a8);
  uint32_t* op = reinterpret_cast<uint32_t*>(ws + 4 * a8);
  char* inner = ws + 4 * a8 + a4;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(dk, keys_in, nnz * 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && vals_in) e = cudaMemcpyAsync(dv, vals_in, nnz * 8, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "lco_permute_host H2D");
  st = lco_permute(h, nnz, dk, vals_in ? dv : nullptr, nullptr, ok, vals_in ? ov : nullptr,
                   perm_out ? op : nullptr, inner, workspace_bytes - (inner - ws), stream);
  if (st) return st;
  e = cudaMemcpyAsync(keys_out, ok, nnz * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && vals_out) e = cudaMemcpyAsync(vals_out, ov, nnz * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && perm_out) e = cudaMemcpyAsync(perm_out, op, nnz * 4, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return cuda_fail(e, "lco_permute_host D2H");
  return LCO_OK;
}

lco_status lco_partition(lco_handle h, uint64_t nnz, const uint64_t* keys_in,
                         const double* vals_in, uint32_t idx_base, int world,
                         const uint64_t* splitters, uint64_t* send_keys, double* send_vals,
                         uint32_t* send_idx, uint64_t* send_counts, void* workspace,
                         size_t workspace_bytes, void* stream) {
  lco_status st = check_handle(h);
  if (st) return st;
  if (world < 1 || world > 2048) {
    set_error("world %d outside 1..2048", world);
    return LCO_ERR_ARG;
  }
  if (nnz > h->max_nnz || nnz >= (1ull << 32)) {
    set_error("nnz above max_nnz or 2^32-1");
    return LCO_ERR_CAPACITY;
  }
  if (!send_counts || (world > 1 && !splitters)) {
    set_error("send_counts (and splitters when world > 1) are required");
    return LCO_ERR_NULL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nnz == 0) {
    cudaError_t e = cudaMemsetAsync(send_counts, 0, (size_t)world * 8, s);
    return e == cudaSuccess ? LCO_OK : cuda_fail(e, "lco_partition");
  }
  if (!keys_in || !send_keys || !send_idx) {
    set_error("keys_in, send_keys and send_idx are required");
    return LCO_ERR_NULL;
  }
  if ((vals_in == nullptr) != (send_vals == nullptr)) {
    set_error("vals_in and send_vals must both be given or both be NULL");
    return LCO_ERR_ARG;
  }
  const int rb = partition_rb(world);
  CallPlan pp;
  memset(&pp, 0, sizeof pp);
  pp.path = kPathOnesweep;
  pp.passes = 1;
  pp.rb = rb;
  const WsLayout w = layout_for(pp, nnz);
  if (!workspace || workspace_bytes < w.total || reinterpret_cast<uintptr_t>(workspace) % kAlign) {
    set_error("workspace needs %zu bytes, 256-byte aligned", w.total);
    return LCO_ERR_WORKSPACE;
  }
  char* ws = static_cast<char*>(workspace);
  // world == 1: every record goes to rank 0; a single splitter-free pass still applies
  // (rank_of returns 0 for world 1), so the same kernels run.
  PassIO io;
  memset(&io, 0, sizeof io);
  io.nnz = nnz;
  io.keys_in = keys_in;
  io.vals_in = vals_in;
  io.keys_out = send_keys;
  io.vals_out = send_vals;
  io.perm_out = send_idx;
  io.ctrl = reinterpret_cast<uint32_t*>(ws + w.ctrl);
  // world == 1: rank_of never reads the splitters, any non-null marker selects the
  // partition mode of the kernels.
  io.splitters = world > 1 ? splitters : reinterpret_cast<const uint64_t*>(send_counts);
  io.world = world;
  io.idx_base = idx_base;
  io.counts64 = send_counts;
  io.tune = &h->tune;
  Launch L{s, nullptr, nullptr};
  ProfCtx pc;
  const bool prof = prof_begin(h, s, &pc, &L);
  cudaError_t e = run_passes(rb, h->kp_full, io, L);
  if (prof) prof_end(&pc);
  if (e != cudaSuccess) return cuda_fail(e, "lco_partition");
  return LCO_OK;
}

// Shared argument checks / setup of lco_partition_counts and lco_partition_direct.
static lco_status partition_setup(lco_handle h, uint64_t nnz, const uint64_t* keys_in,
                                  const double* vals_in, int world, const uint64_t* splitters,
                                  uint64_t* send_counts, void* workspace, size_t workspace_bytes,
                                  int max_world, PassIO* io, int* rb) {
  lco_status st = check_handle(h);
  if (st) return st;
  if (world < 1 || world > max_world) {
    set_error("world %d outside 1..%d", world, max_world);
    return LCO_ERR_ARG;
  }
  if (nnz > h->max_nnz || nnz >= (1ull << 32)) {
    set_error("nnz above max_nnz or 2^32-1");
    return LCO_ERR_CAPACITY;
  }
  if (!send_counts || (world > 1 && !splitters) || (nnz && !keys_in)) {
    set_error("keys_in, send_counts (and splitters when world > 1) are required");
    return LCO_ERR_NULL;
  }
  *rb = partition_rb(world);
  CallPlan pp;
  memset(&pp, 0, sizeof pp);
  pp.path = kPathOnesweep;
  pp.passes = 1;
  pp.rb = *rb;
  const WsLayout w = layout_for(pp, nnz);
  if (nnz && (!workspace || workspace_bytes < w.total ||
              reinterpret_cast<uintptr_t>(workspace) % kAlign)) {
    set_error("workspace needs %zu bytes, 256-byte aligned", w.total);
    return LCO_ERR_WORKSPACE;
  }
  memset(io, 0, sizeof *io);
  io->nnz = nnz;
  io->keys_in = keys_in;
  io->vals_in = vals_in;
  io->ctrl = reinterpret_cast<uint32_t*>(static_cast<char*>(workspace) + w.ctrl);
  io->splitters = world > 1 ? splitters : reinterpret_cast<const uint64_t*>(send_counts);
  io->world = world;
  io->counts64 = send_counts;
  io->tune = &h->tune;
  return LCO_OK;
}

lco_status lco_partition_counts(lco_handle h, uint64_t nnz, const uint64_t* keys_in, int world,
                                const uint64_t* splitters, uint64_t* send_counts,
                                void* workspace, size_t workspace_bytes, void* stream) {
  PassIO io;
  int rb = 8;
  lco_status st = partition_setup(h, nnz, keys_in, nullptr, world, splitters, send_counts,
                                  workspace, workspace_bytes, 2048, &io, &rb);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = nnz == 0 ? cudaMemsetAsync(send_counts, 0, (size_t)world * 8, s)
                           : run_partition(rb, h->kp_full, io, Launch{s, nullptr, nullptr}, true);
  return e == cudaSuccess ? LCO_OK : cuda_fail(e, "lco_partition_counts");
}

lco_status lco_partition_direct(lco_handle h, uint64_t nnz, const uint64_t* keys_in,
                                const double* vals_in, uint32_t idx_base, int world,
                                const uint64_t* splitters, uint64_t* const* recv_keys,
                                double* const* recv_vals, uint32_t* const* recv_idx,
                                const uint64_t* recv_offsets, uint64_t* send_counts,
                                void* workspace, size_t workspace_bytes, void* stream) {
  PassIO io;
  int rb = 8;
  lco_status st = partition_setup(h, nnz, keys_in, vals_in, world, splitters, send_counts,
                                  workspace, workspace_bytes, kMaxDirect, &io, &rb);
  if (st) return st;
  if (!recv_keys || !recv_idx || !recv_offsets || (vals_in && !recv_vals)) {
    set_error("recv_keys, recv_idx, recv_offsets (and recv_vals with values) are required");
    return LCO_ERR_NULL;
  }
  DirectOut d;
  memset(&d, 0, sizeof d);
  for (int r = 0; r < world; ++r) {
    if (!recv_keys[r] || !recv_idx[r] || (vals_in && !recv_vals[r])) {
      set_error("receive buffer of rank %d is NULL", r);
      return LCO_ERR_NULL;
    }
    d.k[r] = recv_keys[r];
    d.v[r] = vals_in ? recv_vals[r] : nullptr;
    d.p[r] = recv_idx[r];
    d.off[r] = recv_offsets[r];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nnz == 0) {
    cudaError_t e = cudaMemsetAsync(send_counts, 0, (size_t)world * 8, s);
    return e == cudaSuccess ? LCO_OK : cuda_fail(e, "lco_partition_direct");
  }
  io.idx_base = idx_base;
  io.direct = &d;
  io.vals_out = vals_in ? reinterpret_cast<double*>(1) : nullptr;  // selects the VALS kernels
  io.keys_out = recv_keys[0];
  Launch L{s, nullptr, nullptr};
  ProfCtx pc;
  const bool prof = prof_begin(h, s, &pc, &L);
  cudaError_t e = run_partition(rb, h->kp_full, io, L, false);
  if (prof) prof_end(&pc);
  return e == cudaSuccess ? LCO_OK : cuda_fail(e, "lco_partition_direct");
}

lco_status lco_compress_workspace_size(uint64_t nnz, int doubly, size_t* bytes) {
  if (!bytes) {
    set_error("bytes is NULL");
    return LCO_ERR_NULL;
  }
  *bytes = doubly ? align_up(compress_ctrl_bytes(nnz)) : 0;
  return LCO_OK;
}

lco_status lco_compress(uint64_t nnz, const uint64_t* keys, uint64_t n_major, uint64_t n_minor,
                        int doubly, uint64_t* ptr, uint64_t* ids, uint64_t* minor,
                        uint64_t* n_nonempty, void* workspace, size_t workspace_bytes,
                        void* stream) {
  if (!ptr || (nnz && (!keys || !minor)) || (doubly && (!ids || !n_nonempty))) {
    set_error("ptr, keys, minor (and ids, n_nonempty when doubly) are required");
    return LCO_ERR_NULL;
  }
  if (n_minor == 0 || n_major == 0 || n_major > 0x7fffffffffffffffull / n_minor) {
    set_error("n_major and n_minor must be positive with a product <= 2^63-1");
    return LCO_ERR_DIM;
  }
  size_t need = 0;
  lco_compress_workspace_size(nnz, doubly, &need);
  if (need && (!workspace || workspace_bytes < need ||
               reinterpret_cast<uintptr_t>(workspace) % kAlign)) {
    set_error("workspace needs %zu bytes, 256-byte aligned", need);
    return LCO_ERR_WORKSPACE;
  }
  Launch L{static_cast<cudaStream_t>(stream), nullptr, nullptr};
  const cudaError_t e = run_compress(nnz, keys, n_major, n_minor, doubly, ptr, ids, minor,
                                     n_nonempty, workspace, L);
  return e == cudaSuccess ? LCO_OK : cuda_fail(e, "lco_compress");
}

int lco_sparsity_class(uint64_t m, uint64_t n, uint64_t nnz, double threshold) {
  if (nnz == 0) return 0;
  const bool row = (double)m / (double)nnz > threshold, col = (double)n / (double)nnz > threshold;
  return row && col ? 3 : (row ? 1 : (col ? 2 : 0));
}

// PAPER.md Table "Multiplication possibilities" (:340-352), rows = A, columns = B, in the
// class order sparse, row-sparse, column-sparse, index-sparse.
int lco_mdt_choice(int class_a, int class_b) {
  enum { CSC_CSR = 0, CSC, CSR, DCSC_DCSR, DCSC, DCSR, CSCNA_CSRNA, CSCNA, CSRNA, SOP };
  static const int table[4][4] = {
      /* A sparse        */ {CSC_CSR, CSC, CSC, CSC},
      /* A row-sparse    */ {CSR, DCSR, CSCNA_CSRNA, CSCNA},
      /* A column-sparse */ {CSR, DCSC_DCSR, DCSC, DCSC},
      /* A index-sparse  */ {CSR, DCSR, CSRNA, SOP}};
  if (class_a < 0 || class_a > 3 || class_b < 0 || class_b > 3) return -1;
  return table[class_a][class_b];
}

const char* lco_mdt_name(int code) {
  static const char* names[] = {"CSC/CSR", "CSC", "CSR", "DCSC/DCSR", "DCSC",
                                "DCSR", "CSCNA/CSRNA", "CSCNA", "CSRNA", "SOP"};
  return code >= 0 && code < 10 ? names[code] : "invalid";
}

lco_status lco_add_workspace_size(lco_handle h, uint64_t nnz_a, uint64_t nnz_b, size_t* bytes) {
  lco_status st = check_handle(h);
  if (st) return st;
  if (!bytes) {
    set_error("bytes is NULL");
    return LCO_ERR_NULL;
  }
  size_t inner = 0;
  if ((st = lco_workspace_size(h, nnz_b, &inner)) != LCO_OK) return st;
  *bytes = 2 * align_up(nnz_b * 8) + align_up(merge_ctrl_bytes(nnz_a, nnz_b)) + inner;
  return LCO_OK;
}

lco_status lco_add(lco_handle h, uint64_t nnz_a, const uint64_t* keys_a, const double* vals_a,
                   uint64_t nnz_b, const uint64_t* keys_b, const double* vals_b, double sign,
                   uint64_t* keys_c, double* vals_c, uint64_t* nnz_c, void* workspace,
                   size_t workspace_bytes, void* stream) {
  lco_status st = check_handle(h);
  if (st) return st;
  if (!nnz_c || !keys_c || !vals_c || (nnz_a && (!keys_a || !vals_a)) ||
      (nnz_b && (!keys_b || !vals_b))) {
    set_error("nnz_c, keys_c, vals_c and the non-empty operands are required");
    return LCO_ERR_NULL;
  }
  if (nnz_b > h->max_nnz || nnz_b >= (1ull << 32) || nnz_a >= (1ull << 32)) {
    set_error("nnz_b above max_nnz, or an operand with 2^32 nonzeros or more");
    return LCO_ERR_CAPACITY;
  }
  size_t need = 0;
  lco_add_workspace_size(h, nnz_a, nnz_b, &need);
  if (!workspace || workspace_bytes < need || reinterpret_cast<uintptr_t>(workspace) % kAlign) {
    set_error("workspace needs %zu bytes, 256-byte aligned", need);
    return LCO_ERR_WORKSPACE;
  }
  const size_t nc = (size_t)(nnz_a + nnz_b);
  const void* ins[4] = {keys_a, vals_a, keys_b, vals_b};
  const size_t insz[4] = {nnz_a * 8, nnz_a * 8, nnz_b * 8, nnz_b * 8};
  const void* outs[3] = {keys_c, vals_c, nnz_c};
  const size_t outsz[3] = {nc * 8, nc * 8, 8};
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 4; ++j)
      if (overlaps(outs[i], outsz[i], ins[j], insz[j])) {
        set_error("output %d overlaps input %d", i, j);
        return LCO_ERR_ALIAS;
      }
    if (overlaps(outs[i], outsz[i], workspace, need)) {
      set_error("output %d overlaps the workspace", i);
      return LCO_ERR_ALIAS;
    }
  }
  char* ws = static_cast<char*>(workspace);
  uint64_t* kb2 = reinterpret_cast<uint64_t*>(ws);
  double* vb2 = reinterpret_cast<double*>(ws + align_up(nnz_b * 8));
  char* mctrl = ws + 2 * align_up(nnz_b * 8);
  char* inner = mctrl + align_up(merge_ctrl_bytes(nnz_a, nnz_b));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // B -> A's order: the permutation hot path ("re-sorted into the {1,0,3,2}
  // lexicographical order")
  st = lco_permute(h, nnz_b, keys_b, vals_b, nullptr, kb2, vb2, nullptr, inner,
                   workspace_bytes - (inner - ws), stream);
  if (st) return st;
  Launch L{s, nullptr, nullptr};
  ProfCtx pc;
  const bool prof = prof_begin(h, s, &pc, &L);
  cudaError_t e = run_merge(nnz_a, keys_a, vals_a, nnz_b, kb2, vb2, sign, keys_c, vals_c, nnz_c,
                            mctrl, L);
  if (prof) prof_end(&pc);
  return e == cudaSuccess ? LCO_OK : cuda_fail(e, "lco_add");
}

lco_status lco_key_histogram(lco_handle h, uint64_t nnz, const uint64_t* keys_in, int bits,
                             uint64_t* counts, void* stream) {
  lco_status st = check_handle(h);
  if (st) return st;
  if (bits < 1 || bits > 14) {
    set_error("bits %d outside 1..14", bits);
    return LCO_ERR_ARG;
  }
  if (nnz == 0) return LCO_OK;
  if (!keys_in || !counts) {
    set_error("keys_in and counts are required");
    return LCO_ERR_NULL;
  }
  const int shift = h->key_bits > bits ? h->key_bits - bits : 0;
  cudaError_t e = run_keyhist(h->kp_full, nnz, keys_in, shift, 1 << bits, counts,
                              static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LCO_OK : cuda_fail(e, "lco_key_histogram");
}

lco_status lco_plan_query(lco_handle h, uint64_t nnz, int sort, lco_plan_info* info) {
  lco_status st = check_handle(h);
  if (st) return st;
  if (!info) {
    set_error("info is NULL");
    return LCO_ERR_NULL;
  }
  memset(info, 0, sizeof *info);
  const OpPlan& op = sort ? h->op_sort : permute_op(h, nnz);
  info->order = h->order;
  for (int t = 0; t < h->order; ++t) info->rearrangement[t] = h->rearr[t];
  info->norm_order = h->norm_n;
  for (int m = 0; m < h->norm_n; ++m) {
    info->norm_dims[m] = h->norm_dims[m];
    info->norm_perm[m] = h->norm_perm[m];
  }
  info->prefix_len = h->prefix_len;
  info->suffix_start = h->suffix_start;
  info->segment_divisor = op.segdiv;
  info->trailing = op.trailing;
  info->middle_size = op.middle;
  info->num_segments = op.segments;
  info->sort_bits = op.sort_bits;
  const CallPlan cp = choose_plan(op, nnz, h->tune);
  info->passes = cp.passes;
  for (int j = 0; j < cp.passes && j < 8; ++j) info->digit_bits[j] = cp.kp.dbits[j];
  if (cp.path == kPathSeg) info->digit_bits[0] = cp.msd.b2;  // the middle digit
  info->radix_bits = (cp.path == kPathOnesweep || cp.path == kPathSingle) ? cp.rb
                                                : (cp.path == kPathMsd ? 8 : (cp.path == kPathSeg ? pass_rb(cp.msd.b2) : 0));
  info->path = cp.path;
  info->tile = cp.path == kPathSingle ? 8192
              : cp.path == kPathOnesweep || cp.path == kPathMsd
                   ? pass_tile()
                   : (cp.path == kPathTile ? (int)tile_nominal(nnz, cp.segments) : 0);
  info->msd_levels = cp.msd.levels;
  info->leaf_bits = cp.path == kPathMsd || cp.path == kPathLocal ? cp.msd.rb : 0;
  info->leaf_kind = (cp.path == kPathLocal || cp.path == kPathTile) ? 2
                                                                     : (cp.path == kPathMsd ? (cp.msd.cta ? 2 : 1) : 0);
  if (cp.path == kPathTile) info->leaf_bits = cp.msd.rb;
  info->model_bytes = cp.cost;
  info->flat_model_bytes = cp.cost;
  if (cp.path == kPathBlock) {
    info->block_grid[0] = cp.nblocks;
    info->block_grid[1] = cp.bg.dA;
    info->block_grid[2] = cp.bg.dB;
    info->block_grid[3] = cp.bg.mid;
    info->block_grid[4] = cp.bg.hi;
  }
  const Hier hp = hier_for(h, sort != 0, nnz);
  info->stages = sort ? 1 : (h->nstages >= 2 ? h->nstages : 1);
  for (int j = 0; j < h->nstages && j < 8 && !sort; ++j) {
    const CallPlan sc = choose_plan(h->stages[j].op, nnz, h->tune);
    info->stage_path[j] = sc.path;
    info->stage_sort_bits[j] = h->stages[j].op.sort_bits;
  }
  if (hp.use) {  // hierarchical: stages run one after another
    info->path = 6;
    info->model_bytes = hp.cost;
    int launches_h = 0;
    for (int j = 0; j < h->nstages; ++j) {
      lco_plan_info si;
      (void)si;
      const CallPlan sc = choose_plan(h->stages[j].op, nnz, h->tune);
      launches_h += sc.path == kPathCopy || sc.path == kPathLocal ? 1
                    : sc.path == kPathTile ? 3
                    : sc.path == kPathBlock ? 7
                    : sc.path == kPathSeg ? 6
                    : sc.path == kPathOnesweep ? 4 * sc.passes
                    : 4 + (sc.msd.levels == 2 ? 5 : 0) + 2;
    }
    info->launches = launches_h;
    return LCO_OK;
  }
  // kernels of this library per call (cudaMemsetAsync not counted)
  int launches = 0;
  if (nnz > 0) {
    if (cp.path == kPathCopy || cp.path == kPathLocal || cp.path == kPathSingle) launches = 1;
    else if (cp.path == kPathTile) launches = 3;  // bounds, tile sorts, deferred tiles
    else if (cp.path == kPathSeg) launches = 6;   // count, scan, tiles, count, offsets, scatter
    else if (cp.path == kPathBlock) launches = 5; // bounds, counts, 2 scan, tiles
    else if (cp.path == kPathOnesweep) launches = 4 * cp.passes;
    else launches = 4 + (cp.msd.levels == 2 ? 5 : 0) + 2;  // passes, leaves, deferred
    // (a sampled level 1 adds sample, caps, the cursor scatter and the finish; level 3
    // and the deferred drains add up to 8 more, most of them empty)
    if (cp.path == kPathMsd && cp.msd.sampled) launches += 4;
  }
  info->launches = launches;
  return LCO_OK;
}

lco_status lco_plan_stage(lco_handle h, int j, int* n_stages, int* order, uint64_t* dims,
                          int32_t* perm) {
  lco_status st = check_handle(h);
  if (st) return st;
  if (!n_stages || !order || !dims || !perm) {
    set_error("n_stages, order, dims and perm are required");
    return LCO_ERR_NULL;
  }
  const int ns = h->nstages >= 2 ? h->nstages : 1;
  *n_stages = ns;
  if (j < 0 || j >= ns) {
    set_error("stage %d outside 0..%d", j, ns - 1);
    return LCO_ERR_ARG;
  }
  if (h->nstages >= 2) {
    *order = h->stages[j].order;
    for (int m = 0; m < *order; ++m) {
      dims[m] = h->stages[j].dims[m];
      perm[m] = h->stages[j].perm[m];
    }
  } else {
    *order = h->norm_n;
    for (int m = 0; m < *order; ++m) {
      dims[m] = h->norm_dims[m];
      perm[m] = h->norm_perm[m];
    }
  }
  return LCO_OK;
}

lco_status lco_fastdiv_host(uint64_t d, uint64_t n, const uint64_t* x, uint64_t* q) {
  if (d == 0) {
    set_error("divisor 0");
    return LCO_ERR_ARG;
  }
  if (n && (!x || !q)) {
    set_error("x and q are required");
    return LCO_ERR_NULL;
  }
  const FastDiv f = make_fastdiv(d);
  for (uint64_t i = 0; i < n; ++i) q[i] = fdiv(f, x[i]);
  return LCO_OK;
}

lco_status lco_profile_enable(lco_handle h, int calls) {
  lco_status st = check_handle(h);
  if (st) return st;
  if (calls < 0 || calls > 64) {
    set_error("calls %d outside 0..64", calls);
    return LCO_ERR_ARG;
  }
  if (h->prof_events) {
    for (int i = 0; i < h->prof_calls_max * (kProfStages + 1); ++i)
      if (h->prof_events[i]) cudaEventDestroy(static_cast<cudaEvent_t>(h->prof_events[i]));
    delete[] h->prof_events;
    h->prof_events = nullptr;
  }
  h->prof_calls_max = calls;
  h->prof_calls = 0;
  h->prof_names[0] = 0;
  if (!calls) return LCO_OK;
  const int n = calls * (kProfStages + 1);
  h->prof_events = new (std::nothrow) void*[n];
  if (!h->prof_events) {
    set_error("out of host memory");
    return LCO_ERR_ARG;
  }
  memset(h->prof_events, 0, sizeof(void*) * n);
  for (int i = 0; i < n; ++i) {
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreate(&ev);
    if (e != cudaSuccess) return cuda_fail(e, "lco_profile_enable");
    h->prof_events[i] = ev;
  }
  return LCO_OK;
}

lco_status lco_profile_read(lco_handle h, int max_calls, int max_stages, float* ms,
                            int* n_calls, int* n_stages, char* names, size_t names_len) {
  lco_status st = check_handle(h);
  if (st) return st;
  const int calls = h->prof_calls < max_calls ? h->prof_calls : max_calls;
  int stages = 0;
  for (int c = 0; c < calls; ++c) {
    const int ns = h->prof_nstages[c < 64 ? c : 63];
    if (ns > stages) stages = ns;
    for (int s = 0; s < ns && s < max_stages; ++s) {
      float t = 0.f;
      cudaError_t e = cudaEventElapsedTime(
          &t, static_cast<cudaEvent_t>(h->prof_events[c * (kProfStages + 1) + s]),
          static_cast<cudaEvent_t>(h->prof_events[c * (kProfStages + 1) + s + 1]));
      if (e != cudaSuccess) return cuda_fail(e, "lco_profile_read");
      if (ms) ms[c * max_stages + s] = t;
    }
  }
  if (n_calls) *n_calls = calls;
  if (n_stages) *n_stages = stages;
  if (names && names_len) {
    strncpy(names, h->prof_names, names_len - 1);
    names[names_len - 1] = 0;
  }
  return LCO_OK;
}

const char* lco_status_string(lco_status s) {
  switch (s) {
    case LCO_OK: return "LCO_OK";
    case LCO_ERR_NULL: return "LCO_ERR_NULL";
    case LCO_ERR_ORDER: return "LCO_ERR_ORDER";
    case LCO_ERR_DIM: return "LCO_ERR_DIM";
    case LCO_ERR_PERM: return "LCO_ERR_PERM";
    case LCO_ERR_OVERFLOW: return "LCO_ERR_OVERFLOW";
    case LCO_ERR_CAPACITY: return "LCO_ERR_CAPACITY";
    case LCO_ERR_WORKSPACE: return "LCO_ERR_WORKSPACE";
    case LCO_ERR_ALIAS: return "LCO_ERR_ALIAS";
    case LCO_ERR_UNSORTED: return "LCO_ERR_UNSORTED";
    case LCO_ERR_KEY_RANGE: return "LCO_ERR_KEY_RANGE";
    case LCO_ERR_CUDA: return "LCO_ERR_CUDA";
    case LCO_ERR_ARG: return "LCO_ERR_ARG";
  }
  return "LCO_ERR_UNKNOWN";
}

const char* lco_last_error(void) { return last_error(); }

const char* lco_version(void) { return "lco-b200 0.1 (sm_100a)"; }

}  // extern "C"
