// launch.h — host-side launcher interface between api.cu and kernels.cu (internal).
#pragma once

#include <cuda_runtime.h>

#include <cmath>

#include "lco_internal.h"

namespace lco {

// Per-device, thread-safe one-time setup of a kernel (runtime.cu): raises its dynamic
// shared-memory limit on the current device when smem > 48 KB and returns the resident
// CTAs per SM (per_sm) and the device's SM count (sms), either pointer may be null.
cudaError_t kernel_setup(const void* fn, size_t smem, int threads, int* per_sm = nullptr,
                         int* sms = nullptr);
cudaError_t device_sms(int* sms);  // SM count of the current device (cached per device)

struct Launch {
  cudaStream_t stream;
  void (*mark)(void* ctx, const char* name);  // profiling hook (before each launch)
  void* ctx;
};

constexpr uint32_t kMaxChunks = 1024;  // persistent CTAs (chunks) per pass, upper bound

// All buffers of one multi-pass run.  Partition mode: splitters != null, single pass.
// Partition straight into the receivers' buffers (peer-mapped device pointers): record
// w of destination d goes to k[d][off[d] + w] (lco_partition_direct).
constexpr int kMaxDirect = 16;
struct DirectOut {
  uint64_t* k[kMaxDirect];
  double* v[kMaxDirect];
  uint32_t* p[kMaxDirect];
  uint64_t off[kMaxDirect];
};

struct PassIO {
  uint64_t nnz;
  const uint64_t* keys_in;
  const double* vals_in;
  const uint32_t* idx_in;
  uint64_t* keys_out;
  double* vals_out;
  uint32_t* perm_out;
  uint32_t* ctrl;  // pass_ctrl_bytes(): chunk histograms, totals, bucket starts, counter
  uint64_t* kA;    // ping-pong buffers (K', V, source position)
  double* vA;
  uint32_t* pA;
  uint64_t* kB;
  double* vB;
  uint32_t* pB;
  const uint64_t* splitters;
  int world;
  uint32_t idx_base;
  uint64_t* counts64;
  const DirectOut* direct;  // partition: scatter into the receivers' buffers
  const Tuning* tune;       // the handle's schedule overrides (never null on a call)
  int unique;               // keys are unique (lco_permute's precondition): MSD passes may
                            // place records unordered inside a digit run (k_scatter UNST)
};

// Pointers into a pass control block (pass_ctrl_bytes()).
struct PassCtrl {
  uint16_t* thist;  // [tiles][bins] tile histograms
  uint32_t* toff;   // [tiles][bins] global position of each tile's digit runs
  uint32_t* csum;   // [chunks][bins] chunk sums -> exclusive prefix over chunks
  uint32_t* totals; // [bins] digit totals
  uint32_t* bucket; // [bins] digit bucket starts
  uint32_t* done;   // k_scan completion counter
  uint32_t tiles, nchunks;
};

// MSD-hybrid schedule (msd.cu): `levels` stable MSD passes of b1 (and b2) bits, then
// on-chip leaf sorts of the remaining rb bits of q.  levels == 0: the whole input is
// one leaf.
struct MsdPlan {
  int levels;
  int b1, b2;
  int rb;
  int cta;     // leaves sorted by one CTA per leaf instead of k_leafw (one warp)
  int staged;  // CTA leaves of <= ~2K nonzeros: the fully staged k_leafs
  int sampled; // level 1 from sampled capacities (buffer A padded: sampled_capacity)
};
// Sampled MSD level 1: one key in kSampleStride is histogrammed (msd.cu k_sample1).
constexpr uint32_t kSampleStride = 512;
// Buffer A's length (records) for a sampled level 1: a bound on the padded capacities'
// sum (k_caps: est_d + 6 sqrt(S est_d) + 4,096 over 256 digits, S = kSampleStride,
// sum est_d <= nnz + S; Cauchy-Schwarz: sum sqrt(est_d) <= 16 sqrt(nnz + S)).
inline uint64_t sampled_capacity(uint64_t nnz) {
  uint64_t r = (uint64_t)std::sqrt((double)(nnz + kSampleStride));
  while (r * r < nnz + kSampleStride) ++r;  // ceil(sqrt(nnz + S))
  const uint64_t k = (uint64_t)std::ceil(96.0 * std::sqrt((double)kSampleStride));  // 6 * 16
  return nnz + kSampleStride + k * r + 256 * 4096 + 4096;
}
constexpr size_t kSampledCtrlBytes = 5 * 1024;

struct PassParams;
struct ScatterIO;

uint64_t pass_tiles(uint64_t nnz, uint32_t tile = 4096);
uint32_t prefetch_distance();  // L2 prefetch distance of the pass kernels (tiles)
int pass_tile();
int pass_rb(int bits);
size_t pass_ctrl_bytes(int rb, uint64_t nnz, uint32_t tile = 4096);
PassCtrl pass_ctrl_layout(int rb, uint64_t nnz, uint32_t* ctrl, uint32_t tile = 4096);
cudaError_t launch_count(int rb, bool first, const PassParams& a, const uint64_t* keys,
                         uint16_t* thist, uint32_t* csum, uint32_t grid, cudaStream_t s);
cudaError_t launch_scatter(int rb, bool first, bool last, bool vals, const PassParams& a,
                           const ScatterIO& io, uint32_t grid, cudaStream_t s);
ScatterIO pass_buffers(const PassIO& io, int j, bool last, const uint32_t* toff);
cudaError_t run_pass(int rb, const PassParams& a, const PassIO& io, int j, bool first, bool last,
                     const Launch& L, bool count_only = false);
cudaError_t run_passes(int rb, const KeyPlan& kp, const PassIO& io, const Launch& L);
// nnz <= 8,192 and one digit of <= 10 bits: one CTA, one stable pass (kernels.cu)
cudaError_t run_single_tile(int rb, const KeyPlan& kp, const PassIO& io, const Launch& L);
// the same pass on a cluster of 8 CTAs exchanging digit counts through DSMEM (small.cu)
cudaError_t run_single_cluster(int rb, const KeyPlan& kp, const PassIO& io, const Launch& L);
// partition (io.splitters set): one pass; count_only stops after the digit totals
// (io.counts64 written)
cudaError_t run_partition(int rb, const KeyPlan& kp, const PassIO& io, const Launch& L,
                          bool count_only);
uint32_t leaf_cap();      // largest leaf one CTA sorts in shared memory
uint32_t leaf_target();   // expected leaf size the MSD digits aim for (warp leaves)
uint32_t cta_leaf_cap();  // largest leaf k_leafc sorts
uint32_t staged_leaf_target();  // expected leaf size for k_leafs
size_t msd_ctrl_bytes(int b1, int b2, uint64_t nnz, uint32_t tile = 4096);
cudaError_t run_msd(const MsdPlan& mp, const KeyPlan& kp, const PassIO& io, const Launch& L);
uint32_t tile_nominal(uint64_t nnz, uint64_t segments);  // segment-local path (msd.cu)
cudaError_t run_seg(int gb, int mb, const KeyPlan& kp, const PassIO& io, const Launch& L);
// exclusive scan of n uint32 counts into uint64 offsets and *total (one CTA, add.cu)
cudaError_t run_count_scan(const uint32_t* counts, uint64_t n, uint64_t* offsets, uint64_t* total,
                           const Launch& L);
// block-transpose schedule (block.cu)
// grid of blocks as (hi, B, mid, A): dims of the old-innermost block mode A and the
// new-innermost block mode B, products of the block modes before B / between B and A
struct BlockGrid {
  uint64_t dA, dB, mid, hi;
};
size_t block_ctrl_bytes(uint64_t nblocks);
cudaError_t run_block(const KeyPlan& kp, const KeyPlan& kb, uint64_t nblocks, uint64_t F,
                      const BlockGrid& bg, const PassIO& io, const Launch& L);
// compressed matrix datatypes (mdt.cu)
size_t compress_ctrl_bytes(uint64_t nnz);
cudaError_t run_compress(uint64_t nnz, const uint64_t* keys, uint64_t n_major, uint64_t n_minor,
                         int doubly, uint64_t* ptr, uint64_t* ids, uint64_t* minor,
                         uint64_t* n_nonempty, void* ctrl, const Launch& L);
// index-matched addition (add.cu)
uint64_t merge_tiles(uint64_t na, uint64_t nb);
size_t merge_ctrl_bytes(uint64_t na, uint64_t nb);
cudaError_t run_merge(uint64_t na, const uint64_t* ka, const double* va, uint64_t nb,
                      const uint64_t* kb, const double* vb, double sign, uint64_t* kc,
                      double* vc, uint64_t* nnz_c, void* ctrl, const Launch& L);
size_t tile_ctrl_bytes(uint64_t nnz, uint64_t segments);
cudaError_t run_tiles(const KeyPlan& kp, uint64_t segdiv, uint64_t segments, int key_bits,
                      const PassIO& io, const Launch& L);
cudaError_t run_copy(uint64_t nnz, const uint64_t* keys_in, const double* vals_in,
                     const uint32_t* idx_in, uint64_t* keys_out, double* vals_out,
                     uint32_t* perm_out, const Launch& L);
cudaError_t run_validate(uint64_t nnz, const uint64_t* keys, uint64_t total, int need_sorted,
                         uint32_t* flag, cudaStream_t s);
cudaError_t run_keyhist(const KeyPlan& kp, uint64_t nnz, const uint64_t* keys, int shift,
                        int bins, uint64_t* counts, cudaStream_t s);

}  // namespace lco
