// launch.h — host-side launcher interface between api.cu and kernels.cu (internal).
#pragma once

#include <cuda_runtime.h>

#include "lco_internal.h"

namespace lco {

struct Launch {
  cudaStream_t stream;
  void (*mark)(void* ctx, const char* name);  // profiling hook (before each launch)
  void* ctx;
};

constexpr uint32_t kMaxChunks = 1024;  // persistent CTAs (chunks) per pass, upper bound

// All buffers of one multi-pass run.  Partition mode: splitters != null, single pass.
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
};

uint64_t pass_tiles(uint64_t nnz);
int pass_tile();
size_t pass_ctrl_bytes(int rb, uint64_t nnz);
cudaError_t run_passes(int rb, const KeyPlan& kp, const PassIO& io, const Launch& L);
cudaError_t run_copy(uint64_t nnz, const uint64_t* keys_in, const double* vals_in,
                     const uint32_t* idx_in, uint64_t* keys_out, double* vals_out,
                     uint32_t* perm_out, const Launch& L);
cudaError_t run_validate(uint64_t nnz, const uint64_t* keys, uint64_t total, int need_sorted,
                         uint32_t* flag, cudaStream_t s);
cudaError_t run_keyhist(const KeyPlan& kp, uint64_t nnz, const uint64_t* keys, int shift,
                        int bins, uint64_t* counts, cudaStream_t s);

}  // namespace lco
