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

// All buffers of one onesweep run.  Partition mode: splitters != null, single pass.
struct OnesweepIO {
  uint64_t nnz;
  const uint64_t* keys_in;
  const double* vals_in;
  const uint32_t* idx_in;
  uint64_t* keys_out;
  double* vals_out;
  uint32_t* perm_out;
  uint32_t* ctrl;
  uint32_t* statusA;
  uint32_t* statusB;
  uint64_t* kA;
  uint32_t* pA;
  uint64_t* kB;
  uint32_t* pB;
  const uint64_t* splitters;
  int world;
  uint32_t idx_base;
  uint64_t* counts64;
};

size_t onesweep_ctrl_bytes(int rb);
uint64_t onesweep_tiles(uint64_t nnz);
int onesweep_tile();
cudaError_t run_onesweep(int rb, const KeyPlan& kp, const OnesweepIO& io, const Launch& L);
cudaError_t run_copy(uint64_t nnz, const uint64_t* keys_in, const double* vals_in,
                     const uint32_t* idx_in, uint64_t* keys_out, double* vals_out,
                     uint32_t* perm_out, const Launch& L);
cudaError_t run_validate(uint64_t nnz, const uint64_t* keys, uint64_t total, int need_sorted,
                         uint32_t* flag, cudaStream_t s);
cudaError_t run_keyhist(const KeyPlan& kp, uint64_t nnz, const uint64_t* keys, int shift,
                        int bins, uint64_t* counts, cudaStream_t s);

}  // namespace lco
