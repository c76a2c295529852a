// runtime.cu — per-device kernel setup shared by every launcher (internal).
//
// cudaFuncAttributeMaxDynamicSharedMemorySize and the occupancy it allows belong to a
// device context, and a handle may be used from several host threads and on several
// devices at once (include/lco.h "Threading").  kernel_setup() therefore keys its cache
// by (device ordinal, kernel, shared-memory bytes, threads) under a mutex: the first
// launch of a kernel on a device sets its attribute there, later launches read the cache.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

#include "launch.h"

namespace lco {

namespace {

struct Setup {
  int per_sm;
};

std::mutex g_mu;
std::map<std::tuple<int, const void*, size_t, int>, Setup> g_setup;
std::map<int, int> g_sms;
std::map<std::pair<int, const void*>, size_t> g_attr;  // largest attribute set per kernel

}  // namespace

cudaError_t device_sms(int* sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_sms.find(dev);
  if (it == g_sms.end()) {
    int n = 0;
    e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    it = g_sms.emplace(dev, n).first;
  }
  *sms = it->second;
  return cudaSuccess;
}

cudaError_t kernel_setup(const void* fn, size_t smem, int threads, int* per_sm, int* sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (sms && (e = device_sms(sms)) != cudaSuccess) return e;
  const auto key = std::make_tuple(dev, fn, smem, threads);
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_setup.find(key);
  if (it == g_setup.end()) {
    // the attribute only grows: a kernel launched with several shared-memory sizes keeps
    // the largest one set
    size_t& cur = g_attr[std::make_pair(dev, fn)];
    if (smem > 48 * 1024 && smem > cur) {
      if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
          cudaSuccess)
        return e;
      cur = smem;
    }
    int n = 1;
    if (threads > 0 &&
        (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem)) != cudaSuccess)
      return e;
    it = g_setup.emplace(key, Setup{n < 1 ? 1 : n}).first;
  }
  if (per_sm) *per_sm = it->second.per_sm;
  return cudaSuccess;
}

}  // namespace lco
