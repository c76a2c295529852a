/*
 * oracle_par.cpp — the oracle's permutation definition (oracle.cpp oracle_permute) run on
 * every core of the process affinity mask: the CPU baseline SURVEY.md §8(d)(ii) asks
 * for beside the single-core oracle.
 *
 * TEST / MEASUREMENT INFRASTRUCTURE ONLY (bench.py's cpu_baseline and tests/); the
 * product path never links or loads it, and it shares no code with csrc/.
 *
 * Same three steps as oracle_permute, each parallelised without changing the result:
 *   1. K'_i = LIV shuffle of keys_in[i] (plain '%' and '/' decode from the last mode,
 *      Horner re-encode under n'_t = n[perm[t]]; §3.1), an OpenMP loop;
 *   2. stable sort of (K'_i, i) by K' only ("original relative ordering is
 *      used to break ties"): __gnu_parallel::stable_sort (libstdc++ parallel mode,
 *      a multiway mergesort — stable, so the output equals std::stable_sort's);
 *   3. keys_out[j] = K'_{pi(j)}, vals_out[j] = vals_in[pi(j)] (8-byte copy), perm_out[j] =
 *      idx_in ? idx_in[pi(j)] : pi(j), an OpenMP loop.
 * Status codes as oracle.cpp.  Pinned by tests/test_oracle.py::test_parallel_oracle_*
 * (bit-identical to oracle_permute, duplicates included).
 */
#include <omp.h>

#include <cstdint>
#include <cstring>
#include <parallel/algorithm>
#include <vector>

namespace {

const uint64_t kMaxLiv = 0x7fffffffffffffffull;  // PAPER.md:173 §3.1

struct KeyIndex {
  uint64_t key;
  uint64_t i;
};

}  // namespace

extern "C" {

int oracle_par_threads(void) { return omp_get_max_threads(); }

int oracle_permute_par(int order, const uint64_t* dims, const int32_t* perm, uint64_t nnz,
                       const uint64_t* keys_in, const double* vals_in, const uint32_t* idx_in,
                       uint64_t* keys_out, double* vals_out, uint32_t* perm_out) {
  if (order < 1 || order > 64) return 1;
  std::vector<int> seen(order, 0);
  for (int t = 0; t < order; ++t) {
    if (perm[t] < 0 || perm[t] >= order || seen[perm[t]]) return 1;
    seen[perm[t]] = 1;
  }
  uint64_t total = 1;
  for (int m = 0; m < order; ++m) {
    if (dims[m] == 0 || total > kMaxLiv / dims[m]) return 3;
    total *= dims[m];
  }
  std::vector<KeyIndex> a(nnz);
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t i = 0; i < (int64_t)nnz; ++i) {
    uint64_t key = keys_in[i];
    if (key >= total) {
      bad |= 1;
      continue;
    }
    uint64_t c[64];
    for (int m = order - 1; m >= 0; --m) {
      c[m] = key % dims[m];
      key = key / dims[m];
    }
    uint64_t k2 = 0;
    for (int t = 0; t < order; ++t) k2 = k2 * dims[perm[t]] + c[perm[t]];
    a[i].key = k2;
    a[i].i = (uint64_t)i;
  }
  if (bad) return 2;
  __gnu_parallel::stable_sort(a.begin(), a.end(),
                              [](const KeyIndex& x, const KeyIndex& y) { return x.key < y.key; });
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < (int64_t)nnz; ++j) {
    keys_out[j] = a[j].key;
    if (vals_out) std::memcpy(&vals_out[j], &vals_in[a[j].i], sizeof(double));
    if (perm_out) perm_out[j] = idx_in ? idx_in[a[j].i] : (uint32_t)a[j].i;
  }
  return 0;
}

}  // extern "C"
