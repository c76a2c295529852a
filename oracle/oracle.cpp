/*
 * oracle.cpp — plain, slow, obviously-correct CPU oracle for permuting a sorted
 * LCO sparse tensor (arXiv 1802.02619, Harrison & Joseph).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_1802_02619_b200/, liblco.so) never links, imports or calls it, and this
 * file shares no code, header, table or constant generator with csrc/.
 *
 * Conventions:
 *   - keys are row-major linear indices: K = ((c0*n1 + c1)*n2 + c2)...; mode 0 is
 *     the most significant.  The paper writes the same encoding with the first
 *     index least significant, LIV = i + n_i(j + n_j k) (§3.1);
 *     relabelling modes mu -> N-1-mu maps one onto the other.
 *   - perm has torch.permute semantics: output mode t is input mode perm[t],
 *     n'_t = n[perm[t]].
 *   - values are moved as 8-byte bit patterns (memcpy), never computed on.
 *
 * Every arithmetic step uses plain '/' and '%' on uint64 and std::stable_sort.
 * Status codes: 0 ok, 1 bad argument, 2 coordinate/key out of range,
 *               3 product of dims overflows 2^63-1, 4 internal claim violated.
 *
 * Parity status: every exported function is pinned by tests/test_oracle.py
 * (worked examples of PAPER.md Table 1 and Fig 3, dense brute-force transposes,
 * closed forms of the stencil operators, invariants).  None is "parity unpinned".
 */
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <vector>

namespace {

const uint64_t kMaxLiv = 0x7fffffffffffffffull;  // signed 64-bit limit, §3.1

// Product of dims; returns false if it exceeds 2^63-1 or a dim is 0.
bool dims_product(int order, const uint64_t* dims, uint64_t* out) {
  uint64_t p = 1;
  for (int m = 0; m < order; ++m) {
    if (dims[m] == 0) return false;
    if (p > kMaxLiv / dims[m]) return false;
    p *= dims[m];
  }
  *out = p;
  return true;
}

bool perm_is_bijection(int order, const int32_t* perm) {
  std::vector<int> seen(order, 0);
  for (int t = 0; t < order; ++t) {
    if (perm[t] < 0 || perm[t] >= order || seen[perm[t]]) return false;
    seen[perm[t]] = 1;
  }
  return true;
}

// Row-major decode with plain % and / from the last mode
// ("indices are computed on-the-fly using integer division and modulo", Fig 3).
void decode(int order, const uint64_t* dims, uint64_t key, uint64_t* coords) {
  for (int m = order - 1; m >= 0; --m) {
    coords[m] = key % dims[m];
    key = key / dims[m];
  }
}

// LIV shuffle of one key (§3.1): decode under the old order, Horner-encode
// under the new order n'_t = n[perm[t]].
uint64_t reencode(int order, const uint64_t* dims, const int32_t* perm, uint64_t key,
                  uint64_t* scratch) {
  decode(order, dims, key, scratch);
  uint64_t k2 = 0;
  for (int t = 0; t < order; ++t) k2 = k2 * dims[perm[t]] + scratch[perm[t]];
  return k2;
}

struct KeyIndex {
  uint64_t key;
  uint64_t i;
};

}  // namespace

extern "C" {

// A1 linearize (§3.1, row-major reading C1).
int oracle_linearize(int order, const uint64_t* dims, const uint64_t* coords, uint64_t* key) {
  uint64_t total;
  if (order < 1 || !dims_product(order, dims, &total)) return 3;
  uint64_t k = 0;
  for (int m = 0; m < order; ++m) {
    if (coords[m] >= dims[m]) return 2;
    k = k * dims[m] + coords[m];
  }
  *key = k;
  return 0;
}

// A2 delinearize (Fig 3 caption).
int oracle_delinearize(int order, const uint64_t* dims, uint64_t key, uint64_t* coords) {
  uint64_t total;
  if (order < 1 || !dims_product(order, dims, &total)) return 3;
  if (key >= total) return 2;
  decode(order, dims, key, coords);
  return 0;
}

// A3 LIV shuffle of an array (§3.1-3.2).  Order of keys unchanged.
int oracle_shuffle(int order, const uint64_t* dims, const int32_t* perm, uint64_t nnz,
                   const uint64_t* keys_in, uint64_t* keys_out) {
  uint64_t total;
  if (order < 1 || order > 64 || !perm_is_bijection(order, perm)) return 1;
  if (!dims_product(order, dims, &total)) return 3;
  uint64_t scratch[64];
  for (uint64_t i = 0; i < nnz; ++i) {
    if (keys_in[i] >= total) return 2;
    keys_out[i] = reencode(order, dims, perm, keys_in[i], scratch);
  }
  return 0;
}

// The permutation result (SURVEY.md §8(c) "Definition"; "result equals
// shuffle_livs(t, new_lex) followed by a full stable sort (the oracle)"):
//   1. K'_i = LIV shuffle of keys_in[i]
//   2. stable sort of (K'_i, i) by K' only; ties keep input order
//   3. keys_out[j] = K'_{pi(j)}, vals_out[j] = vals_in[pi(j)] (bit copy),
//      perm_out[j] = idx_in ? idx_in[pi(j)] : pi(j)
// This definition never relies on keys_in being sorted, so it is also the oracle of
// lco_sort (sorting unsorted LCO data, §3.2).
// vals_in/vals_out/perm_out may be NULL (not produced).
int oracle_permute(int order, const uint64_t* dims, const int32_t* perm, uint64_t nnz,
                   const uint64_t* keys_in, const double* vals_in, const uint32_t* idx_in,
                   uint64_t* keys_out, double* vals_out, uint32_t* perm_out) {
  uint64_t total;
  if (order < 1 || order > 64 || !perm_is_bijection(order, perm)) return 1;
  if (!dims_product(order, dims, &total)) return 3;
  std::vector<KeyIndex> a(nnz);
  uint64_t scratch[64];
  for (uint64_t i = 0; i < nnz; ++i) {
    if (keys_in[i] >= total) return 2;
    a[i].key = reencode(order, dims, perm, keys_in[i], scratch);
    a[i].i = i;
  }
  std::stable_sort(a.begin(), a.end(),
                   [](const KeyIndex& x, const KeyIndex& y) { return x.key < y.key; });
  for (uint64_t j = 0; j < nnz; ++j) {
    keys_out[j] = a[j].key;
    if (vals_out) std::memcpy(&vals_out[j], &vals_in[a[j].i], sizeof(double));
    if (perm_out) perm_out[j] = idx_in ? idx_in[a[j].i] : (uint32_t)a[j].i;
  }
  return 0;
}

int oracle_sort(int order, const uint64_t* dims, const int32_t* perm, uint64_t nnz,
                const uint64_t* keys_in, const double* vals_in, const uint32_t* idx_in,
                uint64_t* keys_out, double* vals_out, uint32_t* perm_out) {
  return oracle_permute(order, dims, perm, nnz, keys_in, vals_in, idx_in, keys_out, vals_out,
                        perm_out);
}

// A9 RP step 1 (§4.1): index perm[t] is a rearrangement index iff it crosses
// an index that originally had a higher significance, i.e. some mode m' that was more
// significant in the old order (m' < perm[t], row-major) is less significant in the new
// order (appears at a position t' > t).  Otherwise it is a resting index.
// out[t] = 1 for rearrangement, 0 for resting, indexed by NEW position t.
int oracle_classify(int order, const int32_t* perm, int32_t* out) {
  if (order < 1 || order > 64 || !perm_is_bijection(order, perm)) return 1;
  for (int t = 0; t < order; ++t) {
    int crosses = 0;
    for (int u = t + 1; u < order; ++u)
      if (perm[u] < perm[t]) crosses = 1;
    out[t] = crosses;
  }
  return 0;
}

// The paper's RP algorithm, step by step (§4.1, Fig 3):
//   1. recompute the LIVs into the new order (LIV shuffle, "the first step");
//   2. classify indices as rearrangement / resting;
//   3. working from highest to lowest significance of the new LIVs: a resting index
//      splits the current regions into regions where it is constant, found by a linear
//      scan; a run of rearrangement indices is handled by stably
//      sorting each region on the shaved key (LIV mod region) div trailing
//      ("(LIV mod 30) div 3"), after which the regions split on that key;
//   4. the final index is always resting, so the process ends.
// A resting split relies on each region already being ordered by that index; the
// oracle checks it and returns 4 if the paper's claim were ever violated.
// keys_in must be sorted ascending (the RP precondition); returns 1 if not.
int oracle_rp_permute(int order, const uint64_t* dims, const int32_t* perm, uint64_t nnz,
                      const uint64_t* keys_in, const double* vals_in, const uint32_t* idx_in,
                      uint64_t* keys_out, double* vals_out, uint32_t* perm_out) {
  uint64_t total;
  if (order < 1 || order > 64 || !perm_is_bijection(order, perm)) return 1;
  if (!dims_product(order, dims, &total)) return 3;
  for (uint64_t i = 1; i < nnz; ++i)
    if (keys_in[i - 1] >= keys_in[i]) return 1;
  // step 1: LIV shuffle
  std::vector<uint64_t> k2(nnz);
  uint64_t scratch[64];
  for (uint64_t i = 0; i < nnz; ++i) {
    if (keys_in[i] >= total) return 2;
    k2[i] = reencode(order, dims, perm, keys_in[i], scratch);
  }
  // step 2: classification
  std::vector<int32_t> rearr(order);
  oracle_classify(order, perm, rearr.data());
  // weights of new positions: W_t = prod_{t' > t} n'_{t'}
  std::vector<uint64_t> w(order);
  {
    uint64_t acc = 1;
    for (int t = order - 1; t >= 0; --t) {
      w[t] = acc;
      acc *= dims[perm[t]];
    }
  }
  std::vector<uint64_t> ord(nnz);
  for (uint64_t i = 0; i < nnz; ++i) ord[i] = i;
  std::vector<std::pair<uint64_t, uint64_t>> regions;  // [begin, end) into ord
  if (nnz) regions.push_back({0, nnz});
  int t = 0;
  while (t < order) {
    int u = t;
    uint64_t radix;  // range of the key examined at this step
    if (!rearr[t]) {
      u = t + 1;
      radix = dims[perm[t]];
    } else {
      radix = 1;
      while (u < order && rearr[u]) radix *= dims[perm[u++]];
      // u < order always: the final index is resting
    }
    // shaved key of new positions [t, u): (K' div W_{u-1}) mod prod n'
    auto shaved = [&](uint64_t i) { return (k2[i] / w[u - 1]) % radix; };
    std::vector<std::pair<uint64_t, uint64_t>> next;
    for (auto& r : regions) {
      if (rearr[t]) {
        std::stable_sort(ord.begin() + r.first, ord.begin() + r.second,
                         [&](uint64_t x, uint64_t y) { return shaved(x) < shaved(y); });
      }
      // linear scan for region ends
      uint64_t b = r.first;
      while (b < r.second) {
        uint64_t e = b + 1;
        uint64_t v = shaved(ord[b]);
        while (e < r.second && shaved(ord[e]) == v) ++e;
        if (e < r.second && shaved(ord[e]) < v) return 4;  // region not ordered: claim violated
        next.push_back({b, e});
        b = e;
      }
    }
    regions.swap(next);
    t = u;
  }
  for (uint64_t j = 0; j < nnz; ++j) {
    keys_out[j] = k2[ord[j]];
    if (vals_out) std::memcpy(&vals_out[j], &vals_in[ord[j]], sizeof(double));
    if (perm_out) perm_out[j] = idx_in ? idx_in[ord[j]] : (uint32_t)ord[j];
  }
  return 0;
}

// Stable partition by destination rank for the sharded path:
// dest(i) = number of splitters s with s <= K'_i (splitters ascending, world-1 of them).
// Records go to send buffers grouped by dest, each group in input order; each record is
// (old key, value, idx_base + i).  counts[r] = records for rank r.
int oracle_partition(int order, const uint64_t* dims, const int32_t* perm, uint64_t nnz,
                     const uint64_t* keys_in, const double* vals_in, uint32_t idx_base,
                     int world, const uint64_t* splitters, uint64_t* send_keys,
                     double* send_vals, uint32_t* send_idx, uint64_t* counts) {
  uint64_t total;
  if (order < 1 || order > 64 || world < 1 || !perm_is_bijection(order, perm)) return 1;
  if (!dims_product(order, dims, &total)) return 3;
  std::vector<int> dest(nnz);
  uint64_t scratch[64];
  for (int r = 0; r < world; ++r) counts[r] = 0;
  for (uint64_t i = 0; i < nnz; ++i) {
    if (keys_in[i] >= total) return 2;
    uint64_t k2 = reencode(order, dims, perm, keys_in[i], scratch);
    int r = 0;
    while (r < world - 1 && splitters[r] <= k2) ++r;
    dest[i] = r;
    counts[r]++;
  }
  uint64_t pos = 0;
  for (int r = 0; r < world; ++r)
    for (uint64_t i = 0; i < nnz; ++i)
      if (dest[i] == r) {
        send_keys[pos] = keys_in[i];
        std::memcpy(&send_vals[pos], &vals_in[i], sizeof(double));
        send_idx[pos] = idx_base + (uint32_t)i;
        ++pos;
      }
  return 0;
}

// Index-matched addition C = A + sign * B (§3.2 "one of the tensors must
// be re-sorted into the {1,0,3,2} lexicographical order ... the run time for the addition
// operation"; SPEC add(tA, tB, match, sign)): B (dims_b, sorted) is permuted by `match`
// into A's mode order with oracle_permute, then the union of the two supports is formed
// with a std::map from key to value (A's value first, then sign * B's added): every key
// of either operand appears once, collisions are summed, explicit zeros are kept, and the
// output is ascending.  A's keys must be unique (a sorted LCO tensor); values are fp64,
// one IEEE addition per collision.  *nnz_c receives the output size (<= nnz_a + nnz_b).
int oracle_add(int order, const uint64_t* dims_b, const int32_t* match, uint64_t nnz_a,
               const uint64_t* keys_a, const double* vals_a, uint64_t nnz_b,
               const uint64_t* keys_b, const double* vals_b, double sign, uint64_t* keys_c,
               double* vals_c, uint64_t* nnz_c) {
  if (order < 1 || !dims_b || !match || !nnz_c || (nnz_a && (!keys_a || !vals_a)) ||
      (nnz_b && (!keys_b || !vals_b)))
    return 1;
  std::vector<uint64_t> kb(nnz_b);
  std::vector<double> vb(nnz_b);
  std::vector<uint32_t> pb(nnz_b);
  int rc = oracle_permute(order, dims_b, match, nnz_b, keys_b, vals_b, nullptr, kb.data(),
                          vb.data(), pb.data());
  if (rc) return rc;
  std::map<uint64_t, double> c;
  for (uint64_t i = 0; i < nnz_a; ++i) {
    if (c.count(keys_a[i])) return 1;  // A must have unique keys
    c[keys_a[i]] = vals_a[i];
  }
  for (uint64_t i = 0; i < nnz_b; ++i) {
    auto it = c.find(kb[i]);
    if (it == c.end()) c[kb[i]] = sign * vb[i];
    else it->second = it->second + sign * vb[i];
  }
  uint64_t j = 0;
  for (const auto& kv : c) {
    keys_c[j] = kv.first;
    vals_c[j] = kv.second;
    ++j;
  }
  *nnz_c = j;
  return 0;
}

// Compression of a major-first LCO matrix into CSR/CSC (doubly = 0) or DCSR/DCSC
// (doubly = 1) (§5.2 step 2, :325-331, :453), by the definitions: major =
// key / n_minor, minor = key % n_minor; singly: ptr[r] = number of nonzeros with major
// < r (r = 0..n_major); doubly: ids = the distinct majors in order, ptr[j] = position of
// the first nonzero of ids[j], ptr[nz] = nnz.  Keys must be strictly increasing.
int oracle_compress(uint64_t nnz, const uint64_t* keys, uint64_t n_major, uint64_t n_minor,
                    int doubly, uint64_t* ptr, uint64_t* ids, uint64_t* minor, uint64_t* nz) {
  if (!ptr || !minor || n_minor == 0 || (nnz && !keys) || (doubly && (!ids || !nz))) return 1;
  for (uint64_t i = 0; i < nnz; ++i) {
    if (keys[i] / n_minor >= n_major) return 2;
    if (i && keys[i] <= keys[i - 1]) return 1;
    minor[i] = keys[i] % n_minor;
  }
  if (!doubly) {
    std::vector<uint64_t> count(n_major, 0);
    for (uint64_t i = 0; i < nnz; ++i) count[keys[i] / n_minor] += 1;
    ptr[0] = 0;
    for (uint64_t r = 0; r < n_major; ++r) ptr[r + 1] = ptr[r] + count[r];
    return 0;
  }
  uint64_t j = 0;
  for (uint64_t i = 0; i < nnz; ++i) {
    const uint64_t r = keys[i] / n_minor;
    if (i == 0 || r != keys[i - 1] / n_minor) {
      ids[j] = r;
      ptr[j] = i;
      ++j;
    }
  }
  ptr[j] = nnz;
  *nz = j;
  return 0;
}

}  // extern "C"
