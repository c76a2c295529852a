/*
 * lco.h — C ABI of the B200-native LCO sparse-tensor permutation library (liblco.so).
 *
 * Operation (§3.1 and §4, arXiv 1802.02619): a sparse tensor in Linearized
 * Coordinate (LCO) form is a contiguous array of linear index values (LIVs, here
 * "keys") plus a separate contiguous value array ("satellite
 * data").  Permuting it into a new lexicographical order means recomputing every key
 * under the new order (the LIV shuffle) and rearranging the
 * already-sorted nonzeros into the new order ("permutation"), which the
 * paper does with a stable radix sort on only the key digits the permutation
 * disturbs (the RP algorithm, §4.1).
 *
 * Conventions (DESIGN.md "Readings" R1/R2):
 *   - keys are row-major: K = ((c_0*n_1 + c_1)*n_2 + c_2)...; mode 0 most significant
 *     (the paper lists the same encoding least-significant index first).
 *   - perm has torch.permute semantics: output mode t is input mode perm[t]; the new
 *     dims are n'_t = n_{perm[t]}; the new key is the row-major encoding of
 *     (c_{perm[0]}, ..., c_{perm[N-1]}).
 *   - keys are uint64 with prod(dims) <= 2^63-1 (PAPER.md:173 signed 64-bit limit);
 *     values are fp64 moved as 8-byte bit patterns (never computed on);
 *     permutation vectors are uint32 (nnz < 2^32).
 *
 * Memory: every array pointer is a CUDA DEVICE pointer unless marked [host].  The
 * caller owns all device memory (outputs and the workspace); the library never calls
 * cudaMalloc.  A handle owns only its host-side plan.  Every device entry point is
 * stream-ordered on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 * stream) and never synchronizes the device, except with LCO_FLAG_VALIDATE (below).
 *
 * Errors: every entry returns an lco_status; the library never aborts or throws across
 * the ABI.  Argument errors are detected on the host before any launch and leave the
 * outputs untouched.  Asynchronous kernel faults surface as LCO_ERR_CUDA on a later
 * call.  lco_last_error() returns a thread-local message for the last non-OK status.
 * A handle is immutable after lco_create and may be used concurrently from several
 * host threads / streams provided each call has its own workspace.
 */
#ifndef LCO_H
#define LCO_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define LCO_API __attribute__((visibility("default")))
#else
#define LCO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum lco_status {
  LCO_OK = 0,
  LCO_ERR_NULL = 1,       /* a required pointer is NULL */
  LCO_ERR_ORDER = 2,      /* order < 1 or order > LCO_MAX_ORDER */
  LCO_ERR_DIM = 3,        /* a dim is 0 */
  LCO_ERR_PERM = 4,       /* perm is not a bijection on 0..order-1 */
  LCO_ERR_OVERFLOW = 5,   /* prod(dims) > 2^63-1 */
  LCO_ERR_CAPACITY = 6,   /* nnz > max_nnz given at create, or nnz >= 2^32 */
  LCO_ERR_WORKSPACE = 7,  /* workspace NULL, too small or not 256-byte aligned */
  LCO_ERR_ALIAS = 8,      /* an output range overlaps an input range or another output */
  LCO_ERR_UNSORTED = 9,   /* LCO_FLAG_VALIDATE: keys_in not strictly increasing */
  LCO_ERR_KEY_RANGE = 10, /* LCO_FLAG_VALIDATE: a key >= prod(dims) */
  LCO_ERR_CUDA = 11,      /* a CUDA runtime error (launch failure, earlier fault) */
  LCO_ERR_ARG = 12        /* any other invalid argument (e.g. vals_in without vals_out) */
} lco_status;

#define LCO_MAX_ORDER 16
#define LCO_FLAG_VALIDATE 1u /* O(nnz) precondition check; SYNCHRONIZES the stream */
#define LCO_FLAG_HIERARCHICAL 2u /* lco_permute runs the hierarchical plan (one stable
                                    sort per run of rearrangement indices, PAPER.md:
                                    245-247) when it has >= 2 stages; default: flat plan */

typedef struct lco_plan_s* lco_handle;

/* Create a permutation plan (host only; no device memory, no CUDA calls).
 *   out      [host] receives the handle.
 *   order    1..LCO_MAX_ORDER.
 *   dims     [host] order positive sizes n_0..n_{N-1}, prod <= 2^63-1.
 *   perm     [host] order ints, a bijection (torch.permute semantics); NULL = identity.
 *   max_nnz  largest nnz the handle will be called with (< 2^32).
 *   flags    0 or LCO_FLAG_VALIDATE | LCO_FLAG_HIERARCHICAL.
 * The plan normalizes the permutation (drops size-1 modes, fuses modes adjacent in
 * both orders), classifies indices as rearrangement / resting, and
 * selects the key digits to sort: the middle modes between the identity prefix and the
 * longest increasing suffix (the paper's key shaving "(LIV mod 30) div 3"). */
LCO_API lco_status lco_create(lco_handle* out, int order, const uint64_t* dims, const int32_t* perm,
                      uint64_t max_nnz, uint32_t flags);

/* Release a handle (host memory only).  NULL is accepted. */
LCO_API lco_status lco_destroy(lco_handle h);

/* Device workspace bytes needed by lco_permute / lco_sort / lco_partition for nnz
 * nonzeros.  bytes [host] receives the size (0 is possible). */
LCO_API lco_status lco_workspace_size(lco_handle h, uint64_t nnz, size_t* bytes);

/* Permute a sorted LCO tensor (§4.1 "RP").
 *   keys_in   nnz uint64 keys, strictly increasing, each < prod(dims)  (precondition;
 *             checked only with LCO_FLAG_VALIDATE, otherwise a violation yields some
 *             permutation of the input and stays memory-safe).
 *   vals_in   nnz fp64 values or NULL (keys only).
 *   idx_in    nnz uint32 source indices or NULL (= 0..nnz-1); reported through perm_out.
 *   keys_out  nnz uint64: the new keys, strictly increasing.
 *   vals_out  nnz fp64 or NULL (must be NULL iff vals_in is NULL): vals_out[i] is a bit
 *             copy of vals_in[p(i)].
 *   perm_out  nnz uint32 or NULL: perm_out[i] = idx_in ? idx_in[p(i)] : p(i), the gather
 *             map of the result.
 *   workspace device scratch of lco_workspace_size() bytes, 256-byte aligned.
 * Output ranges must not overlap the inputs or each other.  nnz == 0 returns LCO_OK
 * without launching anything.  Ties (duplicate keys, a precondition violation) keep
 * input order (stable). */
LCO_API lco_status lco_permute(lco_handle h, uint64_t nnz, const uint64_t* keys_in,
                       const double* vals_in, const uint32_t* idx_in, uint64_t* keys_out,
                       double* vals_out, uint32_t* perm_out, void* workspace,
                       size_t workspace_bytes, void* stream);

/* Sort an LCO tensor given in ANY order into the lexicographical order selected by the
 * handle's perm ("sorting is typically required when non-zero data is
 * unsorted"): stable radix sort of the re-encoded keys over all key digits.  Same
 * arguments and semantics as lco_permute except that keys_in need not be sorted (keys
 * must still be < prod(dims)); equal keys keep input order. */
LCO_API lco_status lco_sort(lco_handle h, uint64_t nnz, const uint64_t* keys_in, const double* vals_in,
                    const uint32_t* idx_in, uint64_t* keys_out, double* vals_out,
                    uint32_t* perm_out, void* workspace, size_t workspace_bytes, void* stream);

/* Same as lco_permute but every array is in HOST memory (pinned for full speed); the
 * call copies the inputs into the device workspace, permutes, and copies the results
 * back, all stream-ordered (the caller synchronizes the stream before reading outputs).
 * Workspace: lco_host_workspace_size() bytes of device memory. */
LCO_API lco_status lco_host_workspace_size(lco_handle h, uint64_t nnz, size_t* bytes);
LCO_API lco_status lco_permute_host(lco_handle h, uint64_t nnz, const uint64_t* keys_in,
                            const double* vals_in, uint64_t* keys_out, double* vals_out,
                            uint32_t* perm_out, void* workspace, size_t workspace_bytes,
                            void* stream);

/* Stable multisplit for the sharded path: route every nonzero of a
 * sorted input slice to the rank owning its NEW key range.
 *   splitters  world-1 ascending uint64 new-key bounds (device); rank r receives the
 *              keys K' with splitters[r-1] <= K' < splitters[r].
 *   idx_base   global index of keys_in[0]; send_idx carries idx_base + i.
 *   send_keys/send_vals/send_idx  nnz records grouped by destination rank, each group in
 *              input order; send_keys carries the OLD key (the receiver re-runs
 *              lco_permute with idx_in = received send_idx).
 *   send_counts world uint64 (device): records per destination.
 * world in 1..2048 (one 11-bit multisplit pass; larger values return LCO_ERR_ARG).  vals may be NULL (both). */
LCO_API lco_status lco_partition(lco_handle h, uint64_t nnz, const uint64_t* keys_in,
                         const double* vals_in, uint32_t idx_base, int world,
                         const uint64_t* splitters, uint64_t* send_keys, double* send_vals,
                         uint32_t* send_idx, uint64_t* send_counts, void* workspace,
                         size_t workspace_bytes, void* stream);

/* The exchange fused into the partition ("the partition scatter IS the
 * exchange"): the same stable multisplit as lco_partition, but every record is stored
 * straight into its destination rank's receive buffer, at recv_*[d][recv_offsets[d] + w]
 * (w = its index among this rank's records for d).  recv_keys / recv_vals / recv_idx
 * are [host] arrays of `world` DEVICE pointers: peer-mapped buffers of the other GPUs
 * (CUDA IPC / symmetric memory over NVLink), or plain local buffers.  recv_offsets
 * [host]: where this rank's chunk starts in each receiver = the sum of the counts of the
 * lower source ranks for that destination (from lco_partition_counts + an all-gather),
 * so receivers see the chunks in source-rank order = global input order.  send_counts
 * (device) as in lco_partition.  world in 1..16; the caller synchronizes the ranks
 * before the receivers read.  Same workspace as lco_partition. */
LCO_API lco_status lco_partition_direct(lco_handle h, uint64_t nnz, const uint64_t* keys_in,
                                const double* vals_in, uint32_t idx_base, int world,
                                const uint64_t* splitters, uint64_t* const* recv_keys,
                                double* const* recv_vals, uint32_t* const* recv_idx,
                                const uint64_t* recv_offsets, uint64_t* send_counts,
                                void* workspace, size_t workspace_bytes, void* stream);

/* Only the per-destination record counts of the partition (device send_counts[world]):
 * the count and scan of the multisplit pass, no data movement.  world in 1..2048 (one 11-bit multisplit pass; larger values return LCO_ERR_ARG). */
LCO_API lco_status lco_partition_counts(lco_handle h, uint64_t nnz, const uint64_t* keys_in,
                                int world, const uint64_t* splitters, uint64_t* send_counts,
                                void* workspace, size_t workspace_bytes, void* stream);

/* Histogram of the top `bits` bits of the re-encoded keys (new-key order), used to
 * choose balanced splitters: counts[b] += #{i : (K'_i >> (keybits - bits)) == b} where
 * keybits = ceil(log2(prod dims)).  counts: 2^bits uint64 on the device, ACCUMULATED
 * (zero it first).  bits in 1..16. */
LCO_API lco_status lco_key_histogram(lco_handle h, uint64_t nnz, const uint64_t* keys_in, int bits,
                             uint64_t* counts, void* stream);

/* Host-side plan introspection (no CUDA calls).  Reports the plan lco_permute (sort=0)
 * or lco_sort (sort=1) uses for nnz nonzeros. */
typedef struct lco_plan_info {
  int order;                           /* as created */
  int32_t rearrangement[LCO_MAX_ORDER];/* by NEW position t: 1 if perm[t] is a
                                          rearrangement index, 0 if resting */
  int norm_order;                      /* modes after dropping size-1 and fusing */
  uint64_t norm_dims[LCO_MAX_ORDER];   /* normalized dims, old order */
  int32_t norm_perm[LCO_MAX_ORDER];    /* normalized perm */
  int prefix_len;                      /* identity prefix length a (normalized) */
  int suffix_start;                    /* start b of the longest increasing suffix */
  uint64_t segment_divisor;            /* D = prod_{m>=a} n_m: segment id = K div D */
  uint64_t trailing;                   /* T = prod_{t>=b} n'_t: sort key q = K' div T */
  uint64_t middle_size;                /* S = prod_{a<=t<b} n'_t */
  uint64_t num_segments;               /* G = prod_{m<a} n_m */
  int sort_bits;                       /* bits of q the passes sort on */
  int passes;                          /* radix passes over HBM (0 = copy) */
  int digit_bits[8];                   /* bits per pass, least significant first */
  int radix_bits;                      /* bins per pass = 2^radix_bits */
  int path;                            /* 0 copy, 1 LSD passes, 2 one on-chip leaf,
                                          3 MSD passes + on-chip leaf sorts, 4 segment-
                                          local tiles, 5 segmented single pass,
                                          6 hierarchical stages, 7 block transpose */
  int launches;                        /* kernels this library launches per call */
  int tile;                            /* nonzeros per tile (CTA) */
  int msd_levels;                      /* path 3: MSD passes before the leaves */
  int leaf_bits;                       /* paths 2/3: bits of q the leaf sorts handle */
  int leaf_kind;                       /* paths 2/3: 1 one warp per leaf (<= 384 nonzeros),
                                          2 one CTA per leaf (<= 8192 nonzeros), 3 one
                                          cluster of 16 CTAs per leaf (<= 65536, DSMEM) */
  double model_bytes;                  /* modelled HBM bytes per nonzero of the plan */
  int stages;                          /* permute: stages of the hierarchical plan (one per
                                          maximal run of rearrangement indices, PAPER.md:
                                          245-247); 1 = flat.  path 6: the stages run */
  int stage_path[8];                   /* path of each stage (0-5 as above) */
  int stage_sort_bits[8];              /* bits of q each stage sorts */
  double flat_model_bytes;             /* modelled bytes of the flat plan */
  uint64_t block_grid[5];              /* path 7: blocks (runs of constant old modes 0..k),
                                          dims of the old-innermost block mode A and of the
                                          new-innermost block mode B, products of the block
                                          modes between B and A and before B; else 0 */
} lco_plan_info;
LCO_API lco_status lco_plan_query(lco_handle h, uint64_t nnz, int sort, lco_plan_info* info);

/* Stage j of the hierarchical plan (host only): the stage permutes keys of `dims` (its
 * input order, normalized modes: size-1 modes dropped, modes that stay adjacent fused,
 * so keys are unchanged) by the relative permutation `perm`.  Composing the stages in
 * order gives the handle's permutation.  *n_stages = number of stages (1: flat plan,
 * stage 0 = the normalized permutation).  dims/perm [host] of LCO_MAX_ORDER entries;
 * LCO_ERR_ARG if j is out of range. */
LCO_API lco_status lco_plan_stage(lco_handle h, int j, int* n_stages, int* order, uint64_t* dims,
                                  int32_t* perm);

/* Host reference of the device fast divisor (test hook for the host plan): writes
 * q[i] = x[i] / d computed with the same magic-number arithmetic the kernels use.
 * d >= 1; x, q [host]. */
LCO_API lco_status lco_fastdiv_host(uint64_t d, uint64_t n, const uint64_t* x, uint64_t* q);

/* Kernel timing hook for measurement (bench.py): after lco_profile_enable(h, calls), the
 * next `calls` device calls on h record a CUDA event before every launch and after the
 * last one.  After synchronizing, lco_profile_read returns, per call c and stage s,
 * ms[c*max_stages + s] (stage durations) and the stage names (separated by ';' in
 * names, capacity names_len).  Host-only bookkeeping; does not change results. */
LCO_API lco_status lco_profile_enable(lco_handle h, int calls);
LCO_API lco_status lco_profile_read(lco_handle h, int max_calls, int max_stages, float* ms,
                            int* n_calls, int* n_stages, char* names, size_t names_len);

/* Index-matched addition C = A + sign * permute(B, match) (§3.2, the
 * sum of c^(y) and c^(x) in Eq (2.3) after re-sorting one term into the {1,0,3,2} order;
 * SURVEY.md §8(f) NEXT 3).  h is the plan of B: B's dims and the match permutation, so
 * that permute(B, match) is in A's mode order (A's dims = B's dims permuted).
 *   keys_a/vals_a  nnz_a nonzeros of A, keys strictly increasing (row-major, A's order).
 *   keys_b/vals_b  nnz_b nonzeros of B, keys strictly increasing in B's own order.
 *   sign           scales B's values (+1 or -1 in the paper; any finite double).
 *   keys_c/vals_c  capacity nnz_a + nnz_b; receive the union of the supports, ascending;
 *                  colliding keys hold a + sign*b (one IEEE addition), explicit zeros kept.
 *   nnz_c          [device] one uint64: the number of outputs written.
 * Workspace: lco_add_workspace_size bytes, 256-byte aligned.  Stream-ordered, no sync.
 * Errors: LCO_ERR_NULL / LCO_ERR_CAPACITY (nnz_b > max_nnz) / LCO_ERR_WORKSPACE /
 * LCO_ERR_ALIAS (outputs overlap inputs or workspace) / LCO_ERR_CUDA. */
LCO_API lco_status lco_add_workspace_size(lco_handle h, uint64_t nnz_a, uint64_t nnz_b,
                                          size_t* bytes);
LCO_API lco_status lco_add(lco_handle h, uint64_t nnz_a, const uint64_t* keys_a,
                           const double* vals_a, uint64_t nnz_b, const uint64_t* keys_b,
                           const double* vals_b, double sign, uint64_t* keys_c, double* vals_c,
                           uint64_t* nnz_c, void* workspace, size_t workspace_bytes, void* stream);

/* ---- Matrix datatypes of a flattened tensor (§5.2 steps 1-2, :325-331;
 * SURVEY.md §8(f) NEXT 4).  Flattening a tensor into an m x n matrix is a permutation
 * (rows modes first, then column modes; lco_permute) -- a row-major LCO matrix has key
 * row * n + col, a column-major one col * m + row.  Compression never sorts. */

/* Compress a major-first LCO matrix: keys strictly increasing, key = major * n_minor +
 * minor (CSR/DCSR from a row-major matrix: major = row; CSC/DCSC from a column-major
 * one: major = column).  The values array of the LCO matrix is the MDT's value array.
 *   doubly = 0 (CSR/CSC): ptr [n_major + 1] with ptr[r] = first nonzero of major >= r.
 *   doubly = 1 (DCSR/DCSC, Buluc & Gilbert): ids [capacity nnz] receives
 *            the non-empty majors ascending, ptr [capacity nnz + 1] their starts and
 *            ptr[nz] = nnz, *n_nonempty [device] = nz; nothing is O(n_major).
 *   minor    [nnz] receives key mod n_minor.
 * Workspace: lco_compress_workspace_size (0 for doubly = 0).  Stream-ordered. */
LCO_API lco_status lco_compress_workspace_size(uint64_t nnz, int doubly, size_t* bytes);
LCO_API lco_status lco_compress(uint64_t nnz, const uint64_t* keys, uint64_t n_major,
                                uint64_t n_minor, int doubly, uint64_t* ptr, uint64_t* ids,
                                uint64_t* minor, uint64_t* n_nonempty, void* workspace,
                                size_t workspace_bytes, void* stream);

/* Hyper-sparsity of an m x n matrix with nnz nonzeros ("the ratio of NNZ to
 * the dimension in question"; LibNT switches algorithms at ratio 3, :483): 0 sparse,
 * 1 row-sparse (m / nnz > threshold, very tall), 2 column-sparse (n / nnz > threshold,
 * very wide), 3 index-sparse (both).  nnz = 0 -> 0.  Host only. */
LCO_API int lco_sparsity_class(uint64_t m, uint64_t n, uint64_t nnz, double threshold);

/* The MDT / algorithm of the multiplication poly-algorithm for C = A B given the classes
 * of A and B (PAPER.md Table "Multiplication possibilities", :340-352): returns a code
 * whose name lco_mdt_name gives ("CSC/CSR", "CSC", "CSR", "DCSC/DCSR", "DCSC", "DCSR",
 * "CSCNA/CSRNA", "CSCNA", "CSRNA", "SOP"); -1 for invalid classes.  Host only. */
LCO_API int lco_mdt_choice(int class_a, int class_b);
LCO_API const char* lco_mdt_name(int code);

LCO_API const char* lco_status_string(lco_status s);
LCO_API const char* lco_last_error(void);
LCO_API const char* lco_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LCO_H */
