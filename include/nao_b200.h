/*
 * nao_b200.h -- C ABI of the B200-native NAO hot path (arXiv 2510.16028).
 *
 * libnao_b200.so (sm_100a) replaces the numpy inner loops of the reference
 * package /root/reference/pkg/src/fpverify behind its own Python API
 * (bounds.op_bound / co_execute, calibration.percentile_profile,
 * dispute.observed_p_max / leaf check, commitments.build_tree / canon_tensor).
 * Each entry point below names the reference function it replaces.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Tensor pointers are DEVICE pointers
 *     owned by the caller; small descriptor arrays (shapes, grids, headers,
 *     thresholds) are HOST pointers read during the call.
 *   - Every call is asynchronous on `stream` (a cudaStream_t passed as void*);
 *     none synchronizes the host.  Scratch comes from a caller workspace
 *     sized by the matching *_workspace() query.
 *   - Return 0 (NAO_OK) or a status; nao_last_error() gives the message
 *     (thread-local).  The Python layer maps NAO_EINVAL to ValueError as the
 *     reference raises (bounds.py:57-58, :108-109; calibration.py:28-29;
 *     commitments.py:116-117).
 *   - No global mutable state; reentrant across streams.
 */
#ifndef NAO_B200_H
#define NAO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum nao_status { NAO_OK = 0, NAO_EINVAL = 1, NAO_ECUDA = 2, NAO_ENONFINITE = 3 };

enum nao_hash_alg { NAO_HASH_SHA256 = 0, NAO_HASH_KECCAK256 = 1 };

/* how nao_check obtains the per-element bound */
enum nao_eps_kind {
    NAO_EPS_TENSOR_F32 = 0,   /* eps array, FP32 rounded up            */
    NAO_EPS_TENSOR_F64 = 1,   /* eps array, FP64 (reference dtype)     */
    NAO_EPS_SCALED_LOCAL = 2, /* eps = scale * |local| (u|y|, 2u|y|)   */
    NAO_EPS_ZERO = 3          /* data movement / relu / max / min      */
};

enum nao_reduce_kind { NAO_RED_SUM = 0, NAO_RED_MEAN = 1, NAO_RED_MAX = 2, NAO_RED_MIN = 3 };
enum nao_unary_kind {
    NAO_UN_EXP = 0, NAO_UN_LOG = 1, NAO_UN_SQRT = 2, NAO_UN_RSQRT = 3,
    NAO_UN_TANH = 4, NAO_UN_GELU = 5, NAO_UN_SILU = 6
};
/* device-profile reduction orders (engine.py:75-113) */
enum nao_order {
    NAO_ORDER_SEQUENTIAL = 0, NAO_ORDER_PAIRWISE = 1, NAO_ORDER_BLOCKED = 2, NAO_ORDER_PERMUTED = 3
};
/* A DeviceProfile (engine.py:29-55) for the FP32 value path: the order of
 * every reduction (matmul inner products, softmax / layernorm / sum / mean
 * folds) and the fma policy of matmul.  perm: device int64[perm_n], the
 * numpy Philox permutation of the reduced length (engine.py:75-77), for
 * NAO_ORDER_PERMUTED.  A NULL profile means sequential, no fma. */
typedef struct nao_profile {
    int32_t order;
    int32_t block_size;
    const int64_t* perm;
    int64_t perm_n;
    int32_t fma;
    int32_t reserved;
} nao_profile;
/* abs-GEMM bound paths: FFMA round-up chains, tcgen05 3-split (TF32 / FP16),
 * and FP64 (the reference's own arithmetic; the API default, eps within
 * ~1e-12 of numpy's -- the streaming verifier uses the tensor-core paths) */
enum nao_gemm_path { NAO_GEMM_FFMA_RU = 0, NAO_GEMM_TC_TF32X3 = 1, NAO_GEMM_TC_F16X3 = 2,
                     NAO_GEMM_FP64 = 3 };

/* ------------------------------------------------------------ library */
int nao_version(void);
/* copies the calling thread's last error message; returns its length */
int nao_last_error(char* buf, size_t buf_len);
/* number of SMs / compute capability of the current device (sanity) */
int nao_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ------------------------------------------------------------- commit */
/* Replaces commitments.build_tree(leaves).root over the chunked leaves of
 * every traced tensor (commitments.py:39-61 canon bytes, :112-142 tree):
 *   leaves(t) = [canon_header(t)] + payload split into chunk_bytes pieces.
 * n_tensors roots (32 B each) are written to roots_out (device).  If
 * leaf_digests_out != NULL the level-0 digests are written there
 * (sum_i (1 + ceil(bytes_i/chunk)) * 32 bytes) and the workspace may omit them.
 * payloads: 16-byte aligned device pointers, byte sizes multiple of 4.
 * headers: host pointers (<= 136 bytes each). */
size_t nao_merkle_commit_workspace(int64_t n_tensors, const uint64_t* payload_bytes,
                                   uint64_t chunk_bytes);
int nao_merkle_commit_tensors(int64_t n_tensors, const void* const* payloads,
                              const uint64_t* payload_bytes, const uint8_t* const* headers,
                              const uint32_t* header_lens, uint64_t chunk_bytes, int hash_alg,
                              uint8_t* roots_out, uint8_t* leaf_digests_out, void* workspace,
                              size_t workspace_bytes, void* stream);
/* leaf_digest(x) = H(0x00 || x) for n byte strings packed in device memory;
 * offsets: device int64[n+1] (commitments.py:137-138). */
int nao_merkle_hash_leaves(const uint8_t* data, const int64_t* offsets, int64_t n_leaves,
                           int hash_alg, uint8_t* digests_out, void* stream);
/* MerkleTree(leaf_digests).root (commitments.py:112-134).  levels_out (device,
 * optional) receives every level concatenated, leaves first (MerkleTree.levels). */
size_t nao_merkle_root_workspace(int64_t n_leaves);
int nao_merkle_root_of(const uint8_t* leaf_digests, int64_t n_leaves, int hash_alg,
                       uint8_t* root_out, uint8_t* levels_out, void* workspace,
                       size_t workspace_bytes, void* stream);

/* -------------------------------------------------------------- check */
typedef struct nao_check_result {
    uint64_t n;
    uint64_t n_violations;   /* #{|claimed-local| > eps}   dispute.py:641-648 */
    uint64_t n_borderline;   /* eps*lo_factor < diff <= eps (verdict-sensitive band) */
    uint64_t n_nonfinite;
    double max_ratio;        /* max diff/eps (inf if diff>0 where eps==0) */
    int32_t threshold_exceeded; /* observed_p_max(...) > 1.0  dispute.py:130-150 */
    int32_t first_exceeded;     /* grid index (abs: i, rel: G+i) or -1 */
    int32_t n_ambiguous;        /* targets settled by the exact second pass */
    int32_t reserved;
} nao_check_result;

/* One pass over (local, claimed[, eps]) per operator: bound violations and
 * the exact p_max > 1 verdict of observed_p_max against (tau_abs, tau_rel) on
 * the percentile grid (calibration.py:16, dispute.py:114-141).  grid/tau are
 * host arrays of n_grid (<= 32) doubles; result is a device pointer.  Single
 * launch: the last CTA finalizes.  The workspace (nao_check_workspace() bytes)
 * is a dedicated accumulator that must be zero before its first use; every
 * call leaves it zeroed again (do not share it with other entry points). */
size_t nao_check_workspace(void);
/* Borderline list (optional, device): uint64 [1 + border_cap]; word 0 counts
 * the borderline elements, words 1.. hold the flat indices of the first
 * border_cap of them (nao_refine_borderline settles them exactly and resets
 * the count).  NULL: borderline elements are only counted. */
int nao_check(const float* local, const float* claimed, int64_t n, int eps_kind, const void* eps,
              double eps_scale, double lo_factor, const double* grid, const double* tau_abs,
              const double* tau_rel, int n_grid, double epsilon, nao_check_result* result,
              void* workspace, size_t workspace_bytes, uint64_t* border_list,
              int64_t border_cap, void* stream);
/* Per-node verdict spec: grid + thresholds prepared once on the host
 * (ThresholdSet.lookup(name), calibration.py:117-191) and kept in device
 * memory; nao_verdict_spec_bytes() bytes, filled by nao_verdict_spec_fill
 * into a HOST buffer the caller then copies to the device. */
size_t nao_verdict_spec_bytes(void);
int nao_verdict_spec_fill(void* spec_host, const double* grid, const double* tau_abs,
                          const double* tau_rel, int n_grid, double epsilon);
/* The check of one claimed tensor, fused into its Merkle commitment
 * (nao_commit_check_tensors).  local/eps/spec/result are device pointers;
 * local == NULL disables the check for that tensor. */
typedef struct nao_check_desc {
    const float* local;          /* recomputed node output, 16-byte aligned */
    const void* eps;             /* eps array for NAO_EPS_TENSOR_* (else NULL) */
    const void* spec;            /* device nao_verdict_spec of the node */
    nao_check_result* result;    /* device record, written by the last CTA */
    double eps_scale;            /* NAO_EPS_SCALED_LOCAL */
    double lo_factor;            /* borderline band (see nao_check) */
    int32_t eps_kind;
    int32_t flags;               /* NAO_CHECK_PARTIAL: `result` is a nao_check_partial */
    uint64_t* border_list;       /* optional borderline list (see nao_check) */
    int64_t border_cap;
} nao_check_desc;
/* A shard's combinable check state (batch-sharded verification):
 * counts per threshold interval (bucket b = keys with b sorted thresholds
 * strictly below them; b = G holds non-finite elements) and the smallest /
 * largest FP64 key per bucket, so the exact p_max > 1 verdict of the whole
 * tensor -- including numpy's interpolation between order statistics -- is
 * decided from the shards' partials alone (paper_2510_16028_b200.dispute.
 * combine_partials).  Empty buckets: min = +inf, max = 0. */
enum { NAO_CHECK_PARTIAL = 1 };
typedef struct nao_check_partial {
    uint64_t n, n_violations, n_borderline, n_nonfinite;
    double max_ratio;
    uint64_t hist_abs[33], hist_rel[33];
    double min_abs[33], max_abs[33], min_rel[33], max_rel[33];
} nao_check_partial;
/* nao_merkle_commit_tensors + nao_check of every tensor in the SAME pass:
 * payloads are the claimed tensors; checks[i] (host array, n_tensors entries)
 * compares payload i with checks[i].local (the reference's leaf route,
 * dispute.py:639-671, one record per tensor; empty tensors get none).
 * accum: device scratch of nao_commit_check_accum_bytes(), zero before its
 * first use and left zeroed by every call (dedicated per stream).
 * Workspace as nao_merkle_commit_workspace. */
/* Chunk-digest reuse (optional, host array of n_tensors entries or NULL): a
 * tensor whose LOCAL recomputation is a data-movement copy of another claimed
 * tensor of the same call (reshape: the same bytes; concat of one tensor with
 * itself: blocks repeated) has chunk c equal, when its claimed chunk equals
 * its local chunk word for word, to source chunk
 *   (c / (block_chunks * repeats)) * block_chunks + c % block_chunks,
 * so its digest is copied instead of re-hashed (leaf = H(0x00 || chunk) is a
 * function of the bytes only; the header leaf and the tree are still built).
 * Chunks that differ are hashed.  src = -1: no reuse.  Needs the fused check
 * (checks[i].local).  Sources are processed in an earlier launch. */
/* mode NAO_REUSE_SAME_OFFSET: an elementwise node whose claimed chunk c is
 * byte-identical to the source's claimed chunk c (e.g. the lower triangle of
 * a causal-mask add, x + 0 = x) copies that digest; the equality is verified
 * word by word on the claimed bytes (block_chunks / repeats unused; same
 * payload size as the source).  Independently of src, every full chunk of a
 * checked tensor whose claimed words are all zero (e.g. the masked half of
 * causal softmax rows) takes the digest of the all-zero chunk (Keccak-256).
 * row_chunks (0 = none): chunks per row of the tensor's last axis, a divisor
 * of 128 -- threads of a commit CTA take chunk j of consecutive rows, so
 * warps meet the same kind of chunk and a warp whose chunks all take a
 * shortcut leaves the sponge pipe to the other warps. */
/* ref_payload / ref_digests / ref_bytes (optional, ref_payload = NULL: none):
 * a static tensor broadcast over the leading dims (ref_bytes a multiple of
 * chunk_bytes dividing the payload size) with its chunk digests (ref_digests:
 * ref_bytes / chunk_bytes digests of 32 bytes, e.g. the leaf digests of its
 * own commit after the header leaf); a claimed chunk c equal to reference
 * chunk c mod (ref_bytes / chunk_bytes) takes that digest (the -1e9 fill of
 * a causal mask add: x + w rounds to w). */
enum nao_reuse_mode { NAO_REUSE_LOCAL_COPY = 0, NAO_REUSE_SAME_OFFSET = 1 };
typedef struct nao_chunk_reuse {
    int64_t src;
    uint64_t block_chunks;
    uint64_t repeats;
    int32_t mode;
    uint32_t row_chunks;
    const void* ref_payload;
    const void* ref_digests;
    uint64_t ref_bytes;
} nao_chunk_reuse;
size_t nao_commit_check_accum_bytes(void);
/* Chunks of nao_commit_check_tensors calls (all streams, since the last reset)
 * whose digest was copied instead of hashed (chunk-digest reuse and digest
 * shortcuts): *out = the device counter; reset != 0 zeroes it.  Synchronises
 * the device (a measurement hook, not for the hot path). */
int nao_commit_stats(uint64_t* reused_chunks, int reset);
int nao_commit_check_tensors(int64_t n_tensors, const void* const* payloads,
                             const uint64_t* payload_bytes, const uint8_t* const* headers,
                             const uint32_t* header_lens, uint64_t chunk_bytes, int hash_alg,
                             const nao_check_desc* checks, const nao_chunk_reuse* reuse,
                             uint8_t* roots_out, void* accum, void* workspace,
                             size_t workspace_bytes, void* stream);
/* Exact numpy method="linear" percentile profiles (calibration.py:33-37):
 * of |local-claimed| and |local-claimed|/(|local|+epsilon) (calibration.py:40-49),
 * or of an arbitrary FP64 array.  Outputs are device arrays of n_grid doubles. */
size_t nao_percentile_workspace(int64_t n);
int nao_error_profiles(const float* local, const float* claimed, int64_t n, double epsilon,
                       const double* grid, int n_grid, double* abs_prof, double* rel_prof,
                       void* workspace, size_t workspace_bytes, void* stream);
int nao_percentile_profile(const double* values, int64_t n, const double* grid, int n_grid,
                           double* out, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------- bounds */
/* All bounds: eps = template(...) * (1 + slack); eps_f64 selects FP64 output
 * (reference dtype) or FP32 rounded toward +inf.  Rows are contiguous
 * [rows, n] with the reduced axis last (the host moves it).  u = unit
 * roundoff, rc = FpModel.reduction_const(n-1) (bounds.py:42-45). */
/* softmax_bound_parts, bounds.py:114-135 (values: engine.py:185-194, sequential) */
int nao_softmax_bound(const float* x, float* y, void* eps, int eps_f64, int64_t rows, int64_t n,
                      double u, double rc, double slack, const nao_profile* profile,
                      void* stream);
/* layernorm_bound_parts, bounds.py:143-169 (values: engine.py:197-213) */
int nao_layernorm_bound(const float* x, float* y, void* eps, int eps_f64, int64_t rows, int64_t n,
                        float ln_eps, double u, double rc, double slack,
                        const nao_profile* profile, void* stream);
/* op_bound sum/mean/max/min, bounds.py:194-208 (values: engine.py:240-251) */
int nao_reduce_bound(const float* x, float* y, void* eps, int eps_f64, int64_t rows, int64_t n,
                     int kind, double u, double rc, double slack, const nao_profile* profile,
                     void* stream);
/* _unary_intrinsic values, engine.py:133-154 (FP64 evaluation, one rounding).
 * The reference's FP64 libm (numpy SIMD exp/log/tanh/pow) is not correctly
 * rounded and differs across CPUs, so each element also gets the range of
 * FP32 results any evaluation within the libm error envelope can produce
 * (exp/log/tanh: 16 FP64 ulps; gelu: its x**3, tanh and the cancellation in
 * 1+tanh propagated).  y = the value of this evaluation; elements whose range
 * holds more than one FP32 value are "value-ambiguous": their flat indices go
 * to amb_list (same layout as the check's borderline list, may be NULL).
 * eps (optional): the intrinsic template eps_scale*|y| (bounds.py:198-199)
 * taken at the largest |candidate|, so eps >= the reference's on every element. */
int nao_unary_fp64(const float* x, float* y, int64_t n, int kind, void* eps, int eps_f64,
                   double eps_scale, uint64_t* amb_list, int64_t amb_cap, void* stream);
/* eps = scale*|y|: single-rounding (u) / intrinsic (2u) templates, bounds.py:196-199 */
int nao_scaled_abs_bound(const float* y, void* eps, int eps_f64, int64_t n, double scale,
                         void* stream);
/* matmul_bound, bounds.py:100-111 (+ linear's u|y|, bounds.py:214-217):
 *   eps[b,m,n] = gamma_const * sum_k |A[b,m,k]||B[b,k,n]| * (1+slack) [+ u|y|]
 * B is [K,N] (ldb) or, with transpose_b, [N,K].  Batch strides may be 0. */
int nao_abs_gemm_bound(const float* A, const float* B, void* eps, int eps_f64, int64_t batch,
                       int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
                       int64_t stride_a, int64_t stride_b, int64_t stride_c, int transpose_b,
                       double gamma_const, const float* y_or_null, double u, double slack,
                       int path, void* stream);
/* tcgen05 path of matmul_bound: |x| -> TF32 (hi, lo) parts, K-major
 * [batch, rows, Kp] with Kp = nao_tf32_split_cols(K) (x is [rows, K] row-major
 * with leading dim ld, or [K, rows] when transpose).  hi <= |x| <= hi + lo. */
int64_t nao_tf32_split_cols(int64_t K);
int nao_tf32_split(const float* x, float* hi, float* lo, int64_t batch, int64_t rows, int64_t K,
                   int64_t ld, int64_t stride_batch, int transpose, void* stream);
/* eps >= gamma_const * sum_k |A||B| from the split parts on tcgen05.mma.kind::tf32
 * (3 products, outward-compensated, within rtol 1e-5 of the FP64 reference);
 * batch_a / batch_b are `batch` or 1 (broadcast).  Output [batch, M, N], ldc. */
/* k-length of one tensor-core accumulation chunk of nao_abs_gemm_tc (its error
 * model: relative loss <= (kchunk/8) * 3 * 2^-23 per chunk, csrc/absgemm_tc.cu). */
int nao_abs_gemm_tc_kchunk(void);
int nao_abs_gemm_tc(const float* a_hi, const float* a_lo, const float* b_hi, const float* b_lo,
                    void* eps, int eps_f64, int64_t batch, int64_t batch_a, int64_t batch_b,
                    int64_t M, int64_t N, int64_t K, int64_t ldc, int64_t stride_c,
                    double gamma_const, const float* y_or_null, double u, double slack,
                    void* stream);
/* FP16 3-split of matmul_bound on tcgen05.mma.kind::f16 (2x the TF32 rate,
 * half the operand bytes).  nao_f16_split: |x| -> K-major FP16 parts
 * [batch, rows, Kp] (Kp = nao_f16_split_cols(K)) and row_info int32[2*batch*rows]:
 * row exponents e then counts of "tiny" elements, with |x| <= 2^e (hi + 2^-10 lo),
 * relative excess <= 2^-20 for |x| >= 2^(e-14) and absolute excess < 2^(e-24)
 * below (tiny; exact power-of-two scaling puts the row max in [2^14, 2^15)).
 * nao_abs_gemm_tc16 = nao_abs_gemm_tc on those parts; outputs whose tiny-part
 * excess could exceed 2^-20 of their value are recomputed exactly in FP64 from
 * the original operands A [batch_a, M, K] / B ([batch_b, K, N], or [batch_b, N, K]
 * with transpose_b), so the result stays within rtol 1e-5 of the FP64 bound.
 * fix_ws: zeroed device scratch of nao_abs_gemm_tc16_fix_workspace() bytes per
 * stream, left zeroed by every call. */
int64_t nao_f16_split_cols(int64_t K);
int nao_f16_split(const float* x, void* hi, void* lo, int32_t* row_info, int64_t batch,
                  int64_t rows, int64_t K, int64_t ld, int64_t stride_batch, int transpose,
                  void* stream);
size_t nao_abs_gemm_tc16_fix_workspace(void);
int nao_abs_gemm_tc16(const void* a_hi, const void* a_lo, const int32_t* a_info, const void* b_hi,
                      const void* b_lo, const int32_t* b_info, const float* A, const float* B,
                      int transpose_b, void* eps, int eps_f64, int64_t batch, int64_t batch_a,
                      int64_t batch_b, int64_t M, int64_t N, int64_t K, int64_t ldc,
                      int64_t stride_c, double gamma_const, const float* y_or_null, double u,
                      double slack, void* fix_ws, size_t fix_ws_bytes, void* stream);
/* matmul_op values (engine.py:157-182) under `profile` (NULL: sequential):
 * FP32 products reduced over K in the profile's order, or with profile->fma
 * the sequential FP64-step loop.  C contiguous [batch, M, N]. */
int nao_matmul_profile(const float* A, const float* B, float* C, int64_t batch, int64_t M,
                       int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t stride_a,
                       int64_t stride_b, int64_t stride_c, int transpose_b,
                       const nao_profile* profile, void* stream);

/* conv2d lowering (SURVEY.md 2.3 extension): patch rows of an NCHW FP32 input,
 * col[b, oh*OW + ow, (c*k + kh)*k + kw] (torch unfold's K order, zero padding
 * included in K), row-major [batch, OH*OW, C*k*k].  OH = (H + 2 pad - k)/stride + 1. */
int nao_im2col_rows(const float* x, float* col, int64_t batch, int64_t C, int64_t H, int64_t W,
                    int64_t k, int64_t stride, int64_t pad, void* stream);

/* ---------------------------------------------- exact re-adjudication */
/* Settles the borderline elements a check recorded (nao_check /
 * nao_check_desc border_list) against the reference's own bound: the
 * streaming bounds over-estimate the reference's by a certified factor R
 * (DESIGN.md 5), so an element with eps/R < diff <= eps is undecided until
 * the reference's eps is recomputed for it.  GEMM / conv: the abs-dot
 * sum_k |a||b| exactly (FP64 products, double-double sum), then the
 * reference's interval eps_ref in const*S*(1 +- (K+4) 2^-53) [+ u|y|] --
 * numpy's BLAS order is unknown, nothing narrower is reproducible.  UNARY:
 * value-ambiguous elements (nao_unary_fp64) -- the verdict
 * |c - y| > scale|y| is evaluated over every candidate y.  Each settled
 * element leaves n_borderline; a certain violation is added to n_violations;
 * a verdict that differs between candidates is moved out of n_violations
 * into n_borderline.  After the pass n_violations counts certain reference
 * violations and n_borderline the undecided rest.  The list count is reset
 * to 0 (graph replay).  One launch for up to 64 descriptors (host array). */
enum nao_refine_kind { NAO_REFINE_GEMM = 0, NAO_REFINE_CONV = 1, NAO_REFINE_UNARY = 2 };
typedef struct nao_refine_desc {
    int32_t kind;               /* NAO_REFINE_* */
    int32_t unary_kind;         /* NAO_UN_* (UNARY) */
    uint64_t* list;             /* border / ambiguity list of the node */
    int64_t cap;
    nao_check_result* result;   /* the node's check record */
    const float* local;         /* recomputed output y */
    const double* local64;      /* GEMM / CONV: FP64 y instead (the leaf route's FP64 oracle
                                   recheck, dispute.py:648-656), else NULL */
    const float* claimed;       /* claimed output y' */
    const float* a;             /* GEMM: A [batch_a, M, K]; CONV: W [N=Cout, C, k, k]; UNARY: x */
    const float* b;             /* GEMM: B [batch_b, K, N] / [batch_b, N, K]; CONV: x [batch, C, H, W] */
    int64_t batch, M, N, K;     /* GEMM output [batch, M, N]; CONV: batch, M=OH*OW, N=Cout, K=C k k */
    int64_t stride_a, stride_b; /* batch strides (0 = broadcast) */
    int32_t transpose_b, has_y; /* has_y: linear's + u|y| */
    int64_t C, H, W, k, stride, pad, OW; /* CONV geometry */
    double gamma_const, u;      /* reduction_const(count); u (linear) / eps_scale (UNARY) */
} nao_refine_desc;
int nao_refine_borderline(const nao_refine_desc* descs, int n_descs, void* stream);

/* ------------------------------------------- FP64 theoretical oracle path */
/* The reference's FP64 execution of one operator (apply_op(fp64=True),
 * engine.py:220-285 via execute_fp64 :369-390; the leaf route's theoretical
 * recheck, dispute.py:648-656): FP32 inputs promoted to FP64, every
 * reduction a sequential FP64 fold (reduce_last_axis(profile=None),
 * engine.py:95-113), so results are bit-identical to numpy's except the
 * transcendentals' last FP64 ulps.  C is FP64 [batch, M, N]. */
int nao_matmul_fp64(const float* A, const float* B, double* C, int64_t batch, int64_t M,
                    int64_t N, int64_t K, int64_t stride_a, int64_t stride_b, int transpose_b,
                    void* stream);
/* rows [rows, n] FP32 -> FP64: kind 0 softmax (engine.py:185-194), 1 layernorm
 * (:197-213, ln_eps as the attribute's double), 2 sum, 3 mean (y: [rows]). */
int nao_rows_fp64(int kind, const float* x, double* y, int64_t rows, int64_t n, double ln_eps,
                  void* stream);
/* _unary_intrinsic(fp64=True): FP64 results of FP32 inputs. */
int nao_unary_f64out(const float* x, double* y, int64_t n, int kind, void* stream);

/* Additive fault / drift hook on a node output (engine.py:325-351 `inject`):
 * out = y with +-1-ulp flips on ~n/period elements and a relative fault
 * `fault_scale` on ~n/fault_period elements (0 disables either).  Used to
 * materialise claimed traces for tests and the benchmark harness. */
int nao_inject_drift(const float* y, float* out, int64_t n, uint32_t seed, uint32_t period,
                     float fault_scale, uint32_t fault_period, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NAO_B200_H */
