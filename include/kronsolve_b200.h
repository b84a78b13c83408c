/*
 * kronsolve_b200 -- C-ABI of the B200-native (sm_100a, FP64) FastKroneckerRegression hot path.
 *
 * Drop-in boundary.  The reference (arXiv 2209.04876, package `kronsolve`) has no FFI: its
 * boundary is the set of Python functions re-exported by pkg/src/kronsolve/__init__.py:3-73.
 * Every entry point below is the device half of one of those functions; the Python mirror in
 * paper_2209_04876_b200/ keeps the reference signature and calls these through ctypes
 * (see INTEGRATION.md).  Each entry cites the reference function it replaces.
 *
 * Conventions
 *   - All matrices are row-major float64 in device memory (HBM); indices are int64.
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous on that stream
 *     unless it documents a host output (it then synchronises the stream).
 *   - Return value: KS_OK or one of the KS_E* codes; ks_last_error() gives a thread-local
 *     message.  The Python shim maps KS_EINVAL -> InvalidInputError, KS_ESIZE ->
 *     SizeGuardError, KS_ENUMERICAL / KS_EDIVERGED -> NumericalFailureError, KS_ECUDA ->
 *     KronsolveError (reference errors.py:4-37).
 *   - Scratch memory is stream-ordered (cudaMallocAsync on the device's default pool).
 *   - No entry point falls back to the CPU.
 */
#ifndef KRONSOLVE_B200_H
#define KRONSOLVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KS_OK 0
#define KS_EINVAL 1
#define KS_ESIZE 2
#define KS_ENUMERICAL 3
#define KS_ECUDA 4
#define KS_EDIVERGED 5

#define KS_ABI_VERSION 1

int ks_abi_version(void);
const char* ks_last_error(void);

/* ---------------------------------------------------------------- dense primitives */

/* Batched strided GEMM: C[b] = alpha * A[b](MxK) * B[b](KxN) + beta * C[b].
 * Element (i,j) of X lives at X[i*x_rs + j*x_cs + b*x_bs].  General building block of the
 * implicit Kronecker multiplies (reference kron.py:66-77 tensordot / matmul). */
int ks_gemm(int64_t M, int64_t N, int64_t K, double alpha,
            const double* A, int64_t a_rs, int64_t a_cs, int64_t a_bs,
            const double* B, int64_t b_rs, int64_t b_cs, int64_t b_bs,
            double beta, double* C, int64_t c_rs, int64_t c_cs, int64_t c_bs,
            int64_t batch, void* stream);

/* Deterministic split-K product C(MxN) = alpha * A^T B for tall A (KxM), B (KxN), M,N <= 128.
 * Element (k,m) of A at A[k*a_ks + m*a_ms]; (k,n) of B at B[k*b_ks + n*b_ns].
 * Replaces the Gram / projection products a.T @ a (solvers.py:146, :439) and g @ a_tilde
 * (leverage.py:127). */
int ks_gemm_tn_tall(int64_t M, int64_t N, int64_t K, double alpha,
                    const double* A, int64_t a_ks, int64_t a_ms,
                    const double* B, int64_t b_ks, int64_t b_ns,
                    double* C, void* stream);

/* out = (F_0 kron ... kron F_{nf-1}) b with b of shape (prod cols, ncols), row-major.
 * Replaces kron.kron_mat_mul (kron.py:44-77) and kron_vec_square (kron.py:80-100). */
int ks_kron_mat_mul(int32_t nf, const double* const* factors, const int64_t* rows,
                    const int64_t* cols, const double* b, int64_t ncols, double* out,
                    void* stream);

/* K1: T(p x q) = L^T (m x p) . B (m x k, leading dim ldb) . R (k x q).
 * The n^2 pass of kronmatmul_svd_solve: kron_mat_mul([U1^T, U2^T], b) (solvers.py:314). */
int ks_kron2_contract(const double* L, const double* B, int64_t ldb, const double* R,
                      int64_t m, int64_t k, int32_t p, int32_t q, double* T, void* stream);
/* K1 with ||B||^2 from the same pass (bsq: one device double).  The exact solve's loss then follows
 * from ||b||^2 - sum_k s_k^2 t_k^2 / (s_k^2 + lam) without a second pass over b (solvers.py:318). */
int ks_kron2_contract_sumsq(const double* L, const double* B, int64_t ldb, const double* R,
                            int64_t m, int64_t k, int32_t p, int32_t q, double* T, double* bsq,
                            void* stream);

/* K13: T (R0 x R1 R2) = (U0 kron U1 kron U2)^T b for the n0 x n1 x n2 tensor b, one streaming pass
 * over b in the reference's rightmost-first order (kron.py:66-77 at N = 3, reached from the Tucker
 * exact core update tucker.py:120 -> solvers.py:314).  U_k: n_k x R_k row-major.
 * ks_kron3_supported returns 1 for the geometries the kernel handles (n2 % 8 == 0, n2 <= 128,
 * R1 <= 32, R2 <= 8, R0 R1 R2 <= 2048), else 0; ks_kron3_contract returns KS_ESIZE for the others. */
int ks_kron3_supported(int64_t n0, int64_t n1, int64_t n2, int32_t R0, int32_t R1, int32_t R2);
int ks_kron3_contract(const double* U0, const double* U1, const double* U2, const double* B,
                      int64_t n0, int64_t n1, int64_t n2, int32_t R0, int32_t R1, int32_t R2,
                      double* T, void* stream);
/* K13 with ||b||^2 (bsq: one device double) from the same pass when n2 <= 64 (else a second pass). */
int ks_kron3_contract_sumsq(const double* U0, const double* U1, const double* U2, const double* B,
                            int64_t n0, int64_t n1, int64_t n2, int32_t R0, int32_t R1, int32_t R2,
                            double* T, double* bsq, void* stream);
/* Profiling aid: while set (a cudaEvent_t; NULL clears it), the fused Richardson loop records this
 * event (external) right before its persistent kernel's launch. */
int ks_debug_loop_kernel_event(void* event);
/* Profiling aid: later K13 launches only stream b through their ring (no arithmetic). */
int ks_debug_kron3_stream_only(int32_t on);

/* K2: out[0] = sum_{i,j} ((L X R^T)[i,j] - B[i,j])^2 without materialising K x.
 * L: m x p, X: p x q, R: k x q, B: m x k.  The n^2 pass of ridge_loss (solvers.py:251-262). */
int ks_kron2_residual_sumsq(const double* L, const double* X, const double* R,
                            const double* B, int64_t ldb, int64_t m, int64_t k, int32_t p,
                            int32_t q, double* out, void* stream);

/* out[0] = sum (a - b)^2 (b may be NULL -> sum a^2).  Deterministic. */
int ks_sumsq_diff(const double* a, const double* b, int64_t n, double* out, void* stream);

/* flags[0] = any non-finite entry, flags[1] = any nonzero entry (int32, device).
 * Mirrors tensor.as_matrix (tensor.py:35-42) and solvers._validated_problem (:265-274). */
int ks_check_finite_nonzero(const double* a, int64_t n, int32_t* flags, void* stream);

/* ---------------------------------------------------------------- small dense (d <= 128) */

/* R factor (d x d, upper) of a Householder TSQR of A (n x d).  Rows beyond n zero-padded. */
int ks_qr_r(const double* A, int64_t n, int32_t d, double* R, void* stream);

/* One-sided Jacobi SVD of a d x d matrix M: sigma descending (d), V (d x d, row-major,
 * column j = right singular vector j).  Used for compact_svd (tensor.py:76-107) via QR and
 * for factor_gram's eigendecomposition of a PSD Gram (solvers.py:143-150). */
int ks_svd_small(const double* M, int32_t d, double* sigma, double* V, void* stream);

/* X = M^-1 for a d x d matrix (LU with partial pivoting, LAPACK getrf pivot rule).
 * info (device int32[2]): info[0] = k+1 if pivot k is exactly zero (np.linalg.solve's
 * LinAlgError, leverage.py:114-119), info[1] = 1 if X has non-finite entries (:120-123). */
int ks_inverse_small(const double* M, int32_t d, double* X, int32_t* info, void* stream);

/* Batched ks_svd_small over `batch` contiguous d x d problems (one CTA each, concurrently). */
int ks_svd_small_batched(const double* M, int32_t batch, int32_t d, double* sigma, double* V,
                         void* stream);

/* Eigen-decomposition of nb (<= 8) symmetric PSD d x d Gram matrices at separate device
 * addresses, each read as 0.5 (M + M^T) (the symmetrisation before eigh, solvers.py:440-446);
 * outputs as ks_svd_small_batched: sigma (nb x d, descending) = eigenvalues, V (nb x d x d). */
int ks_sym_eig_batched(int32_t nb, const double* const* mats, int32_t d, double* sigma, double* V,
                       void* stream);

/* Thin SVD of A (n x d): U (n x d), sigma (d, descending), V (d x d).  Columns past the
 * numerical rank (sigma <= rank_tol*sigma_max) are zeroed and *rank (host) reports it.
 * Replaces tensor.compact_svd (tensor.py:76-107).  Synchronises the stream, unless rank is NULL
 * (the caller then counts sigma_j > rank_tol * sigma_0 itself, e.g. for several factors at once). */
int ks_compact_svd(const double* A, int64_t n, int32_t d, double rank_tol, double* U,
                   double* sigma, double* V, int32_t* rank, void* stream);
/* The same without any host synchronisation (CUDA-graph capturable): no rank, and the QR's
 * CholeskyQR2 status words go to info_dev (2 x int32, device; nonzero = declined, the result is
 * undefined and the caller redoes it with ks_compact_svd). */
int ks_compact_svd_async(const double* A, int64_t n, int32_t d, double rank_tol, double* U,
                         double* sigma, double* V, int32_t* info_dev, void* stream);

/* ---------------------------------------------------------------- NumPy-exact random streams */

/* out[i] = Generator.random() draw number (skip + i) of a PCG64 stream with the given
 * 128-bit state/increment ((raw >> 11) * 2^-53).  Bit-exact with numpy.random.PCG64. */
int ks_pcg64_random(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                    uint64_t skip, int64_t count, double* out, void* stream);

/* out[i] = Generator.standard_normal() draw i / divisor (ziggurat; tables from the installed
 * NumPy, passed in ki[256] (uint64), wi[256], fi[256] on the device).  Bit-exact with
 * numpy.random.Generator(PCG64).standard_normal except for ulp-level differences of libm
 * log1p/exp in the (rare) tail branch.  Replaces the host draw of leverage.py:124-126.
 * status: optional device int32 (zeroed by the caller).  When given and count <= 2^25 the call
 * is fully asynchronous and chain-resolution failures are OR-ed into *status (nonzero = the
 * draw is invalid, KS_ENUMERICAL); otherwise the call synchronises the stream and returns
 * KS_ENUMERICAL itself. */
int ks_pcg64_standard_normal(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                             uint64_t inc_lo, int64_t count, double divisor,
                             const uint64_t* ki, const double* wi, const double* fi,
                             double* out, int32_t* status, void* stream);

/* ---------------------------------------------------------------- leverage scores & sampling */

/* scores[i] = ||Q a_i||^2 / denom for rows a_i of A (n x d), Q (r x d).
 * JL estimator body of approx_leverage_scores_jl (leverage.py:114-129). */
int ks_jl_scores(const double* A, int64_t n, int32_t d, const double* Q, int32_t r,
                 double denom, double* scores, void* stream);

/* Q (r x d) = scale * GA G^-1 for symmetric positive definite G (d x d) and GA (r x d) by a
 * one-CTA Cholesky solve (the (1+eps/4) (g a_tilde) gram_tilde^-1 factor, leverage.py:114-127).
 * info[0] (device int32) = k+1 if pivot k is not positive (the caller then uses LU). */
int ks_jl_projection(const double* G, int32_t d, const double* GA, int32_t r, double scale,
                     double* Q, int32_t* info, void* stream);

/* The two halves of ks_jl_projection, so the factorization (which needs only the Gram) can run
 * while GA is still being drawn: ks_jl_cholesky factors G into the workspace Lws
 * (d (d + 1) + d doubles; info as above), ks_jl_solve forms Q from Lws and GA. */
int ks_jl_cholesky(const double* G, int32_t d, double* Lws, int32_t* info, void* stream);
int ks_jl_solve(const double* Lws, int32_t d, const double* GA, int32_t r, double scale, double* Q, void* stream);

/* exact statistical leverage scores: scores[i] = sum_k U[i,k]^2 * wts[k] (leverage.py:51-64) */
int ks_row_weighted_sumsq(const double* U, int64_t n, int32_t d, const double* wts,
                          double* scores, void* stream);

/* ProductSampler per-factor tables (leverage.py:159-175): total = pairwise sum (NumPy order),
 * probs = scores / total, cdf = sequential cumsum (bit-exact, parallel verified scan).
 * flags[0]: 1 if any score < 0 or non-finite, 2 if total <= 0.  If renormalise != 0 the cdf is
 * additionally divided by its last entry (Generator.choice with p, used by sample_rows with an
 * explicit distribution, leverage.py:222-230). */
int ks_sampler_tables(const double* scores, int64_t n, int32_t renormalise, double* probs,
                      double* cdf, int32_t* flags, void* stream);

/* ks_sampler_tables for nf <= 8 score vectors at once (one CTA per factor, concurrently);
 * flags holds one int32 per factor.  cdf may be NULL (probabilities only). */
int ks_sampler_tables_batched(int32_t nf, const double* const* scores, const int64_t* n,
                              int32_t renormalise, double* const* probs, double* const* cdf,
                              int32_t* flags, void* stream);

/* Inverse-CDF draws: idx[t*stride + off] = clip(upper_bound(cdf, u[t]), 0, n-1) (leverage.py:196-200). */
int ks_searchsorted_right(const double* cdf, int64_t n, const double* u, int64_t s,
                          int64_t* idx, int64_t stride, int64_t off, void* stream);

/* Sketch weights (leverage.py:220-231): prob[t] = prod_f probs_f[idx[t, f]];
 * w[t] = 1 / sqrt(prob[t] * s). */
int ks_sketch_weights(int32_t nf, const double* const* probs, const int64_t* idx, int64_t s,
                      double* w, void* stream);

/* sparse_diagonal_from_sketch (kron.py:173-190): flat = ravel(idx) (C order), stable sort,
 * unique, values = sqrt(w2[first] + pairwise_sum(w2[rest])) in NumPy reduceat order.
 * sd_idx / sd_val must hold s entries; *nnz (host) is set.  Synchronises the stream. */
int ks_sketch_diag(int32_t nf, const int64_t* idx, const int64_t* row_shape, const double* w,
                   int64_t s, int64_t* sd_idx, double* sd_val, int64_t* nnz, void* stream);

/* Gather b_at[t] = b[idx[t]] (solvers.py:451). */
int ks_gather(const double* b, const int64_t* idx, int64_t n, double* out, void* stream);

/* out[t] = b[idx[t]] for t < *count_dev (device count, cap = buffer capacity); b may be device
 * memory or page-locked host memory (mapped: only the gathered entries cross PCIe). */
int ks_gather_count(const double* b, const int64_t* idx, const int64_t* count_dev, int64_t cap, double* out,
                    void* stream);

/* ---------------------------------------------------------------- sketched operator & solver */

/* Grouped view of a sparse diagonal for the two-group scheme of kron.py:258-354.
 * The nnz samples are ordered by (left group row, right group row); `seg` (u_left+1) are
 * CSR offsets of each distinct left row, `lrow[u]` its row in Lmat (u_left x dL, ld ldl),
 * `rrow[t]` the right-group row of sample t in Rmat (ld ldr), `v[t]` the diagonal value. */
typedef struct ks_sketch_view {
  const double* Lmat; int64_t ldl; int32_t dL;
  const double* Rmat; int64_t ldr; int32_t dR;
  int64_t u_left; int64_t nnz;
  const int64_t* seg; const int64_t* lrow; const int64_t* rrow; const double* v;
} ks_sketch_view;

/* Two-factor fused form of ks_sketch_diag + ks_sketch_group (left group {0}, right group {1}):
 * from the s draws idx (s x 2) and weights w builds the sparse diagonal (sd_idx, sd_val, sorted
 * and deduplicated exactly as ks_sketch_diag) and its grouped view in the same pass: rrow[t] = i1
 * of entry t, seg (u_left + 1 segment starts over the entries), lrow (u_left first-factor rows);
 * the grouped order is the sparse-diagonal order (perm = identity, v = sd_val).  nnz and u_left
 * go to counts (host, 2; the call then synchronises the stream) and/or counts_dev (device, 2;
 * with counts NULL the call is asynchronous and graph-capturable).  Buffers hold s (seg: s + 1)
 * entries. */
int ks_sketch_diag_grouped2(const int64_t* idx, const int64_t* row_shape, const double* w, int64_t s,
                            int64_t* sd_idx, double* sd_val, int64_t* seg, int64_t* lrow, int64_t* rrow,
                            int64_t* counts, int64_t* counts_dev, void* stream);

/* ks_sketch_diag_grouped2 that also writes first_raw[t] (s entries) = the index, in draw order, of
 * the first draw of sparse-diagonal entry t, so b can be gathered at the raw draws (ks_gather_draws2)
 * while the sketch is sorted, and then permuted on the device (ks_gather_count). */
int ks_sketch_diag_grouped2_ex(const int64_t* idx, const int64_t* row_shape, const double* w, int64_t s,
                               int64_t* sd_idx, double* sd_val, int64_t* seg, int64_t* lrow, int64_t* rrow,
                               int64_t* counts, int64_t* counts_dev, int64_t* first_raw, void* stream);

/* out[q] = b[draws[q,0] * n1 + draws[q,1]] for the s two-factor draws (b device or page-locked
 * host memory): the right-hand side's b entries read at the raw draws (solvers.py:451). */
int ks_gather_draws2(const double* b, const int64_t* draws, int64_t n1, int64_t s, double* out, void* stream);

/* Build the grouped view of a sparse diagonal (sorted unique flat row indices sd_idx with values
 * sd_val, nnz entries) for the factor split left_pos | right_pos (kron.balanced_partition,
 * kron.py:117-144).  Outputs (caller-allocated, nnz-sized): seg (nnz+1), lrow, rrow, v, perm
 * (grouped position -> position in sd_idx).  Lbuf (nnz x dL) must be given iff the left group
 * is not a single factor (Khatri-Rao rows are materialised, kron.py:193-205), Rbuf (nnz x dR)
 * iff the right group is not a single factor.  *u_left (host) receives the number of distinct
 * left rows.  Synchronises the stream. */
int ks_sketch_group(int32_t nf, const double* const* factors, const int64_t* rows,
                    const int64_t* cols, int32_t nleft, const int32_t* left_pos, int32_t nright,
                    const int32_t* right_pos, const int64_t* sd_idx, const double* sd_val,
                    int64_t nnz, int64_t* seg, int64_t* lrow, int64_t* rrow, double* v,
                    int64_t* perm, double* Lbuf, double* Rbuf, int64_t* u_left, void* stream);

/* vals[perm[t]] = v[t] * Lrow_t^T X Rrow_t  (sketched_kron_apply, kron.py:258-300), X: dL x dR
 * in grouped column order.  perm may be NULL (identity). */
int ks_sketched_apply(const ks_sketch_view* sk, const double* X, const int64_t* perm,
                      double* vals, void* stream);

/* G(dL x dR) = sum_t bv[perm[t]] v[t] Lrow_t Rrow_t^T (sketched_kron_transpose_apply,
 * kron.py:312-354). */
int ks_sketched_transpose_apply(const ks_sketch_view* sk, const double* bv, const int64_t* perm,
                                double* G, void* stream);

/* Fused Richardson loop of fast_kronecker_regression (solvers.py:201-248 with the operator of
 * :454-456 and KronPreconditioner.apply of :180-183), all on device:
 *   step = P (H x - rhs),  H x = sum_t v_t^2 (Lrow_t^T X Rrow_t) Lrow_t Rrow_t^T + lam x,
 *   P y = (VL kron VR) diag(dinv) (VL kron VR)^T y  (VL dL x dL, VR dR x dR).
 * x (dL x dR) starts at zero.  hist (max_iters doubles) receives the step norms; *iters and
 * *hist_len (host) are set.  Returns KS_EDIVERGED on the reference's divergence rule.
 * Synchronises the stream at the end. */
int ks_richardson_sketched(const ks_sketch_view* sk, const double* VL, const double* VR,
                           const double* dinv, const double* rhs, double lam, double damping,
                           int32_t max_iters, double residual_tol, double* x, double* hist,
                           int32_t* iters, int32_t* hist_len, void* stream);

/* Fused Richardson for single-factor groups (dL, dR in {16, 32, 64}) on the persistent path:
 * additionally builds the right-hand side (SK)^T S b = sum_t v_t (v_t b_t) L_u R_t^T (solvers.py:455,
 * kron.py:303-354) inside the loop kernel from b_at (b at the sparse-diagonal rows, in
 * sparse-diagonal order; perm maps grouped -> sparse-diagonal position, NULL if identical) and
 * returns it in rhs_out (dL x dR).  dinv may be NULL: then dinv = pseudo-reciprocal(wL (x) wR + lam)
 * (solvers.py:186-198) with wL, wR the two Gram eigenvalue vectors.  Other arguments and
 * returns as ks_richardson_sketched; KS_ESIZE when the shape is not supported. */
int ks_richardson_fused(const ks_sketch_view* sk, const int64_t* perm, const double* b_at, const double* VL,
                        const double* wL, const double* VR, const double* wR, const double* dinv, double lam,
                        double damping, int32_t max_iters, double residual_tol, double* x, double* hist,
                        double* rhs_out, int32_t* iters, int32_t* hist_len, void* stream);

/* Asynchronous ks_richardson_fused for CUDA-graph capture: sk->nnz / sk->u_left are capacities,
 * the real counts are read on the device from counts_dev ([nnz, u_left], as written by
 * ks_sketch_diag_grouped2), and the loop state [status (1 converged, 2 diverged), iterations,
 * history length] is written to state_dev (device, 3 int32).  No host synchronisation. */
int ks_richardson_fused_async(const ks_sketch_view* sk, const int64_t* counts_dev, const int64_t* perm,
                              const double* b_at, const double* VL, const double* wL, const double* VR,
                              const double* wR, const double* dinv, double lam, double damping, int32_t max_iters,
                              double residual_tol, double* x, double* hist, double* rhs_out, int32_t* state_dev,
                              const void* plan_ws, void* stream);

/* The persistent loop's work plan (chunks of <= 16 left rows / <= 64 samples, balanced CTA
 * ranges) built ahead of time, e.g. while the eigensolves still run: plan_ws (device,
 * ks_richardson_plan_bytes(u_left capacity, nnz capacity) bytes) is then passed to
 * ks_richardson_fused_async.  Asynchronous. */
int64_t ks_richardson_plan_bytes(int64_t u_left_cap, int64_t nnz_cap);
int ks_richardson_plan_async(const ks_sketch_view* sk, const int64_t* counts_dev, void* plan_ws, void* stream);

/* Profiling aid: globaltimer stamps (ns) of CTA 0 of the last ks_jl_projection: entry,
 * operands staged, Cholesky done, exit. */
int ks_debug_jl_projection_stamps(uint64_t* out4);

/* Profiling aid: sweeps used by the last one-sided Jacobi launch (first 8 problems, host out8). */
int ks_debug_jacobi_sweeps(int32_t* out8);


/* Row-sharded Richardson loop (distributed.py; replaces the per-rank part of
 * richardson_solve, solvers.py:201-248, in a row-sharded fast_kronecker_regression).  Per rank:
 *   ks_shard_loop_sizes  workspace capacities for a sketch view: out4 = [Lpack doubles, Rpack
 *                        doubles, partial-sum doubles, plan + barrier bytes];
 *   ks_shard_loop_pack   the rank's sampled rows in the preconditioner's eigenbasis (L VL, R VR,
 *                        v_t and v_t b_t in the padding) and the kernel's work plan;
 *   ks_shard_loop_apply  one apply-only launch of the persistent eigenbasis kernel: mode 1 = the
 *                        rank's right-hand-side partial, mode 2 = its normal-operator partial at
 *                        x_in; the reduced d_L x d_R partial goes to g_out (to be all-reduced);
 *                        a no-op once *stop != 0;
 *   ks_shard_loop_update one CTA: it < 0 stores rhs' = g and tol; it >= 0 forms step' = dinv o
 *                        (g + lam x' - rhs'), records ||step'||, applies the stopping and divergence
 *                        rules and updates x'.  state = [stopped, status (1 converged, 2 diverged),
 *                        iterations, history length], aux[0] = tol.
 * All asynchronous (capturable, with the all-reduces between them, as one CUDA graph). */
int ks_shard_loop_sizes(const ks_sketch_view* sk, int64_t* out4);
int ks_shard_loop_pack(const ks_sketch_view* sk, const int64_t* counts_dev, const double* VL, const double* VR,
                       const double* b_at, const int64_t* perm, double* Lpack, double* Rpack, void* plan_ws,
                       void* stream);
int ks_shard_loop_apply(const ks_sketch_view* sk, const double* Lpack, const double* Rpack, const void* plan_ws,
                        int32_t mode, const double* x_in, double* g_out, const int32_t* stop, double* part_ws,
                        void* stream);
int ks_shard_loop_update(int32_t it, const double* g, double* x, double* rhs, const double* wL, const double* wR,
                         int32_t dL, int32_t dR, double lam, double damping, double residual_tol, double* hist,
                         int32_t* state, double* aux, void* stream);

/* Profiling aid: with on != 0, later launches of the phase-separated eigenbasis Richardson loop
 * run its profiling instantiation (CTA 0 records clock64 at every phase boundary); the product
 * path runs the instantiation without instrumentation.  Process-wide, default off. */
int ks_debug_richardson_profile(int32_t on);

/* Profiling aid: average SM cycles per phase of the last profiled eigenbasis loop run
 * (CTA 0): apply, flag barrier 1, reduce, flag barrier 2, norm + stop rules + x update, loop
 * overhead. */
int ks_debug_richardson_phases(int32_t iters, double* out6);

/* Profiling aid: CTA 0's apply phase of the last profiled run split per iteration (SM cycles):
 * L load wait, Y phase, sample phase, G phase (out8[4..7] unused). */
int ks_debug_richardson_apply_split(int32_t iters, double* out8);

/* Profiling aid: per-CTA apply start / end (%globaltimer, ns) of iteration 5 of the last profiled
 * run: out[2 b], out[2 b + 1] for b < nctas <= 256. */
int ks_debug_richardson_cta_apply(int32_t nctas, uint64_t* out);

/* Preconditioner apply y = (VL kron VR) diag(dinv) (VL kron VR)^T r (solvers.py:180-183). */
int ks_kron_precond_apply(const double* VL, const double* VR, int32_t dL, int32_t dR,
                          const double* dinv, const double* r, double* y, void* stream);


/* ---------------------------------------------------------------- Tucker factor-matrix updates
 * (reference tucker.py).  The "other" factors of a mode-n update are
 * M (1..4) matrices A_m (I_m x R_m, row-major); leftover Kronecker vectors (length
 * R_rest = prod R_m <= 4096) are indexed C-order by (r_0, ..., r_{M-1}).  V_m / G_m / E_m are the
 * eigenvectors (R_m x R_m, column j = vector j), Gram matrices and eigenvalues of each A_m^T A_m
 * (FactorGram, solvers.py:126-150).  gn = G (R_n x R_rest, core unfolding), gnp = G^+ (R_rest x R_n),
 * R_n <= 64. */

/* PCG64 draws of many streams: out[m*rows*s + row*s + t] = random() draw (m*s + t) of stream row;
 * states holds 4 words per stream: (state hi, state lo, inc hi, inc lo) when seeded == 0, or the
 * pcg64_set_seed inputs (initstate hi, lo, initseq hi, lo) when seeded != 0 (the kernel then
 * seeds the stream as PCG64(SeedSequence) does).  The per-row sampler streams of
 * fast_factor_matrix_update (tucker.py:361-369). */
int ks_pcg64_random_streams(const uint64_t* states, int32_t seeded, int64_t rows, int32_t nf, int64_t s,
                            double* out, void* stream);

/* Product-sampler draws of `rows` independent sketches of s samples each (leverage.py:196-231 per
 * row): idx ((rows*s) x (M+1), column 0 = row, then clip(upper_bound(cdf_m, u)) per factor) and
 * w = 1/sqrt(prod_m prob_m[idx_m] * s), from uniforms laid out as ks_pcg64_random_streams. */
int ks_factor_draws_rows(int32_t M, const double* const* cdf, const double* const* prob, const int64_t* n,
                         const double* u, int64_t rows, int64_t s, int64_t* idx, double* w, void* stream);

/* build_factor_workspace (tucker.py:217-280) minus the R_n x R_n inverse: power iteration
 * (_power_iteration, :283-313, start vector v0 = default_rng(0).standard_normal(R_rest)) on the
 * constrained Gram, wout[0] = w = (1 + 12/eps) * estimate * 1.05, wout[1] = estimate,
 * bdiag = pseudo_reciprocal(kron(E) + w), right = lam (G^T)^+ - w G and
 * cm = I + right (V diag(bdiag) V^T) G^+ (the Woodbury core matrix; its inverse = correction_mid,
 * via ks_inverse_small).  flags[0] |= 1 if a power iterate is non-finite. */
int ks_factor_workspace(int32_t M, const int32_t* R, const double* const* V, const double* const* G,
                        const double* const* E, int32_t Rn, const double* gn, const double* gnp,
                        double lam, double eps, const double* v0, double* wout, double* bdiag,
                        double* right, double* cm, int32_t* flags, void* stream);

/* FactorUpdateWorkspace.apply (which = 0), .apply_base (1), .apply_penalized_normal (2) of one
 * vector z (tucker.py:185-214). */
int ks_factor_ws_apply(int32_t M, const int32_t* R, const double* const* V, const double* const* G,
                       int32_t Rn, const double* gn, const double* gnp, const double* mid,
                       const double* right, const double* bdiag, const double* wdev, double lam,
                       const double* z, int32_t which, double* out, void* stream);

/* Dynamic shared memory bytes of one factor-row solve (ks_factor_rows_richardson) with `threads`
 * threads per row. */
int64_t ks_factor_rows_smem(int32_t Rrest, int32_t Rright, int32_t Rn, int32_t max_iters, int32_t cap,
                            int32_t ucap, int32_t threads);

/* The per-row loop of fast_factor_matrix_update (tucker.py:361-379), one CTA per row: the row's
 * segment of the sparse diagonal (sd_idx = row * I_rest + flat index, sorted, or plain flat
 * indices when shared != 0 and every row uses the same sketch), b_at gathered in place from the
 * tensor x (stride xs_n of mode n, xs[m] of the other modes), rhs, damped Richardson with the
 * Woodbury preconditioner and the exact stopping / divergence rules of richardson_solve
 * (solvers.py:201-248), projection and out[row] = (G^T)^+ G^T (G^T)^+ z.  iters[row] = completed
 * updates; flags[row] = 1 if the row diverged, 2 if it holds more than cap samples.  kr:
 * nnz x prod_{m>=1} R_m scratch (required when M >= 3).  hist (rows x max_iters) optional. */
int ks_factor_rows_richardson(int32_t M, const double* const* A, const int64_t* I, const int32_t* R,
                              const double* const* V, int32_t Rn, const double* gn, const double* gnp,
                              const double* mid, const double* right, const double* bdiag,
                              const double* wdev, double lam, const int64_t* sd_idx, const double* sd_val,
                              int64_t nnz, int32_t shared, int64_t rows, const double* x, int64_t xs_n,
                              const int64_t* xs, double* kr, double damping, int32_t max_iters,
                              double residual_tol, int32_t cap, double* out, int32_t* iters,
                              int32_t* flags, double* hist, void* stream);

/* Q (n x k) of np.linalg.qr(A) (reduced): Householder QR with LAPACK's dgeqrf / dorg2r
 * conventions, one CTA.  initial_model (tucker.py:400-409). */
int ks_qr_explicit(const double* A, int64_t n, int32_t k, double* Q, void* stream);

/* X (d x n) = (V / sigma) U^T for a compact SVD (U: n x k, sigma: k, V: d x k): pseudo_inverse
 * (tensor.py:110-115) and np.linalg.pinv of naive_factor_update (tucker.py:157). */
int ks_pinv_compose(const double* U, int64_t n, const double* sigma, const double* V, int64_t d,
                    int32_t k, double* X, void* stream);


/* sketch_rows_of_kron (kron.py:208-222): out (s x prod cols) = w[t] * (A_0[j_0] (x) ... (x) A_{nf-1}[j_{nf-1}])
 * for draw t; idx holds s x nf multi-indices (flat == 0) or s flat row indices (flat != 0).  The
 * materialised S K of sketch_and_solve_ridge (solvers.py:334-369). */
/* Explicit Kronecker product C = A kron B of row-major A (m x p) and B (k x q) into C (m k x p q)
 * (tensor.py:186-198 for two factors; the materialised right group of the N >= 3 KronMatMul and
 * loss passes, solvers.py:314 / :261).  Asynchronous. */
int ks_kron_explicit2(const double* A, int64_t m, int32_t p, const double* B, int64_t k, int32_t q, double* C,
                      void* stream);

/* The spectral-row sample of one factor (leverage.py:235-252, scaled as solvers.py:424-427):
 * out (m x d) row t = (w[t] * A[idx[t], :]) / divisor, for row-major A (n x d); indices are not
 * range-checked (they come from the device sampler).  Asynchronous. */
int ks_scaled_row_gather(const double* A, int64_t n, int32_t d, const int64_t* idx, const double* w, int64_t m,
                         double divisor, double* out, void* stream);

int ks_sketch_rows(int32_t nf, const double* const* factors, const int64_t* rows, const int32_t* cols,
                   const int64_t* idx, int32_t flat, const double* w, int64_t s, double* out, void* stream);


/* CholeskyQR2 of a tall A (n x d, n >= d, d <= 128): R (d x d upper) with R^T R = A^T A; *ok (host)
 * = 0 when A is too ill-conditioned (kappa^2 > ~1e13) and R is undefined.  ks_qr_r uses it for
 * n >= 4d before falling back to Householder TSQR.  Synchronises the stream. */
int ks_chol_qr2_r(const double* A, int64_t n, int32_t d, double* R, int32_t* ok, void* stream);

/* Statistical leverage scores of a numerically full-rank tall A: scores[i] = ||(A R^-1)_i||^2 with
 * R = R2 R1 from CholeskyQR2, formed as ||(Q1 R2^-1)_i||^2 from the first pass's Q1 = A R1^-1
 * (= ridge_leverage_scores(compact_svd(a), 0), leverage.py:51-64, for
 * kappa(A) < ~3e6).  *ok = 0 when A is too ill-conditioned (scores undefined; use the compact SVD).
 * Synchronises the stream.  spectral_approx_rows' scores (leverage.py:235-252). */
int ks_leverage_scores_tall(const double* A, int64_t n, int32_t d, double* scores, int32_t* ok, void* stream);

/* ks_leverage_scores_tall without a host round trip: info_dev (device, 2 x int32) is written with
 * the two Cholesky status words (nonzero = declined, scores undefined).  Graph-capturable. */
int ks_leverage_scores_tall_async(const double* A, int64_t n, int32_t d, double* scores, int32_t* info_dev,
                                  void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KRONSOLVE_B200_H */
