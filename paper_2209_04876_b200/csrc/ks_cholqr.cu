// CholeskyQR2 for tall factor matrices (n >> d, d <= 128) and leverage scores from it.
//
// The R factor of A (reference: the QR inside tensor.compact_svd, tensor.py:76-107, LAPACK
// Householder) is computed as R = R2 R1 with R1 = chol(A^T A), Q1 = A R1^-1, R2 = chol(Q1^T Q1):
// two Gram passes on the FP64 tensor pipe (ks_gemm_tn_tall) and one streaming triangular solve,
// instead of a latency-bound Householder TSQR.  R is unique up to row signs; every consumer (the
// one-sided Jacobi SVD of R, U = A V Sigma^-1, scores) is invariant to them.  CholeskyQR2 is
// backward stable like Householder for kappa(A) below ~1e7; a Cholesky pivot that is not
// comfortably positive (ill-conditioned or rank-deficient A) reports failure and the caller falls
// back to Householder TSQR (ks_qr_r).
//
// Statistical leverage scores (ridge_leverage_scores(compact_svd(a), 0), leverage.py:51-64) of a
// numerically full-rank A are the squared row norms of A R^-1; ks_leverage_scores_tall fuses the
// triangular solve and the row norms in one pass.
#include "ks_common.cuh"

namespace ks {
int gemm_tn_tall(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t a_ks,
                 int64_t a_ms, const double* B, int64_t b_ks, int64_t b_ns, double* C);
int gemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t a_rs,
         int64_t a_cs, int64_t a_bs, const double* B, int64_t b_rs, int64_t b_cs, int64_t b_bs, double beta,
         double* C, int64_t c_rs, int64_t c_cs, int64_t c_bs, int64_t batch);
}  // namespace ks

namespace {

constexpr int CT = 256;

// Upper Cholesky factor R (R^T R = 0.5 (G + G^T)) of a d x d Gram in one CTA (right-looking, in
// shared memory).  info[slot] = k + 1 if pivot k is below tol * max diag (not comfortably PD).
__global__ void __launch_bounds__(CT) chol_upper_kernel(const double* __restrict__ G, int d, double* __restrict__ R,
                                                       int32_t* __restrict__ info, int slot) {
  extern __shared__ double S[];  // d x d, row-major, upper triangle used
  __shared__ double s_piv, s_dmax;
  __shared__ int s_bad;
  for (int e = threadIdx.x; e < d * d; e += CT) {
    const int i = e / d, j = e - i * d;
    S[e] = i <= j ? 0.5 * (G[i * d + j] + G[j * d + i]) : 0.0;
  }
  if (threadIdx.x == 0) {
    s_bad = 0;
    double m = 0.0;
    for (int i = 0; i < d; i++) m = fmax(m, 0.5 * (G[i * d + i] + G[i * d + i]));
    s_dmax = m;
  }
  __syncthreads();
  const double tol = 1e-13 * s_dmax;  // kappa(A)^2 below ~1e13: CholeskyQR2 regime
  for (int k = 0; k < d; k++) {
    if (threadIdx.x == 0) {
      const double p = S[k * d + k];
      if (!(p > tol) || !isfinite(p)) {
        s_bad = k + 1;
        s_piv = 1.0;
      } else {
        s_piv = sqrt(p);
      }
      S[k * d + k] = s_piv;
    }
    __syncthreads();
    if (s_bad) break;
    const double r = s_piv;
    for (int j = k + 1 + threadIdx.x; j < d; j += CT) S[k * d + j] /= r;
    __syncthreads();
    const int m = d - k - 1;
    for (int e = threadIdx.x; e < m * m; e += CT) {
      const int i = k + 1 + e / m, j = k + 1 + e % m;
      if (i <= j) S[i * d + j] = fma(-S[k * d + i], S[k * d + j], S[i * d + j]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && info) info[slot] = s_bad;
  for (int e = threadIdx.x; e < d * d; e += CT) {
    const int i = e / d, j = e - i * d;
    R[e] = i <= j ? S[e] : 0.0;
  }
}

// Row-wise triangular solve X = A R^-1 (R upper, d x d) for a tall A (n x d): 64 rows per CTA
// staged through shared memory, one thread per row (forward substitution x_j = (a_j -
// sum_{k<j} x_k R_kj) / R_jj).  Writes X (if given) and/or the squared row norms of X (scores).
constexpr int TR_ROWS = 64;
__global__ void __launch_bounds__(TR_ROWS) trsm_rows_kernel(const double* __restrict__ A, int64_t n, int d,
                                                           const double* __restrict__ R, double* __restrict__ X,
                                                           double* __restrict__ sq) {
  extern __shared__ double S[];
  double* Rs = S;                          // d x d
  double* As = Rs + (size_t)d * d;         // TR_ROWS x (d + 1)
  const int ld = d + 1;
  const int64_t r0 = (int64_t)blockIdx.x * TR_ROWS;
  const int rows = (int)ks_min64(TR_ROWS, n - r0);
  for (int e = threadIdx.x; e < d * d; e += TR_ROWS) Rs[e] = R[e];
  for (int e = threadIdx.x; e < rows * d; e += TR_ROWS) {
    const int i = e / d, j = e - i * d;
    As[i * ld + j] = A[(r0 + i) * d + j];
  }
  __syncthreads();
  if (threadIdx.x < rows) {
    double* x = As + threadIdx.x * ld;  // solved in place
    double s2 = 0.0;
    for (int j = 0; j < d; j++) {
      // four independent partial sums (the chain over k is latency-bound otherwise)
      double a0 = x[j], a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int k = 0;
      for (; k + 4 <= j; k += 4) {
        a0 = fma(-x[k], Rs[k * d + j], a0);
        a1 = fma(-x[k + 1], Rs[(k + 1) * d + j], a1);
        a2 = fma(-x[k + 2], Rs[(k + 2) * d + j], a2);
        a3 = fma(-x[k + 3], Rs[(k + 3) * d + j], a3);
      }
      for (; k < j; k++) a0 = fma(-x[k], Rs[k * d + j], a0);
      const double acc = (a0 + a1) + (a2 + a3);
      const double v = acc / Rs[j * d + j];
      x[j] = v;
      s2 = fma(v, v, s2);
    }
    if (sq) sq[r0 + threadIdx.x] = s2;
  }
  __syncthreads();
  if (X)
    for (int e = threadIdx.x; e < rows * d; e += TR_ROWS) {
      const int i = e / d, j = e - i * d;
      X[(r0 + i) * d + j] = As[i * ld + j];
    }
}

int chol_upper(cudaStream_t st, const double* G, int d, double* R, int32_t* info, int slot) {
  const size_t smem = (size_t)d * d * sizeof(double);
  KS_TRY_CUDA(cudaFuncSetAttribute(chol_upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  chol_upper_kernel<<<1, CT, smem, st>>>(G, d, R, info, slot);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

int trsm_rows(cudaStream_t st, const double* A, int64_t n, int d, const double* R, double* X, double* sq) {
  const size_t smem = sizeof(double) * ((size_t)d * d + (size_t)TR_ROWS * (d + 1));
  KS_REQUIRE(smem <= 227 * 1024, KS_ESIZE, "trsm_rows: d = %d too large", d);
  KS_TRY_CUDA(cudaFuncSetAttribute(trsm_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  trsm_rows_kernel<<<ceil_div_u(n, TR_ROWS), TR_ROWS, smem, st>>>(A, n, d, R, X, sq);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

}  // namespace

namespace ks {

// R (d x d, upper) of A (n x d) by CholeskyQR2.  *ok (host) = 1 on success, 0 if A is too
// ill-conditioned for it (R is then undefined; use Householder).  Synchronises the stream.
int chol_qr2_r(cudaStream_t st, const double* A, int64_t n, int d, double* R, int* ok) {
  KS_REQUIRE(d >= 1 && d <= 128 && n >= d, KS_ESIZE, "chol_qr2 needs n >= d, d <= 128");
  Scratch<double> G((int64_t)d * d, st), R1((int64_t)d * d, st), R2((int64_t)d * d, st), Q((int64_t)n * d, st);
  Scratch<int32_t> info(2, st);
  KS_REQUIRE(G.p && R1.p && R2.p && Q.p && info.p, KS_ECUDA, "scratch allocation failed");
  int rc = gemm_tn_tall(st, d, d, n, 1.0, A, d, 1, A, d, 1, G.p);
  if (rc) return rc;
  if ((rc = chol_upper(st, G.p, d, R1.p, info.p, 0))) return rc;
  if ((rc = trsm_rows(st, A, n, d, R1.p, Q.p, nullptr))) return rc;
  if ((rc = gemm_tn_tall(st, d, d, n, 1.0, Q.p, d, 1, Q.p, d, 1, G.p))) return rc;
  if ((rc = chol_upper(st, G.p, d, R2.p, info.p, 1))) return rc;
  // R = R2 R1 (both upper)
  if ((rc = gemm(st, d, d, d, 1.0, R2.p, d, 1, 0, R1.p, d, 1, 0, 0.0, R, d, 1, 0, 1))) return rc;
  int32_t h[2];
  KS_TRY_CUDA(cudaMemcpyAsync(h, info.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  KS_TRY_CUDA(cudaStreamSynchronize(st));
  *ok = (h[0] == 0 && h[1] == 0);
  return KS_OK;
}

}  // namespace ks

// scores[i] = ||(A R^-1)_i||^2 = a_i^T (A^T A)^-1 a_i with R from CholeskyQR2: the statistical
// leverage scores of a numerically full-rank tall A (ridge_leverage_scores(compact_svd(a), 0),
// leverage.py:51-64).  *ok = 0 (scores undefined) when A is too ill-conditioned; callers then
// use the compact-SVD path.  Synchronises the stream.
extern "C" int ks_leverage_scores_tall(const double* A, int64_t n, int32_t d, double* scores, int32_t* ok,
                                       void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_REQUIRE(d >= 1 && d <= 128 && n >= d, KS_ESIZE, "leverage_scores_tall needs n >= d, 1 <= d <= 128");
  ks::Scratch<double> R((int64_t)d * d, st);
  KS_REQUIRE(R.p, KS_ECUDA, "scratch allocation failed");
  int good = 0;
  int rc = ks::chol_qr2_r(st, A, n, d, R.p, &good);
  if (rc) return rc;
  *ok = good;
  if (!good) return KS_OK;
  return trsm_rows(st, A, n, d, R.p, nullptr, scores);
}

// R factor by CholeskyQR2 (ok = 1) -- exported for tests and the compact SVD.
extern "C" int ks_chol_qr2_r(const double* A, int64_t n, int32_t d, double* R, int32_t* ok, void* stream) {
  int good = 0;
  int rc = ks::chol_qr2_r((cudaStream_t)stream, A, n, d, R, &good);
  *ok = good;
  return rc;
}
