// CholeskyQR2 for tall factor matrices (n >> d, d <= 128) and leverage scores from it.
//
// The R factor of A (reference: the QR inside tensor.compact_svd, tensor.py:76-107, LAPACK
// Householder) is computed as R = R2 R1 with R1 = chol(A^T A), Q1 = A R1^-1, R2 = chol(Q1^T Q1):
// two Gram passes on the FP64 tensor pipe (ks_gemm_tn_tall) and one streaming product with R1^-1,
// instead of a latency-bound Householder TSQR.  R is unique up to row signs; every consumer (the
// one-sided Jacobi SVD of R, U = A V Sigma^-1, scores) is invariant to them.  CholeskyQR2 is
// backward stable like Householder for kappa(A) below ~1e6; a Cholesky pivot that is not
// comfortably positive (ill-conditioned or rank-deficient A) reports failure and the caller falls
// back to Householder TSQR (ks_qr_r).
//
// Statistical leverage scores (ridge_leverage_scores(compact_svd(a), 0), leverage.py:51-64) of a
// numerically full-rank A are the squared row norms of A R^-1; ks_leverage_scores_tall fuses the
// product and the row norms in one pass.
#include "ks_common.cuh"
#include "ks_tma.cuh"

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
// shared memory) and, if asked, its inverse (upper) by column-parallel back substitution.
// info[slot] = k + 1 if pivot k is below tol * max diag (not comfortably positive definite).
__global__ void __launch_bounds__(CT) chol_upper_kernel(const double* __restrict__ G, int d, double* __restrict__ R,
                                                       double* __restrict__ Rinv, int32_t* __restrict__ info,
                                                       int slot, int near_identity) {
  extern __shared__ double S[];      // d x d (row-major, upper triangle used), then row k / packed R^-1
  double* W = S + (size_t)d * d;
  __shared__ int s_bad;
  __shared__ double s_dmax;
  __shared__ double s_emax[CT / 32];
  if (near_identity) {  // the closed form of chol_reg_kernel for G = I + E, |E| <= 1e-8
    double em = 0.0;
    for (int e = threadIdx.x; e < d * d; e += CT) {
      const int i = e / d, j = e % d;
      em = fmax(em, fabs(0.5 * (G[i * d + j] + G[j * d + i]) - (i == j ? 1.0 : 0.0)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) em = fmax(em, __shfl_xor_sync(0xffffffffu, em, o));
    if ((threadIdx.x & 31) == 0) s_emax[threadIdx.x >> 5] = em;
    __syncthreads();
    em = 0.0;
    for (int w = 0; w < CT / 32; w++) em = fmax(em, s_emax[w]);
    if (em <= 1e-8) {
      for (int e = threadIdx.x; e < d * d; e += CT) {
        const int i = e / d, j = e % d;
        const double ev = 0.5 * (G[i * d + j] + G[j * d + i]) - (i == j ? 1.0 : 0.0);
        const double up = i < j ? ev : (i == j ? 0.5 * ev : 0.0);
        R[e] = (i == j ? 1.0 : 0.0) + up;
        if (Rinv) Rinv[e] = (i == j ? 1.0 : 0.0) - up;
      }
      if (threadIdx.x == 0 && info) info[slot] = 0;
      return;
    }
  }
  for (int e = threadIdx.x; e < d * d; e += CT) {
    const int i = e / d, j = e - i * d;
    S[e] = i <= j ? 0.5 * (G[i * d + j] + G[j * d + i]) : 0.0;
  }
  if (threadIdx.x == 0) {
    s_bad = 0;
    double m = 0.0;
    for (int i = 0; i < d; i++) m = fmax(m, G[i * d + i]);
    s_dmax = m;
  }
  __syncthreads();
  const double tol = 1e-12 * s_dmax;  // kappa(A)^2 below ~1e12: the CholeskyQR2 regime
  for (int k = 0; k < d; k++) {
    const double p = S[k * d + k];    // every thread reads the pivot: no broadcast step
    if (!(p > tol) || !isfinite(p)) {
      if (threadIdx.x == 0) s_bad = k + 1;
      break;
    }
    const double r = sqrt(p);
    for (int j = k + threadIdx.x; j < d; j += CT) W[j] = (j == k) ? r : S[k * d + j] / r;
    __syncthreads();
    for (int j = k + threadIdx.x; j < d; j += CT) S[k * d + j] = W[j];
    const int m = d - k - 1;
    for (int e = threadIdx.x; e < m * m; e += CT) {
      const int i = k + 1 + e / m, j = k + 1 + e % m;
      if (i <= j) S[i * d + j] = fma(-W[i], W[j], S[i * d + j]);
    }
    __syncthreads();
  }
  __syncthreads();
  const int bad = s_bad;
  if (threadIdx.x == 0 && info) info[slot] = bad;
  for (int e = threadIdx.x; e < d * d; e += CT) {
    const int i = e / d, j = e - i * d;
    R[e] = i <= j ? S[e] : 0.0;
  }
  if (!Rinv || bad) return;
  // column j of R^-1 (one thread per column) in packed upper-triangular shared memory after S:
  // X_jj = 1 / R_jj, X_ij = -(sum_{k=i+1..j} R_ik X_kj) / R_ii for i < j; X(k, j) at P[k d - k(k-1)/2 + j - k]
  double* P = S + (size_t)d * d;
  auto po = [d](int k, int j) { return k * d - (k * (k - 1)) / 2 + (j - k); };
  for (int j = threadIdx.x; j < d; j += CT) {
    P[po(j, j)] = 1.0 / S[j * d + j];
    for (int i = j - 1; i >= 0; i--) {
      double a0 = 0.0, a1 = 0.0;
      int k = i + 1;
      for (; k + 2 <= j + 1; k += 2) {
        a0 = fma(S[i * d + k], P[po(k, j)], a0);
        a1 = fma(S[i * d + k + 1], P[po(k + 1, j)], a1);
      }
      for (; k <= j; k++) a0 = fma(S[i * d + k], P[po(k, j)], a0);
      P[po(i, j)] = -(a0 + a1) / S[i * d + i];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < d * d; e += CT) {
    const int i = e / d, j = e - i * d;
    Rinv[e] = i <= j ? P[po(i, j)] : 0.0;
  }
}

// X = A B for a tall A (n x d) and a small B (d x d): tm rows of A and all of B staged in shared
// memory, every thread computes independent dot products.  Writes X (if given) and/or the
// squared row norms of X (sq).
__global__ void __launch_bounds__(CT) tallmm_kernel(const double* __restrict__ A, int64_t n, int d, int tm,
                                                   const double* __restrict__ B, double* __restrict__ X,
                                                   double* __restrict__ sq) {
  extern __shared__ double S[];
  double* Bs = S;                           // d x d
  double* As = Bs + (size_t)d * d;          // tm x (d + 1)
  double* Xs = As + (size_t)tm * (d + 1);   // tm x (d + 1)
  const int ld = d + 1;
  const int64_t r0 = (int64_t)blockIdx.x * tm;
  const int rows = (int)ks_min64(tm, n - r0);
  for (int e = threadIdx.x; e < d * d; e += CT) Bs[e] = B[e];
  for (int e = threadIdx.x; e < rows * d; e += CT) {
    const int i = e / d, j = e - i * d;
    As[i * ld + j] = A[(r0 + i) * d + j];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < rows * d; e += CT) {
    const int i = e / d, j = e - i * d;
    const double* a = As + i * ld;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int k = 0;
    for (; k + 4 <= d; k += 4) {
      a0 = fma(a[k], Bs[k * d + j], a0);
      a1 = fma(a[k + 1], Bs[(k + 1) * d + j], a1);
      a2 = fma(a[k + 2], Bs[(k + 2) * d + j], a2);
      a3 = fma(a[k + 3], Bs[(k + 3) * d + j], a3);
    }
    for (; k < d; k++) a0 = fma(a[k], Bs[k * d + j], a0);
    const double v = (a0 + a1) + (a2 + a3);
    if (X) X[(r0 + i) * d + j] = v;
    Xs[i * ld + j] = v;
  }
  if (!sq) return;
  __syncthreads();
  for (int i = threadIdx.x; i < rows; i += CT) {
    double s2 = 0.0;
    for (int j = 0; j < d; j++) s2 = fma(Xs[i * ld + j], Xs[i * ld + j], s2);
    sq[r0 + i] = s2;
  }
}

// Upper Cholesky factor R of a d x d Gram (d = 16 TBS) and optionally R^-1, register-resident:
// thread (bi, bj) of a 16 x 16 grid owns the TBS x TBS block (rows bi TBS.., columns bj TBS..).
// Right-looking, one barrier per step: at step k every thread reads the published column k
// (updated through step k-1), forms r = sqrt(a_kk) and l_ik = a_ik / r for its rows and columns,
// applies a_ij -= l_ik l_jk to its lower-triangle entries and, if it owns column k + 1, publishes it
// for the next step.  R^-1 by the row-oriented right-looking back substitution (one barrier per
// row).  The same pivot test as chol_upper_kernel (info = k + 1 if pivot k <= 1e-12 max diag).
template <int TBS>
__global__ void __launch_bounds__(CT) chol_reg_kernel(const double* __restrict__ G, double* __restrict__ R,
                                                     double* __restrict__ Rinv, int32_t* __restrict__ info,
                                                     int slot, int near_identity) {
  constexpr int d = 16 * TBS, LDR = d + 1;
  extern __shared__ double rsm[];
  double* Rs = rsm;                // d x LDR: R (upper)
  double* colb = Rs + d * LDR;     // 2 x d: published column / X row
  __shared__ int s_bad;
  __shared__ double s_dmax;
  __shared__ double s_emax[CT / 32];
  const int tid = threadIdx.x, bi = tid >> 4, bj = tid & 15;
  const int i0 = bi * TBS, j0 = bj * TBS;
  if (near_identity) {
    // CholeskyQR2's second Gram Q1^T Q1 = I + E with E ~ kappa(A)^2 eps: chol(I + E) =
    // I + strict_upper(E) + diag(E) / 2 + O(|E|^2) and its inverse I - strict_upper(E) - diag(E) / 2
    // + O(|E|^2), exact to rounding once |E| <= 1e-8; otherwise the factorisation below
    for (int e = tid; e < d * d; e += CT) Rs[(e / d) * LDR + (e % d)] = G[e];  // coalesced, then transposed reads
    __syncthreads();
    double em = 0.0;
    for (int e = tid; e < d * d; e += CT) {
      const int i = e / d, j = e % d;
      em = fmax(em, fabs(0.5 * (Rs[i * LDR + j] + Rs[j * LDR + i]) - (i == j ? 1.0 : 0.0)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) em = fmax(em, __shfl_xor_sync(0xffffffffu, em, o));
    if ((tid & 31) == 0) s_emax[tid >> 5] = em;
    __syncthreads();
    em = 0.0;
    for (int w = 0; w < CT / 32; w++) em = fmax(em, s_emax[w]);
    if (em <= 1e-8) {
      for (int e = tid; e < d * d; e += CT) {
        const int i = e / d, j = e % d;
        const double ev = 0.5 * (Rs[i * LDR + j] + Rs[j * LDR + i]) - (i == j ? 1.0 : 0.0);
        const double up = i < j ? ev : (i == j ? 0.5 * ev : 0.0);
        R[e] = (i == j ? 1.0 : 0.0) + up;
        if (Rinv) Rinv[e] = (i == j ? 1.0 : 0.0) - up;
      }
      if (tid == 0 && info) info[slot] = 0;
      return;
    }
  }
  double a[TBS][TBS];
#pragma unroll
  for (int r = 0; r < TBS; r++)
#pragma unroll
    for (int c = 0; c < TBS; c++) {
      const int i = i0 + r, j = j0 + c;
      a[r][c] = i >= j ? 0.5 * (G[i * d + j] + G[j * d + i]) : 0.0;
    }
  if (tid == 0) {
    s_bad = 0;
    double m = 0.0;
    for (int i = 0; i < d; i++) m = fmax(m, G[i * d + i]);
    s_dmax = m;
  }
  for (int e = tid; e < d * LDR; e += CT) Rs[e] = 0.0;
  if (j0 == 0)  // column 0 published by its owners
#pragma unroll
    for (int r = 0; r < TBS; r++) colb[i0 + r] = a[r][0];
  __syncthreads();
  const double tol = 1e-12 * s_dmax;
  for (int k = 0; k < d; k++) {
    const double* pc = colb + (k & 1) * d;
    const double p = pc[k];
    if (!(p > tol) || !isfinite(p)) {
      if (tid == 0) s_bad = k + 1;
      break;
    }
    const double rr = sqrt(p), ri = 1.0 / rr;
    double lr[TBS], lc[TBS];
#pragma unroll
    for (int r = 0; r < TBS; r++) lr[r] = i0 + r > k ? pc[i0 + r] * ri : 0.0;
#pragma unroll
    for (int c = 0; c < TBS; c++) lc[c] = j0 + c > k ? pc[j0 + c] * ri : 0.0;
    if (bi == (k / TBS) ) {  // one row of threads writes row k of R: R[k][j] = l_jk (j > k), R[k][k] = r
#pragma unroll
      for (int c = 0; c < TBS; c++) {
        const int j = j0 + c;
        if (j > k) Rs[k * LDR + j] = lc[c];
      }
      if (bj == 0) Rs[k * LDR + k] = rr;
    }
#pragma unroll
    for (int r = 0; r < TBS; r++)  // (entries above the diagonal are updated too: never published)
#pragma unroll
      for (int c = 0; c < TBS; c++) a[r][c] = fma(-lr[r], lc[c], a[r][c]);
    if (k + 1 < d && k + 1 >= j0 && k + 1 < j0 + TBS) {  // publish column k + 1 (rows >= k + 1)
      const int cc = k + 1 - j0;
#pragma unroll
      for (int r = 0; r < TBS; r++) {
        double v = a[r][0];  // select column cc without indexing the register block dynamically
#pragma unroll
        for (int c = 1; c < TBS; c++) v = cc == c ? a[r][c] : v;
        if (i0 + r >= k + 1) colb[((k + 1) & 1) * d + i0 + r] = v;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  const int bad = s_bad;
  if (tid == 0 && info) info[slot] = bad;
  for (int e = tid; e < d * d; e += CT) R[e] = Rs[(e / d) * LDR + (e % d)];
  if (!Rinv || bad) return;
  // X = R^-1 (upper) by 16 x 16 blocks: the diagonal blocks inverted concurrently (one lane per
  // column, back substitution), then the off-diagonal blocks by block diagonals,
  // X_ij = -X_ii (sum_{i<k<=j} R_ik X_kj), two small block products per diagonal with a barrier
  // between -- log-depth in the block count instead of one barrier per row
  constexpr int NBK = d / 16;
  double* Xs = colb + 2 * d;            // d x LDR: X
  double* Ts = Xs + d * LDR;            // (NBK - 1) x 256: the block sums of one diagonal
  {
    const int wq = tid >> 5, ln = tid & 31;
    if (wq < NBK && ln < 16) {          // warp wq inverts diagonal block wq, lane ln = column
      const int o = wq * 16, j = ln;
      for (int i = 15; i >= 0; i--) {
        double acc = i == j ? 1.0 : 0.0;
        for (int k = i + 1; k <= j; k++) acc = fma(-Rs[(o + i) * LDR + o + k], Xs[(o + k) * LDR + o + j], acc);
        Xs[(o + i) * LDR + o + j] = i <= j ? acc / Rs[(o + i) * LDR + o + i] : 0.0;
      }
    }
    // zero the blocks below the diagonal and the upper off-diagonal blocks (filled below)
    for (int e = tid; e < d * d; e += CT) {
      const int i = e / d, j = e % d;
      if (i / 16 != j / 16) Xs[i * LDR + j] = 0.0;
    }
    __syncthreads();
    for (int dl = 1; dl < NBK; dl++) {
      const int np = NBK - dl;          // block pairs (i, i + dl) on this diagonal
      for (int e = tid; e < np * 256; e += CT) {  // T = sum_{i<k<=j} R_ik X_kj
        const int pr = e >> 8, rr = (e >> 4) & 15, cc = e & 15;
        const int bi_ = pr, bj_ = pr + dl;
        double acc = 0.0;
        for (int k = (bi_ + 1) * 16; k < (bj_ + 1) * 16; k++)
          acc = fma(Rs[(bi_ * 16 + rr) * LDR + k], Xs[k * LDR + bj_ * 16 + cc], acc);
        Ts[e] = acc;
      }
      __syncthreads();
      for (int e = tid; e < np * 256; e += CT) {  // X_ij = -X_ii T
        const int pr = e >> 8, rr = (e >> 4) & 15, cc = e & 15;
        const int bi_ = pr, bj_ = pr + dl;
        double acc = 0.0;
        for (int k = rr; k < 16; k++) acc = fma(Xs[(bi_ * 16 + rr) * LDR + bi_ * 16 + k], Ts[(pr << 8) + (k << 4) + cc], acc);
        Xs[(bi_ * 16 + rr) * LDR + bj_ * 16 + cc] = -acc;
      }
      __syncthreads();
    }
    for (int e = tid; e < d * d; e += CT) Rinv[e] = Xs[(e / d) * LDR + (e % d)];
  }
}

// X = A B (A n x D row-major, B D x D) on the FP64 tensor pipe: 64-row blocks of A and all of B
// staged with 16-byte cp.async, m16n8k4 tiles (each warp one m-tile and D / 16 n-tiles), X
// written from the fragments and / or the squared row norms (per-row partials summed in a fixed
// order: lanes, then the two warps sharing the m-tile).
template <int D>
__global__ void __launch_bounds__(CT) tallmm_dmma_kernel(const double* __restrict__ A, int64_t n,
                                                        const double* __restrict__ B, double* __restrict__ X,
                                                        double* __restrict__ sq) {
  constexpr int TMR = 64, LD = D + 4, NTW = D / 16;  // rows per block, smem stride, n-tiles per warp
  extern __shared__ __align__(16) double tsmm[];
  double* Bs = tsmm;          // D x LD
  double* As = Bs + D * LD;   // TMR x LD
  __shared__ double rsq[2][TMR];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  const int64_t r0 = (int64_t)blockIdx.x * TMR;
  auto cp16 = [](void* dst, const void* src, bool ok) {
    const unsigned dd = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dd), "l"(src), "r"(ok ? 16 : 0) : "memory");
  };
  for (int e = tid; e < D * (D / 2); e += CT) {
    const int k = e / (D / 2), c = 2 * (e % (D / 2));
    cp16(&Bs[k * LD + c], B + k * D + c, true);
  }
  for (int e = tid; e < TMR * (D / 2); e += CT) {
    const int i = e / (D / 2), c = 2 * (e % (D / 2));
    const bool ok = r0 + i < n;
    cp16(&As[i * LD + c], ok ? A + (r0 + i) * D + c : A, ok);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int mt = warp & 3, half = warp >> 2, m0 = mt * 16;
  double acc[NTW][4];
#pragma unroll
  for (int t = 0; t < NTW; t++) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.0;
#pragma unroll 4
  for (int k = 0; k < D / 4; k++) {
    const double a0 = As[(m0 + g) * LD + 4 * k + t4], a1 = As[(m0 + g + 8) * LD + 4 * k + t4];
#pragma unroll
    for (int t = 0; t < NTW; t++) {
      const int n0 = (half * NTW + t) * 8;
      dmma_16x8x4(acc[t], a0, a1, Bs[(4 * k + t4) * LD + n0 + g]);
    }
  }
  const int64_t ra = r0 + m0 + g, rb = ra + 8;
  if (X) {
#pragma unroll
    for (int t = 0; t < NTW; t++) {
      const int c = (half * NTW + t) * 8 + 2 * t4;
      if (ra < n) *reinterpret_cast<double2*>(&X[ra * D + c]) = make_double2(acc[t][0], acc[t][1]);
      if (rb < n) *reinterpret_cast<double2*>(&X[rb * D + c]) = make_double2(acc[t][2], acc[t][3]);
    }
  }
  if (!sq) return;
  double sa = 0.0, sb = 0.0;
#pragma unroll
  for (int t = 0; t < NTW; t++) {
    sa = fma(acc[t][1], acc[t][1], fma(acc[t][0], acc[t][0], sa));
    sb = fma(acc[t][3], acc[t][3], fma(acc[t][2], acc[t][2], sb));
  }
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  if (t4 == 0) {
    rsq[half][m0 + g] = sa;
    rsq[half][m0 + g + 8] = sb;
  }
  __syncthreads();
  for (int i = tid; i < TMR; i += CT)
    if (r0 + i < n) sq[r0 + i] = rsq[0][i] + rsq[1][i];
}

template <int D>
int launch_tallmm_dmma(cudaStream_t st, const double* A, int64_t n, const double* B, double* X, double* sq) {
  const size_t smem = sizeof(double) * (size_t)(D + 64) * (D + 4);
  KS_TRY_CUDA(cudaFuncSetAttribute(tallmm_dmma_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tallmm_dmma_kernel<D><<<ceil_div_u(n, 64), CT, smem, st>>>(A, n, B, X, sq);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

int chol_upper(cudaStream_t st, const double* G, int d, double* R, double* Rinv, int32_t* info, int slot,
               int near_identity = 0) {
  // register-resident factor for d = 32 / 64 (at d = 128 the 8 x 8 blocks per thread run slower
  // than the shared-memory kernel)
  if (!ks::env(ks::ENV_TALL_OLD) && (d == 32 || d == 64)) {
    // R, the published column, X = R^-1 and the block sums of one diagonal of X
    const size_t smem = sizeof(double) * (2 * (size_t)d * (d + 1) + 2 * d + (size_t)(d / 16) * 256);
#define KS_CHOL(TB)                                                                                            \
    if (d == 16 * TB) {                                                                                        \
      KS_TRY_CUDA(cudaFuncSetAttribute(chol_reg_kernel<TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
      chol_reg_kernel<TB><<<1, CT, smem, st>>>(G, R, Rinv, info, slot, near_identity);                         \
      KS_CHECK_LAUNCH();                                                                                       \
      return KS_OK;                                                                                            \
    }
    KS_CHOL(2) KS_CHOL(4)
#undef KS_CHOL
  }
  const size_t smem = ((size_t)d * d + (size_t)d * (d + 1) / 2 + d) * sizeof(double);
  KS_TRY_CUDA(cudaFuncSetAttribute(chol_upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  chol_upper_kernel<<<1, CT, smem, st>>>(G, d, R, Rinv, info, slot, near_identity);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

int tallmm(cudaStream_t st, const double* A, int64_t n, int d, const double* B, double* X, double* sq) {
  if (!ks::env(ks::ENV_TALL_OLD) && (((uintptr_t)A | (uintptr_t)B | (uintptr_t)X) & 15) == 0) {
    if (d == 16) return launch_tallmm_dmma<16>(st, A, n, B, X, sq);
    if (d == 32) return launch_tallmm_dmma<32>(st, A, n, B, X, sq);
    if (d == 64) return launch_tallmm_dmma<64>(st, A, n, B, X, sq);
    if (d == 128) return launch_tallmm_dmma<128>(st, A, n, B, X, sq);
  }
  const int tm = d > 64 ? 32 : 64;
  const size_t smem = sizeof(double) * ((size_t)d * d + 2 * (size_t)tm * (d + 1));
  KS_REQUIRE(smem <= 227 * 1024, KS_ESIZE, "tallmm: d = %d too large", d);
  KS_TRY_CUDA(cudaFuncSetAttribute(tallmm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tallmm_kernel<<<ceil_div_u(n, tm), CT, smem, st>>>(A, n, d, tm, B, X, sq);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

}  // namespace

namespace ks {

// R (d x d, upper) of A (n x d) by CholeskyQR2, and R^-1 if Rinv is given.  *ok (host) = 1 on
// success, 0 if A is too ill-conditioned (R undefined; use Householder).  Synchronises the stream.
// Asynchronous form: info_dev (device, 2 x int32) receives the two factorisations' status words
// (nonzero = CholeskyQR2 declined; R / Rinv are then undefined).
int chol_qr2_r_async(cudaStream_t st, const double* A, int64_t n, int d, double* R, double* Rinv,
                     int32_t* info_dev) {
  KS_REQUIRE(d >= 1 && d <= 128 && n >= d, KS_ESIZE, "chol_qr2 needs n >= d, d <= 128");
  Scratch<double> G((int64_t)d * d, st), R1((int64_t)d * d, st), R1i((int64_t)d * d, st), R2((int64_t)d * d, st),
      R2i((int64_t)d * d, st), Q((int64_t)n * d, st);
  KS_REQUIRE(G.p && R1.p && R1i.p && R2.p && R2i.p && Q.p, KS_ECUDA, "scratch allocation failed");
  int rc = gemm_tn_tall(st, d, d, n, 1.0, A, d, 1, A, d, 1, G.p);
  if (rc) return rc;
  if ((rc = chol_upper(st, G.p, d, R1.p, R1i.p, info_dev, 0))) return rc;
  if ((rc = tallmm(st, A, n, d, R1i.p, Q.p, nullptr))) return rc;  // Q1 = A R1^-1
  if ((rc = gemm_tn_tall(st, d, d, n, 1.0, Q.p, d, 1, Q.p, d, 1, G.p))) return rc;
  if ((rc = chol_upper(st, G.p, d, R2.p, Rinv ? R2i.p : nullptr, info_dev, 1, 1))) return rc;
  if ((rc = gemm(st, d, d, d, 1.0, R2.p, d, 1, 0, R1.p, d, 1, 0, 0.0, R, d, 1, 0, 1))) return rc;
  if (Rinv && (rc = gemm(st, d, d, d, 1.0, R1i.p, d, 1, 0, R2i.p, d, 1, 0, 0.0, Rinv, d, 1, 0, 1))) return rc;
  return KS_OK;
}

int chol_qr2_r(cudaStream_t st, const double* A, int64_t n, int d, double* R, int* ok, double* Rinv) {
  KS_REQUIRE(d >= 1 && d <= 128 && n >= d, KS_ESIZE, "chol_qr2 needs n >= d, d <= 128");
  Scratch<double> G((int64_t)d * d, st), R1((int64_t)d * d, st), R1i((int64_t)d * d, st), R2((int64_t)d * d, st),
      R2i((int64_t)d * d, st), Q((int64_t)n * d, st);
  Scratch<int32_t> info(2, st);
  KS_REQUIRE(G.p && R1.p && R1i.p && R2.p && R2i.p && Q.p && info.p, KS_ECUDA, "scratch allocation failed");
  int rc = gemm_tn_tall(st, d, d, n, 1.0, A, d, 1, A, d, 1, G.p);
  if (rc) return rc;
  if ((rc = chol_upper(st, G.p, d, R1.p, R1i.p, info.p, 0))) return rc;
  if ((rc = tallmm(st, A, n, d, R1i.p, Q.p, nullptr))) return rc;  // Q1 = A R1^-1
  if ((rc = gemm_tn_tall(st, d, d, n, 1.0, Q.p, d, 1, Q.p, d, 1, G.p))) return rc;
  if ((rc = chol_upper(st, G.p, d, R2.p, Rinv ? R2i.p : nullptr, info.p, 1, 1))) return rc;
  // R = R2 R1 and R^-1 = R1^-1 R2^-1 (all upper triangular)
  if ((rc = gemm(st, d, d, d, 1.0, R2.p, d, 1, 0, R1.p, d, 1, 0, 0.0, R, d, 1, 0, 1))) return rc;
  if (Rinv && (rc = gemm(st, d, d, d, 1.0, R1i.p, d, 1, 0, R2i.p, d, 1, 0, 0.0, Rinv, d, 1, 0, 1))) return rc;
  int32_t h[2];
  KS_TRY_CUDA(cudaMemcpyAsync(h, info.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  KS_TRY_CUDA(cudaStreamSynchronize(st));
  *ok = (h[0] == 0 && h[1] == 0);
  return KS_OK;
}

}  // namespace ks

namespace {

// scores[i] = ||(Q1 R2^-1)_i||^2 with Q1 = A R1^-1 (the CholeskyQR2 first pass, kept) and R2 the
// second pass's factor: the same Q as A (R2 R1)^-1 without the two d x d products R2 R1 and
// R1^-1 R2^-1 (~13 us each as small-GEMM launches at d = 64).  info (device, 2 x int32): nonzero =
// declined, scores undefined.
int chol_qr2_scores(cudaStream_t st, const double* A, int64_t n, int d, double* scores, int32_t* info) {
  using ks::Scratch;
  Scratch<double> G((int64_t)d * d, st), R1((int64_t)d * d, st), R1i((int64_t)d * d, st), R2((int64_t)d * d, st),
      R2i((int64_t)d * d, st), Q((int64_t)n * d, st);
  KS_REQUIRE(G.p && R1.p && R1i.p && R2.p && R2i.p && Q.p, KS_ECUDA, "scratch allocation failed");
  // defined inputs of the last two products when a factorisation declines
  KS_TRY_CUDA(cudaMemsetAsync(R1i.p, 0, sizeof(double) * d * d, st));
  KS_TRY_CUDA(cudaMemsetAsync(R2i.p, 0, sizeof(double) * d * d, st));
  int rc = ks::gemm_tn_tall(st, d, d, n, 1.0, A, d, 1, A, d, 1, G.p);
  if (rc) return rc;
  if ((rc = chol_upper(st, G.p, d, R1.p, R1i.p, info, 0))) return rc;
  if ((rc = tallmm(st, A, n, d, R1i.p, Q.p, nullptr))) return rc;  // Q1 = A R1^-1
  if ((rc = ks::gemm_tn_tall(st, d, d, n, 1.0, Q.p, d, 1, Q.p, d, 1, G.p))) return rc;
  if ((rc = chol_upper(st, G.p, d, R2.p, R2i.p, info, 1, 1))) return rc;
  return tallmm(st, Q.p, n, d, R2i.p, nullptr, scores);
}

}  // namespace

// scores[i] = ||(A R^-1)_i||^2 = a_i^T (A^T A)^-1 a_i with R from CholeskyQR2: the statistical
// leverage scores of a numerically full-rank tall A (ridge_leverage_scores(compact_svd(a), 0),
// leverage.py:51-64).  *ok = 0 (scores undefined) when A is too ill-conditioned; callers then
// use the compact-SVD path.  Synchronises the stream.
extern "C" int ks_leverage_scores_tall(const double* A, int64_t n, int32_t d, double* scores, int32_t* ok,
                                       void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_REQUIRE(d >= 1 && d <= 128 && n >= d, KS_ESIZE, "leverage_scores_tall needs n >= d, 1 <= d <= 128");
  ks::Scratch<int32_t> info(2, st);
  KS_REQUIRE(info.p, KS_ECUDA, "scratch allocation failed");
  int rc = chol_qr2_scores(st, A, n, d, scores, info.p);
  if (rc) return rc;
  int32_t h[2];
  KS_TRY_CUDA(cudaMemcpyAsync(h, info.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  KS_TRY_CUDA(cudaStreamSynchronize(st));
  *ok = (h[0] == 0 && h[1] == 0);
  return KS_OK;
}

// Asynchronous ks_leverage_scores_tall: no host round trip; info_dev (device, 2 x int32, zeroed by
// the caller or not -- both words are written) nonzero = declined, scores undefined.
extern "C" int ks_leverage_scores_tall_async(const double* A, int64_t n, int32_t d, double* scores, int32_t* info_dev,
                                             void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_REQUIRE(d >= 1 && d <= 128 && n >= d, KS_ESIZE, "leverage_scores_tall needs n >= d, 1 <= d <= 128");
  return chol_qr2_scores(st, A, n, d, scores, info_dev);
}

// R factor by CholeskyQR2 (ok = 1) -- exported for tests; ks_qr_r uses it internally.
extern "C" int ks_chol_qr2_r(const double* A, int64_t n, int32_t d, double* R, int32_t* ok, void* stream) {
  int good = 0;
  int rc = ks::chol_qr2_r((cudaStream_t)stream, A, n, d, R, &good, nullptr);
  *ok = good;
  return rc;
}

