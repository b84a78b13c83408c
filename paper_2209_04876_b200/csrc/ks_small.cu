// Small dense linear algebra on device (d <= 128): Householder TSQR (R only), one-sided
// Jacobi SVD, thin SVD driver.  Replaces the LAPACK calls of the reference hot path:
// np.linalg.svd in tensor.compact_svd (tensor.py:76-107) and np.linalg.eigh in
// solvers.factor_gram (solvers.py:143-150).  No host LAPACK is used.
#include "ks_common.cuh"

#include <cstdlib>
#include <vector>
#include <algorithm>

namespace ks {
int gemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t a_rs, int64_t a_cs, int64_t a_bs, const double* B, int64_t b_rs, int64_t b_cs,
         int64_t b_bs, double beta, double* C, int64_t c_rs, int64_t c_cs, int64_t c_bs,
         int64_t batch);
}

namespace {

constexpr int QR_THREADS = 256;
__device__ int g_jacobi_sweeps[8];
constexpr size_t QR_SMEM_CAP = 200 * 1024;

// Householder QR of one panel of `rows` x d (rows <= prows) taken from src rows
// [blockIdx.x*prows, ...).  Writes the d x d upper-triangular R of the panel to
// dst + blockIdx.x*d*d (row-major, zero below the diagonal).  Panel storage is column-major
// (column j contiguous) either in shared memory or in a per-block global workspace.
template <bool SMEM>
__global__ void __launch_bounds__(QR_THREADS) qr_panel_kernel(const double* __restrict__ src,
                                                             int64_t n, int d, int prows,
                                                             double* __restrict__ dst,
                                                             double* __restrict__ gwork) {
  extern __shared__ double dyn[];
  __shared__ double red[32];
  __shared__ double s_tau, s_beta;
  const int64_t r0 = (int64_t)blockIdx.x * prows;
  const int rows = (int)ks_min64(prows, n - r0);
  double* P = SMEM ? dyn : gwork + (int64_t)blockIdx.x * prows * d;
  const int tid = threadIdx.x;
  for (int e = tid; e < rows * d; e += QR_THREADS) {
    const int i = e / d, j = e - i * d;
    P[(int64_t)j * rows + i] = src[(r0 + i) * d + j];
  }
  __syncthreads();
  const int steps = min(rows, d);
  // threads per column group for the trailing update
  for (int j = 0; j < steps; j++) {
    double* x = P + (int64_t)j * rows;
    double part = 0.0;
    for (int i = j + 1 + tid; i < rows; i += QR_THREADS) part = fma(x[i], x[i], part);
    const double tail2 = block_sum(part, red);
    if (tid == 0) {
      const double alpha = x[j];
      if (tail2 == 0.0) {
        s_tau = 0.0;
        s_beta = alpha;
      } else {
        const double nrm = sqrt(fma(alpha, alpha, tail2));
        const double beta = alpha >= 0.0 ? -nrm : nrm;
        s_tau = (beta - alpha) / beta;
        s_beta = beta;
        x[j] = alpha - beta;  // v0 (unnormalised); scaled below
      }
    }
    __syncthreads();
    const double tau = s_tau;
    if (tau != 0.0) {
      const double inv_v0 = 1.0 / x[j];
      for (int i = j + 1 + tid; i < rows; i += QR_THREADS) x[i] *= inv_v0;
      __syncthreads();
      // trailing columns: w_k = v^T P[:,k]; P[:,k] -= tau w_k v  (v_j = 1)
      const int ncols = d - j - 1;
      if (ncols > 0) {
        const int gsz = max(1, min(32, QR_THREADS / ncols));  // power of two not required
        int g = 1;
        while (g * 2 <= gsz) g *= 2;
        const int ngroups = QR_THREADS / g;
        const int lane_g = tid % g;
        for (int c0 = tid / g; c0 < ncols; c0 += ngroups) {
          double* col = P + (int64_t)(j + 1 + c0) * rows;
          double w = 0.0;
          for (int i = j + 1 + lane_g; i < rows; i += g) w = fma(x[i], col[i], w);
          const unsigned gm = (g == 32) ? 0xffffffffu : (((1u << g) - 1u) << ((tid & 31) & ~(g - 1)));
          for (int o = g >> 1; o > 0; o >>= 1) w += __shfl_xor_sync(gm, w, o, g);
          w += col[j];
          const double tw = tau * w;
          if (lane_g == 0) col[j] -= tw;
          for (int i = j + 1 + lane_g; i < rows; i += g) col[i] = fma(-tw, x[i], col[i]);
        }
      }
    }
    __syncthreads();
    if (tid == 0) x[j] = s_beta;  // R diagonal
    __syncthreads();
  }
  double* R = dst + (int64_t)blockIdx.x * d * d;
  for (int e = tid; e < d * d; e += QR_THREADS) {
    const int i = e / d, j = e - i * d;
    R[e] = (i <= j && i < rows) ? P[(int64_t)j * rows + i] : 0.0;
  }
}

// One-sided (Hestenes) Jacobi SVD of a d x d matrix in one CTA.  W = M (column-major in
// smem), V = I; round-robin parallel ordering, one thread group per column pair.
// Output sigma descending, V row-major (column j = right singular vector j).
template <bool VSMEM>
__global__ void jacobi_svd_kernel(const double* __restrict__ M, int d, double* __restrict__ sigma,
                                  double* __restrict__ Vout, double* __restrict__ vwork) {
  extern __shared__ double dyn[];
  // batched: problem blockIdx.x of a contiguous batch
  M += (size_t)blockIdx.x * d * d;
  sigma += (size_t)blockIdx.x * d;
  Vout += (size_t)blockIdx.x * d * d;
  if (vwork) vwork += (size_t)blockIdx.x * (d + 1) * (d + 1);
  __shared__ int s_rot;
  __shared__ int s_order[130];
  __shared__ double s_norm[130];
  const int dp = d + (d & 1);
  double* W = dyn;                                      // dp columns x d rows
  double* V = VSMEM ? dyn + (size_t)dp * d : vwork;     // dp columns x dp rows
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < dp * d; e += nt) {
    const int j = e / d, i = e - j * d;
    W[e] = (j < d) ? M[(int64_t)i * d + j] : 0.0;
  }
  for (int e = tid; e < dp * dp; e += nt) {
    const int j = e / dp, i = e - j * dp;
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int npairs = dp / 2;
  // dot products carry ~d*eps relative rounding: a tighter threshold never converges
  const double tol = 2.0 * d * 2.220446049250313e-16;
  int g = 1;
  while (g * 2 * npairs <= nt && g < 32) g *= 2;
  const int group = tid / g, lg = tid % g;
  const bool active = group < npairs;
  const unsigned gmask = (g == 32) ? 0xffffffffu : (((1u << g) - 1u) << ((tid & 31) & ~(g - 1)));
  for (int sweep = 0; sweep < 40; sweep++) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int r = 0; r < dp - 1; r++) {
      if (active) {
        // circle method: position 0 fixed, others rotate
        auto player = [&](int pos) {
          int x = pos - 1 + r;  // < 2 (dp - 1): one conditional subtraction instead of a modulo
          if (x >= dp - 1) x -= dp - 1;
          return pos == 0 ? 0 : 1 + x;
        };
        const int p = player(group), q = player(dp - 1 - group);
        double* wp = W + (size_t)p * d;
        double* wq = W + (size_t)q * d;
        double a = 0.0, b = 0.0, c = 0.0;
        for (int i = lg; i < d; i += g) {
          const double x = wp[i], y = wq[i];
          a = fma(x, x, a);
          b = fma(y, y, b);
          c = fma(x, y, c);
        }
        for (int o = g >> 1; o > 0; o >>= 1) {
          a += __shfl_xor_sync(gmask, a, o, g);
          b += __shfl_xor_sync(gmask, b, o, g);
          c += __shfl_xor_sync(gmask, c, o, g);
        }
        // rotate unless the pair is orthogonal to working precision (dgesvj-style threshold)
        // (c^2 > tol^2 a b avoids two square roots on the serial path of every round)
        if (c != 0.0 && a != 0.0 && b != 0.0 && c * c > tol * tol * a * b) {
          // t only has to be close to tan(theta): any t gives an exact rotation as long as
          // cs = 1/sqrt(1+t^2) and sn = t cs are consistent, so t uses fast reciprocals and the
          // orthogonality-critical cs an accurate rsqrt.
          const double zeta = (b - a) * __drcp_rn(2.0 * c);
          const double az = fabs(zeta);
          const double tt = __drcp_rn(az + sqrt(fma(az, az, 1.0)));
          const double t = zeta >= 0.0 ? tt : -tt;
          const double cs = rsqrt(fma(t, t, 1.0));
          const double sn = cs * t;
          for (int i = lg; i < d; i += g) {
            const double x = wp[i], y = wq[i];
            wp[i] = cs * x - sn * y;
            wq[i] = sn * x + cs * y;
          }
          double* vp = V + (size_t)p * dp;
          double* vq = V + (size_t)q * dp;
          for (int i = lg; i < dp; i += g) {
            const double x = vp[i], y = vq[i];
            vp[i] = cs * x - sn * y;
            vq[i] = sn * x + cs * y;
          }
          if (lg == 0) s_rot = 1;
        }
      }
      __syncthreads();
    }
    if (tid == 0) g_jacobi_sweeps[blockIdx.x & 7] = sweep + 1;
    if (s_rot == 0) break;
    __syncthreads();
  }
  // singular values and descending order (ties broken by index -> deterministic)
  for (int j = tid; j < dp; j += nt) {
    double s = 0.0;
    if (j < d)
      for (int i = 0; i < d; i++) s = fma(W[(size_t)j * d + i], W[(size_t)j * d + i], s);
    s_norm[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < d; j += nt) {
    int rank = 0;
    // total order even for non-finite input (NaN ranks last): every rank is assigned exactly once
    const double sj = isnan(s_norm[j]) ? -1.0 : s_norm[j];
    for (int k = 0; k < d; k++) {
      const double sk = isnan(s_norm[k]) ? -1.0 : s_norm[k];
      rank += (sk > sj) || (sk == sj && k < j);
    }
    s_order[rank] = j;
  }
  __syncthreads();
  for (int k = tid; k < d; k += nt) sigma[k] = s_norm[s_order[k]];
  for (int e = tid; e < d * d; e += nt) {
    const int i = e / d, k = e - i * d;
    Vout[e] = V[(size_t)s_order[k] * dp + i];
  }
}

// Fixed-size variant (D = 16, 32, 64) of the one-sided Jacobi above: 8 threads per column pair,
// every loop unrolled, the pair's column slices kept in registers between the dot products and
// the rotation, constant-width shuffles.  Column j is stored rotated by 8 elements when j is odd
// so the two pairs sharing a half-warp hit disjoint banks.  SYM: read 0.5 (M + M^T) (the
// reference symmetrises the Gram before eigh).  Ms: optional per-problem pointers.
constexpr int JF_G = 8;
struct MatPtrs {
  const double* p[8];
};

// column j of W / V at stride D + 8: the two pairs sharing a half-warp (consecutive players,
// opposite parity) land 16 banks apart, and element offsets are compile-time immediates
template <int D>
__device__ __forceinline__ int jf_off(int j, int i) {
  return j * (D + 8) + i;
}

// C = A B for D x D operands in shared memory with NT = D / 2 * JF_G threads: thread t owns row
// i = t % D (consecutive across a warp: conflict-free A reads) and NJ = D * D / NT consecutive
// columns (the same for the whole warp: B reads are broadcasts).  a(i, k), b(k, j) are loaders.
template <int D, class LA, class LB, class Out>
__device__ __forceinline__ void smem_gemm_rows(LA a, LB b, Out out) {
  constexpr int NT = D / 2 * JF_G, NJ = D * D / NT;
  const int i = threadIdx.x % D, j0 = (threadIdx.x / D) * NJ;
  double c[NJ];
#pragma unroll
  for (int q = 0; q < NJ; q++) c[q] = 0.0;
#pragma unroll 2
  for (int k = 0; k < D; k++) {
    const double x = a(i, k);
#pragma unroll
    for (int q = 0; q < NJ; q++) c[q] = fma(x, b(k, j0 + q), c[q]);
  }
#pragma unroll
  for (int q = 0; q < NJ; q++) out(i, j0 + q, c[q]);
}

// C = A B for D x D operands in shared memory, TM x TN register blocks per thread (D = 64: 4 x 4,
// half the shared-memory instructions per FMA of smem_gemm_rows).  Thread (ib, jb) owns rows
// ib TM + r and columns jb + c (D / TN): consecutive lanes read consecutive columns of B (b(k, j)
// must be contiguous in j) and share their rows of A (broadcast reads).
template <int D, class LA, class LB, class Out>
__device__ __forceinline__ void smem_gemm_blk(LA a, LB b, Out out) {
  constexpr int NT = D / 2 * JF_G, PER = D * D / NT;
  constexpr int TM = D >= 64 ? 4 : 2, TN = PER / TM, NJB = D / TN;
  static_assert(TM * TN == PER && (D / TM) * NJB == NT, "gemm blocking");
  const int jb = threadIdx.x % NJB, ib = threadIdx.x / NJB;
  double c[TM][TN];
#pragma unroll
  for (int r = 0; r < TM; r++)
#pragma unroll
    for (int q = 0; q < TN; q++) c[r][q] = 0.0;
#pragma unroll 4
  for (int k = 0; k < D; k++) {
    double av[TM], bv[TN];
#pragma unroll
    for (int r = 0; r < TM; r++) av[r] = a(ib * TM + r, k);
#pragma unroll
    for (int q = 0; q < TN; q++) bv[q] = b(k, jb + q * NJB);
#pragma unroll
    for (int r = 0; r < TM; r++)
#pragma unroll
      for (int q = 0; q < TN; q++) c[r][q] = fma(av[r], bv[q], c[r][q]);
  }
#pragma unroll
  for (int r = 0; r < TM; r++)
#pragma unroll
    for (int q = 0; q < TN; q++) out(ib * TM + r, jb + q * NJB, c[r][q]);
}

// FP32 prelude of the symmetric (Gram) eigensolve: `sweeps32` one-sided Jacobi sweeps in single
// precision (cheaper rounds: 32-bit shuffles, 4-cycle FMAs, MUFU rsqrt), then the accumulated
// rotations are re-orthonormalised in FP64 by two Newton-Schulz steps V <- V (3I - V^T V) / 2 and
// the FP64 sweeps restart from W = G V: the double-precision phase then starts close to the
// eigenbasis and converges in about half the sweeps (measured 5 instead of 9 at d = 64), to the
// same FP64 accuracy (the FP64 phase alone decides convergence).
template <int D, bool track_v>
__device__ void jacobi_fp32_prelude(const double* __restrict__ M, double* W, double* V, float* W32, float* V32,
                                    int sweeps32, bool want_w) {
  constexpr int NP = D / 2, NT = NP * JF_G, E = D / JF_G;
  __shared__ int s_rot32;
  const int tid = threadIdx.x;
  for (int e = tid; e < D * D; e += NT) {
    const int i = e / D, j = e % D;
    W32[jf_off<D>(j, i)] = (float)(0.5 * (M[i * D + j] + M[j * D + i]));
    V32[jf_off<D>(j, i)] = (i == j) ? 1.0f : 0.0f;
  }
  __syncthreads();
  const int group = tid / JF_G, lg = tid % JF_G;
  const float tol = 2.0f * D * 1.1920929e-7f;
  for (int sweep = 0; sweep < sweeps32; sweep++) {
    if (tid == 0) s_rot32 = 0;
    __syncthreads();
    for (int r = 0; r < D - 1; r++) {
      auto player = [&](int pos) {
        int x = pos - 1 + r;
        if (x >= D - 1) x -= D - 1;
        return pos == 0 ? 0 : 1 + x;
      };
      const int p = player(group), q = player(D - 1 - group);
      float x[E], y[E], u[E], v[E];
#pragma unroll
      for (int k = 0; k < E; k++) {
        x[k] = W32[jf_off<D>(p, lg + k * JF_G)];
        y[k] = W32[jf_off<D>(q, lg + k * JF_G)];
        if constexpr (track_v) {
          u[k] = V32[jf_off<D>(p, lg + k * JF_G)];
          v[k] = V32[jf_off<D>(q, lg + k * JF_G)];
        }
      }
      float a = 0.0f, b = 0.0f, c = 0.0f;
#pragma unroll
      for (int k = 0; k < E; k++) {
        a = fmaf(x[k], x[k], a);
        b = fmaf(y[k], y[k], b);
        c = fmaf(x[k], y[k], c);
      }
#pragma unroll
      for (int o = JF_G / 2; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
      }
      if (c != 0.0f && a != 0.0f && b != 0.0f && c * c > tol * tol * a * b) {
        const float x2 = b - a, y2 = 2.0f * c;
        const float qq = fmaf(x2, x2, y2 * y2);
        const float den = fmaf(qq, rsqrtf(qq), fabsf(x2));
        const float tt = __fdividef(y2, den);
        const float t = x2 >= 0.0f ? tt : -tt;
        const float cs = rsqrtf(fmaf(t, t, 1.0f));
        const float sn = cs * t;
#pragma unroll
        for (int k = 0; k < E; k++) {
          W32[jf_off<D>(p, lg + k * JF_G)] = cs * x[k] - sn * y[k];
          W32[jf_off<D>(q, lg + k * JF_G)] = sn * x[k] + cs * y[k];
          if constexpr (track_v) {
            V32[jf_off<D>(p, lg + k * JF_G)] = cs * u[k] - sn * v[k];
            V32[jf_off<D>(q, lg + k * JF_G)] = sn * u[k] + cs * v[k];
          }
        }
        if (lg == 0) s_rot32 = 1;
      }
      __syncthreads();
    }
    if (s_rot32 == 0) break;
    __syncthreads();
  }
  // V (FP64) = V32, then two Newton-Schulz steps and W = G V.  X (the FP32 buffers, D (D + 8)
  // doubles) and Y (D (D + 8) doubles after them) are scratch; every product below is laid out so
  // that a warp's threads read consecutive elements or one broadcast element (no bank conflicts).
  if constexpr (track_v) {
    for (int e = tid; e < D * D; e += NT) {
      const int j = e / D, i = e % D;
      V[jf_off<D>(j, i)] = (double)V32[jf_off<D>(j, i)];
    }
  } else {  // W = G V = V diag(lambda) at convergence, G positive semidefinite: V = W's normalised columns
    for (int j = tid; j < D; j += NT) {
      double nn = 0.0;
      for (int i = 0; i < D; i++) {
        const double x = (double)W32[jf_off<D>(j, i)];
        nn = fma(x, x, nn);
      }
      const double sc = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
      for (int i = 0; i < D; i++) V[jf_off<D>(j, i)] = nn > 0.0 ? sc * (double)W32[jf_off<D>(j, i)] : (i == j ? 1.0 : 0.0);
    }
  }
  double* X = reinterpret_cast<double*>(W32);
  double* Y = X + D * (D + 8);
  __syncthreads();
  constexpr int LD = D + 8;   // jf layout: V(i, j) = V[j * LD + i]
  constexpr int LT = D + 2;   // row-major transposed copy (even stride)
  for (int step = 0; step < 2; step++) {
    // X = V^T row-major: X[k * LT + i] = V(k, i)... stored as Xt(k, i) with k = row of V
    for (int e = tid; e < D * D; e += NT) {
      const int i = e / D, k = e % D;
      X[k * LT + i] = V[i * LD + k];
    }
    __syncthreads();
    // Y = C = 1.5 I - 0.5 V^T V: (V^T V)(i, j) = sum_k V(k, i) V(k, j) = sum_k X[k LT + i] X[k LT + j]
    smem_gemm_blk<D>([&](int i, int k) { return X[k * LT + i]; }, [&](int k, int j) { return X[k * LT + j]; },
                     [&](int i, int j, double v) { Y[i * D + j] = (i == j ? 1.5 : 0.0) - 0.5 * v; });
    __syncthreads();
    // X = V C (jf layout), then V = X
    smem_gemm_blk<D>([&](int i, int k) { return V[k * LD + i]; }, [&](int k, int j) { return Y[k * D + j]; },
                     [&](int i, int j, double v) { X[j * LD + i] = v; });
    __syncthreads();
    for (int e = tid; e < D * LD; e += NT) V[e] = X[e];
    __syncthreads();
  }
  if (!want_w) return;  // the refinement forms G V itself
  // Y = G (symmetrised, row-major), then W = G V
  for (int e = tid; e < D * D; e += NT) {
    const int i = e / D, k = e % D;
    Y[e] = 0.5 * (M[i * D + k] + M[k * D + i]);
  }
  __syncthreads();
  smem_gemm_rows<D>([&](int i, int k) { return Y[k * D + i]; }, [&](int k, int j) { return V[j * LD + k]; },
                    [&](int i, int j, double v) { W[j * LD + i] = v; });
  __syncthreads();
}

// Dominant-eigenpair deflation of a symmetric Gram matrix G (row-major, shared memory), before the
// Jacobi sweeps.  Gram matrices of factors whose columns share a large mean (BASELINE's
// N(1, 0.001) factors: one eigenvalue ~n d, the others ~n 1e-3) carry the small eigenvalues in the
// low bits of every entry, so the FP32 prelude cannot resolve them and the FP64 phase needs ~5
// sweeps.  When one eigenvalue dominates (power iteration from the all-ones vector converges to a
// residual ||G v - lam v|| <= 16 D eps lam, and ||G - lam v v^T||_F <= 1e-3 lam), G is replaced
// by H G H with the Householder reflector H = I - beta u u^T, H v = -sign(v_0) e_1, and the
// (rounding-level) off-diagonal entries of its first row and column are set to zero: the
// eigenvalues and eigenvectors change by O(||r||^2 / lam) and O(||r|| / lam) ~ 1e-16, far below
// the reference's own eigensolver rounding.  The sweeps then see a block-diagonal matrix whose
// small block is well scaled; the eigenvectors of G are H V.  Returns beta (0: not deflated) and
// leaves u in `u`.  All threads of the block call it.
template <int D>
__device__ double jacobi_deflate(double* G, double* u, double* v, double* w, double* red) {
  constexpr int NT = D / 2 * JF_G, TPR = NT / D;  // threads per row of a product
  static_assert(TPR * D == NT && (TPR & (TPR - 1)) == 0 && TPR <= 32, "row groups within a warp");
  const int tid = threadIdx.x, row = tid / TPR, part = tid % TPR;
  auto matvec = [&](const double* x, double* y) {  // y = G x
    double t = 0.0;
    for (int k = part; k < D; k += TPR) t = fma(G[row * D + k], x[k], t);
#pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (part == 0) y[row] = t;
    __syncthreads();
  };
  for (int i = tid; i < D; i += NT) v[i] = rsqrt((double)D);
  __syncthreads();
  for (int it = 0; it < 5; it++) {  // (lam_2 / lam_1)^5 ~ 1e-23 at BASELINE's Grams; checked below
    matvec(v, w);
    const double nn = block_sum(tid < D ? w[tid] * w[tid] : 0.0, red);
    if (!(nn > 0.0) || !isfinite(nn)) return 0.0;
    const double sc = rsqrt(nn);
    for (int i = tid; i < D; i += NT) v[i] = w[i] * sc;
    __syncthreads();
  }
  matvec(v, w);
  const double lam = block_sum(tid < D ? v[tid] * w[tid] : 0.0, red);
  const double res = block_sum(tid < D ? (w[tid] - lam * v[tid]) * (w[tid] - lam * v[tid]) : 0.0, red);
  double off = 0.0;
  for (int e = tid; e < D * D; e += NT) {
    const double r = G[e] - lam * v[e / D] * v[e % D];
    off = fma(r, r, off);
  }
  off = block_sum(off, red);
  if (!(lam > 0.0) || !(sqrt(res) <= 16.0 * D * 2.220446049250313e-16 * lam) || !(sqrt(off) <= 1e-3 * lam))
    return 0.0;
  // u = v + sign(v_0) e_1, beta = 2 / u^T u = 1 / (1 + |v_0|)
  const double s0 = v[0] >= 0.0 ? 1.0 : -1.0, beta = 1.0 / (1.0 + fabs(v[0]));
  for (int i = tid; i < D; i += NT) u[i] = v[i] + (i == 0 ? s0 : 0.0);
  __syncthreads();
  matvec(u, w);  // p = G u
  const double K = block_sum(tid < D ? u[tid] * w[tid] : 0.0, red);
  for (int i = tid; i < D; i += NT) w[i] = beta * w[i] - 0.5 * beta * beta * K * u[i];  // H G H = G - u w^T - w u^T
  __syncthreads();
  for (int e = tid; e < D * D; e += NT) {
    const int i = e / D, j = e % D;
    const double g = G[e] - u[i] * w[j] - w[i] * u[j];
    G[e] = (i == 0) != (j == 0) ? 0.0 : g;
  }
  __syncthreads();
  return beta;
}

// Iterative refinement of an approximate eigenbasis of a symmetric G (Ogita & Aishima 2018,
// "Iterative refinement for symmetric eigenvalue decomposition"), replacing the FP64 Jacobi
// sweeps after the FP32 prelude.  With R = I - V^T V and S = V^T G V, the Rayleigh quotients
// lam_i = S_ii / (1 - R_ii) and the correction E_ij = (S_ij + lam_j R_ij) / (lam_j - lam_i)
// (i != j), E_ii = R_ii / 2 give V <- V + V E; the error (departure from orthonormality and from
// the eigenbasis) squares every iteration, so an FP32-accurate start converges in 2-3 steps of
// four D x D products, against three FP64 sweeps of 63 shared-memory-bound rounds.  Pairs whose
// Rayleigh quotients are too close to be separated at the current accuracy (|E_ij| would exceed
// 0.25) get only the orthogonality correction E_ij = R_ij / 2, as in the paper's clustered case.
// Returns the iterations used; on exit W = G V.  Shared memory: G (row-major D x D, symmetric),
// W / V (jf layout), scratch X, Y, S (D x (D + 8) doubles each), lam (D).
template <int D>
__device__ int jacobi_oa_refine(const double* G, double* W, double* V, double* X, double* Y, double* S,
                                double* lam, double* red) {
  constexpr int NT = D / 2 * JF_G, LD = D + 8, LT = D + 2;
  const int tid = threadIdx.x;
  double* Wr = W;  // G V row-major during the iterations (jf layout again on exit)
  // X = V row-major; Wr = G V (G symmetric: G(i, k) read as G[k D + i])
  for (int e = tid; e < D * D; e += NT) {
    const int i = e / D, k = e % D;
    X[k * LT + i] = V[i * LD + k];
  }
  __syncthreads();
  smem_gemm_blk<D>([&](int i, int k) { return G[k * D + i]; }, [&](int k, int j) { return X[k * LT + j]; },
                   [&](int i, int j, double v) { Wr[i * LT + j] = v; });
  __syncthreads();
  int it = 0;
  for (; it < 8; it++) {
    // Y = R = I - V^T V; S = V^T W; lam_i = S_ii / (1 - R_ii)
    smem_gemm_blk<D>([&](int i, int k) { return X[k * LT + i]; }, [&](int k, int j) { return X[k * LT + j]; },
                     [&](int i, int j, double v) { Y[i * LT + j] = (i == j ? 1.0 : 0.0) - v; });
    smem_gemm_blk<D>([&](int i, int k) { return X[k * LT + i]; }, [&](int k, int j) { return Wr[k * LT + j]; },
                     [&](int i, int j, double v) { S[i * LT + j] = v; });
    __syncthreads();
    for (int i = tid; i < D; i += NT) lam[i] = S[i * LT + i] / (1.0 - Y[i * LT + i]);
    __syncthreads();
    // E in place of R; S symmetrised (its rounding is not: an asymmetric S would leave
    // E + E^T != R and stall the orthogonality at ~eps ||G|| / gap)
    double emax = 0.0;
    for (int e = tid; e < D * D; e += NT) {
      const int i = e / D, j = e % D;
      const double rij = Y[i * LT + j];
      double ev;
      if (i == j) {
        ev = 0.5 * rij;
      } else {
        const double sij = 0.5 * (S[i * LT + j] + S[j * LT + i]);
        const double num = fma(lam[j], rij, sij), gap = lam[j] - lam[i];
        ev = fabs(num) < 0.25 * fabs(gap) ? num / gap : 0.5 * rij;
        emax = fmax(emax, fabs(ev));
      }
      Y[i * LT + j] = ev;
    }
    __syncthreads();
    // X = V + V E (row-major), then V (jf) from it, then Wr = G V
    smem_gemm_blk<D>([&](int i, int k) { return V[k * LD + i]; }, [&](int k, int j) { return Y[k * LT + j]; },
                     [&](int i, int j, double v) { X[i * LT + j] = V[j * LD + i] + v; });
    __syncthreads();
    for (int e = tid; e < D * D; e += NT) {
      const int j = e / D, i = e % D;
      V[j * LD + i] = X[i * LT + j];
    }
    smem_gemm_blk<D>([&](int i, int k) { return G[k * D + i]; }, [&](int k, int j) { return X[k * LT + j]; },
                     [&](int i, int j, double v) { Wr[i * LT + j] = v; });
    emax = block_max(emax, red);  // ends with a barrier
    if (emax <= 1e-8) {  // the update just applied was <= 1e-8: the remaining error is ~1e-16 / gap
      it++;
      break;
    }
  }
  // W back to the jf layout
  for (int e = tid; e < D * D; e += NT) {
    const int i = e / D, j = e % D;
    Y[i * LT + j] = Wr[i * LT + j];
  }
  __syncthreads();
  for (int e = tid; e < D * D; e += NT) {
    const int j = e / D, i = e % D;
    W[j * LD + i] = Y[i * LT + j];
  }
  __syncthreads();
  return it;
}

template <int D, bool SYM>
__global__ void __launch_bounds__(D / 2 * JF_G) jacobi_fixed_kernel(MatPtrs Ms, const double* __restrict__ Mc,
                                                                   double* __restrict__ sigma,
                                                                   double* __restrict__ Vout, int sweeps32,
                                                                   int deflate, int refine) {
  constexpr int NP = D / 2, NT = NP * JF_G, E = D / JF_G;
  extern __shared__ double jf_sm[];
  double* W = jf_sm;
  double* V = jf_sm + D * (D + 8);
  __shared__ int s_rot;
  __shared__ int s_order[D];
  __shared__ double s_norm[D];
  const double* M = Mc ? Mc + (size_t)blockIdx.x * D * D : Ms.p[blockIdx.x];
  sigma += (size_t)blockIdx.x * D;
  Vout += (size_t)blockIdx.x * D * D;
  const int tid = threadIdx.x;
  double beta = 0.0;
  __shared__ double s_u[D], s_v[D], s_w[D], s_red[32];
  if (SYM && sweeps32 > 0) {
    // the Gram matrix, symmetrised, in the Y/Z scratch past the FP32 buffers; deflated in place
    double* Gs = jf_sm + 4 * D * (D + 8);
    for (int e = tid; e < D * D; e += NT) {
      const int i = e / D, j = e % D;
      Gs[e] = 0.5 * (M[(size_t)i * D + j] + M[(size_t)j * D + i]);
    }
    __syncthreads();
    if (deflate) beta = jacobi_deflate<D>(Gs, s_u, s_v, s_w, s_red);
    float* W32 = reinterpret_cast<float*>(jf_sm + 2 * D * (D + 8));
    // with the dominant eigenpair deflated (the remaining spectrum well scaled) and the
    // refinement to follow, the prelude tracks W only and takes V from W's normalised columns
    // (half the shared-memory traffic per FP32 round)
    if (refine && beta != 0.0)
      jacobi_fp32_prelude<D, false>(Gs, W, V, W32, W32 + D * (D + 8), sweeps32, false);
    else
      jacobi_fp32_prelude<D, true>(Gs, W, V, W32, W32 + D * (D + 8), sweeps32, !refine);
    if (refine) {
      double* X = jf_sm + 2 * D * (D + 8);
      const int its = jacobi_oa_refine<D>(Gs, W, V, X, X + D * (D + 8), Gs + D * D, s_w, s_red);
      if (tid == 0) g_jacobi_sweeps[blockIdx.x & 7] = 100 + its;
    }
  } else {
    for (int e = tid; e < D * D; e += NT) {
      const int i = e / D, j = e % D;  // M row i, column j
      const double m = SYM ? 0.5 * (M[(size_t)i * D + j] + M[(size_t)j * D + i]) : M[(size_t)i * D + j];
      W[jf_off<D>(j, i)] = m;
      V[jf_off<D>(j, i)] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
  }
  const int group = tid / JF_G, lg = tid % JF_G;
  const double tol = 2.0 * D * 2.220446049250313e-16;
  // symmetric problems: after a sweep whose rotations all had c^2 <= MU2_DONE a b (column cosines
  // <= 1e-9), the next sweep's would be O(1e-18 / relative gap), below tol: that confirmation
  // sweep is skipped (measured at d = 64: cosines 2e-5, 1e-9, then none above tol)
  constexpr double MU2_DONE = 1e-18;
  __shared__ int s_big;
  const int fp64_sweeps = (SYM && sweeps32 > 0 && refine) ? 0 : 40;
  for (int sweep = 0; sweep < fp64_sweeps; sweep++) {
    if (tid == 0) {
      s_rot = 0;
      s_big = 0;
    }
    __syncthreads();
    for (int r = 0; r < D - 1; r++) {
      auto player = [&](int pos) {
        int x = pos - 1 + r;
        if (x >= D - 1) x -= D - 1;
        return pos == 0 ? 0 : 1 + x;
      };
      const int p = player(group), q = player(D - 1 - group);
      double x[E], y[E], u[E], v[E];
#pragma unroll
      for (int k = 0; k < E; k++) {
        x[k] = W[jf_off<D>(p, lg + k * JF_G)];
        y[k] = W[jf_off<D>(q, lg + k * JF_G)];
      }
      // V columns do not depend on the rotation: their loads overlap the dot products
#pragma unroll
      for (int k = 0; k < E; k++) {
        u[k] = V[jf_off<D>(p, lg + k * JF_G)];
        v[k] = V[jf_off<D>(q, lg + k * JF_G)];
      }
      double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
      for (int k = 0; k < E; k++) {
        a = fma(x[k], x[k], a);
        b = fma(y[k], y[k], b);
        c = fma(x[k], y[k], c);
      }
#pragma unroll
      for (int o = JF_G / 2; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
      }
      if (c != 0.0 && a != 0.0 && b != 0.0 && c * c > tol * tol * a * b) {
        // t ~ tan(theta) = sign(x) y / (|x| + sqrt(x^2 + y^2)), x = b - a, y = 2c, from hardware
        // approximations refined by one Newton step each (t only steers the rotation; cs, and so
        // cs^2 + sn^2 = 1, is computed to full precision)
        const double x2 = b - a, y2 = 2.0 * c;
        const double qq = fma(x2, x2, y2 * y2);
        double rq;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rq) : "d"(qq));
        rq = rq * fma(-0.5 * qq * rq, rq, 1.5);
        const double den = fma(qq, rq, fabs(x2));
        double ri;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(ri) : "d"(den));
        ri = ri * fma(-den, ri, 2.0);
        const double tt = y2 * ri;
        const double t = x2 >= 0.0 ? tt : -tt;
        const double cs = rsqrt(fma(t, t, 1.0));
        const double sn = cs * t;
#pragma unroll
        for (int k = 0; k < E; k++) {
          W[jf_off<D>(p, lg + k * JF_G)] = cs * x[k] - sn * y[k];
          W[jf_off<D>(q, lg + k * JF_G)] = sn * x[k] + cs * y[k];
          V[jf_off<D>(p, lg + k * JF_G)] = cs * u[k] - sn * v[k];
          V[jf_off<D>(q, lg + k * JF_G)] = sn * u[k] + cs * v[k];
        }
        if (lg == 0) {
          s_rot = 1;
          if (SYM && c * c > MU2_DONE * a * b) s_big = 1;
        }
      }
      __syncthreads();
    }
    if (tid == 0) g_jacobi_sweeps[blockIdx.x & 7] = sweep + 1;
    if (s_rot == 0 || (SYM && s_big == 0)) break;
    __syncthreads();
  }
  for (int j = tid; j < D; j += NT) {
    double s = 0.0;
    for (int i = 0; i < D; i++) s = fma(W[jf_off<D>(j, i)], W[jf_off<D>(j, i)], s);
    s_norm[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < D; j += NT) {
    int rank = 0;
    // total order even for non-finite input (NaN ranks last): every rank is assigned exactly once
    const double sj = isnan(s_norm[j]) ? -1.0 : s_norm[j];
    for (int k = 0; k < D; k++) {
      const double sk = isnan(s_norm[k]) ? -1.0 : s_norm[k];
      rank += (sk > sj) || (sk == sj && k < j);
    }
    s_order[rank] = j;
  }
  __syncthreads();
  for (int k = tid; k < D; k += NT) sigma[k] = s_norm[s_order[k]];
  if (SYM && beta != 0.0) {  // eigenvectors of G: H V' = V' - beta u (u^T V')
    __syncthreads();  // sigma has read the norms
    for (int j = tid; j < D; j += NT) {
      double t = 0.0;
      for (int i = 0; i < D; i++) t = fma(s_u[i], V[jf_off<D>(j, i)], t);
      s_norm[j] = beta * t;  // the norms are no longer needed
    }
    __syncthreads();
    for (int e = tid; e < D * D; e += NT) {
      const int j = e / D, i = e % D;
      V[jf_off<D>(j, i)] -= s_u[i] * s_norm[j];
    }
    __syncthreads();
  }
  for (int e = tid; e < D * D; e += NT) {
    const int i = e / D, k = e % D;
    Vout[e] = V[jf_off<D>(s_order[k], i)];
  }
}

__global__ void symmetrize_kernel(const double* __restrict__ M, int d, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)d * d) return;
  const int64_t i = e / d, j = e - i * d;
  out[e] = 0.5 * (M[i * d + j] + M[j * d + i]);
}

// U[:, j] *= 1/sigma[j] for j < rank, zero otherwise (U = A V Sigma^-1, tensor.py:102-107)
__global__ void scale_cols_kernel(double* U, int64_t n, int d, const double* __restrict__ sigma,
                                  double rank_tol) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * d) return;
  const int j = (int)(e % d);
  const double s0 = sigma[0];
  const double sj = sigma[j];
  const bool keep = s0 > 0.0 && sj > rank_tol * s0;
  U[e] = keep ? U[e] / sj : 0.0;
}

__global__ void transpose_kernel(const double* __restrict__ a, int64_t rows, int64_t cols,
                                 double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t i = e / cols, j = e - i * cols;
  out[j * rows + i] = a[e];
}


// LU with partial pivoting (LAPACK dgetrf pivot rule: first max |a|) in shared memory, then
// X = A^-1 by forward/back substitution, one thread per column of the identity.
// info[0] = k+1 if U(k,k) is exactly zero (np.linalg.solve raises LinAlgError), else 0;
// info[1] = 1 if the inverse has a non-finite entry.
__global__ void inverse_small_kernel(const double* __restrict__ M, int d, double* __restrict__ X,
                                     int32_t* __restrict__ info) {
  extern __shared__ double LU[];
  __shared__ int piv[128];
  __shared__ int s_p;
  __shared__ int s_info;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < d * d; e += nt) LU[e] = M[e];
  if (tid == 0) s_info = 0;
  __syncthreads();
  for (int k = 0; k < d; k++) {
    if (tid == 0) {
      int p = k;
      double best = fabs(LU[k * d + k]);
      for (int i = k + 1; i < d; i++) {
        const double v = fabs(LU[i * d + k]);
        if (v > best) { best = v; p = i; }
      }
      s_p = p;
      piv[k] = p;
      if (LU[p * d + k] == 0.0 && s_info == 0) s_info = k + 1;
    }
    __syncthreads();
    const int p = s_p;
    if (p != k)
      for (int j = tid; j < d; j += nt) {
        const double t = LU[k * d + j];
        LU[k * d + j] = LU[p * d + j];
        LU[p * d + j] = t;
      }
    __syncthreads();
    const double pivv = LU[k * d + k];
    if (pivv != 0.0)
      for (int i = k + 1 + tid; i < d; i += nt) LU[i * d + k] /= pivv;
    __syncthreads();
    for (int e = tid; e < (d - k - 1) * (d - k - 1); e += nt) {
      const int i = k + 1 + e / (d - k - 1), j = k + 1 + e % (d - k - 1);
      LU[i * d + j] = fma(-LU[i * d + k], LU[k * d + j], LU[i * d + j]);
    }
    __syncthreads();
  }
  bool bad = false;
  for (int j = tid; j < d; j += nt) {
    // column j of P*I: apply the row interchanges to e_j
    int src = j;
    // position of e_j after the swaps: track where row j ends up
    for (int k = 0; k < d; k++) {
      if (piv[k] == src) src = k; else if (k == src) src = piv[k];
    }
    for (int i = 0; i < d; i++) X[i * d + j] = (i == src) ? 1.0 : 0.0;
    for (int i = 0; i < d; i++) {
      double s = X[i * d + j];
      for (int k = 0; k < i; k++) s = fma(-LU[i * d + k], X[k * d + j], s);
      X[i * d + j] = s;
    }
    for (int i = d - 1; i >= 0; i--) {
      double s = X[i * d + j];
      for (int k = i + 1; k < d; k++) s = fma(-LU[i * d + k], X[k * d + j], s);
      const double v = s / LU[i * d + i];
      X[i * d + j] = v;
      bad |= !isfinite(v);
    }
  }
  bad = __syncthreads_or(bad);
  if (tid == 0) {
    info[0] = s_info;
    info[1] = bad ? 1 : 0;
  }
}

}  // namespace

namespace ks {

int chol_qr2_r(cudaStream_t st, const double* A, int64_t n, int d, double* R, int* ok, double* Rinv);
int chol_qr2_r_async(cudaStream_t st, const double* A, int64_t n, int d, double* R, double* Rinv,
                     int32_t* info_dev);

// info_dev (device, 2 x int32, may be null): the CholeskyQR2 path runs without its host check and
// leaves its status words there (nonzero: R undefined, the caller redoes the factorisation); the
// Householder path zeroes them.  Null: the check synchronises and falls back to Householder itself.
int qr_r(cudaStream_t st, const double* A, int64_t n, int d, double* R, int32_t* info_dev = nullptr) {
  KS_REQUIRE(d >= 1 && d <= 128, KS_ESIZE, "qr_r supports 1 <= d <= 128 (got %d)", d);
  // tall and well-conditioned: CholeskyQR2 (two Gram passes + one streaming triangular solve,
  // ks_cholqr.cu); otherwise Householder TSQR below
  const bool cq = n >= 4 * (int64_t)d && !ks::env(ks::ENV_TSQR);
  if (info_dev && cq) return chol_qr2_r_async(st, A, n, d, R, nullptr, info_dev);
  if (info_dev) KS_TRY_CUDA(cudaMemsetAsync(info_dev, 0, 2 * sizeof(int32_t), st));
  if (cq) {
    int ok = 0;
    int rc = chol_qr2_r(st, A, n, d, R, &ok, nullptr);
    if (rc) return rc;
    if (ok) return KS_OK;
  }
  const bool smem = (size_t)d * 2 * d * sizeof(double) * 2 <= QR_SMEM_CAP;  // panel >= 4d rows fits
  int prows;
  if (smem) {
    prows = (int)(QR_SMEM_CAP / (sizeof(double) * d));
    prows = std::min(prows, 2048);
  } else {
    prows = 4 * d;
  }
  if (prows < 2 * d) prows = 2 * d;
  const double* src = A;
  int64_t rows = n;
  Scratch<double> buf0((int64_t)((n + prows - 1) / prows) * d * d + d * d, st);
  Scratch<double> buf1((int64_t)((n + prows - 1) / prows) * d * d + d * d, st);
  KS_REQUIRE(buf0.p && buf1.p, KS_ECUDA, "scratch allocation failed");
  Scratch<double> gwork(smem ? 0 : (int64_t)((n + prows - 1) / prows) * prows * d, st);
  double* bufs[2] = {buf0.p, buf1.p};
  int which = 0;
  while (true) {
    const int64_t nparts = (rows + prows - 1) / prows;
    double* out = (nparts == 1) ? R : bufs[which];
    const int cur_rows = (int)ks_min64(prows, rows);
    if (smem) {
      const size_t sm = (size_t)cur_rows * d * sizeof(double);
      KS_TRY_CUDA(cudaFuncSetAttribute(qr_panel_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QR_SMEM_CAP + 1024));
      qr_panel_kernel<true><<<(unsigned)nparts, QR_THREADS, sm, st>>>(src, rows, d, prows, out, nullptr);
    } else {
      qr_panel_kernel<false><<<(unsigned)nparts, QR_THREADS, 0, st>>>(src, rows, d, prows, out, gwork.p);
    }
    KS_CHECK_LAUNCH();
    if (nparts == 1) break;
    src = out;
    rows = nparts * d;
    which ^= 1;
  }
  return KS_OK;
}

template <int D, bool SYM>
static void launch_jacobi_fixed(cudaStream_t st, const MatPtrs& Ms, const double* M, double* sigma, double* V,
                                int batch) {
  // symmetric (Gram) problems: FP32 prelude sweeps (KS_JACOBI_FP32=<n>, default 6; 0 = off)
  int sweeps32 = 0;
  if (SYM) {
    const char* e = ks::env(ks::ENV_JACOBI_FP32);
    sweeps32 = e ? atoi(e) : 6;
  }
  // symmetric problems with the FP32 prelude also hold the Gram matrix (D x D) for the deflation
  // plus S (D x (D + 8)) for the refinement
  const int smem = ((sweeps32 > 0 ? 5 : 2) * D * (D + 8) + (sweeps32 > 0 ? D * D : 0)) * (int)sizeof(double);
  const int deflate = SYM && !ks::env(ks::ENV_NO_DEFLATE);
  const int refine = SYM && !ks::env(ks::ENV_NO_OA);
  cudaFuncSetAttribute(jacobi_fixed_kernel<D, SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  jacobi_fixed_kernel<D, SYM><<<batch, D / 2 * JF_G, smem, st>>>(Ms, M, sigma, V, sweeps32, deflate, refine);
}


// d = 128: the fixed-size one-sided Jacobi with W (128 x 136 doubles, 139 KB) in shared memory; the
// accumulated rotations V keep rows 0..63 in shared memory (70 KB) and rows 64..127 in a
// per-problem global scratch (L2-resident).  Both halves of a pair's V columns are loaded at the
// start of the round (their latency hides behind the dot products) and written after the
// rotation; the block barrier publishes them to the next round.  512 threads: 64 column pairs x 8
// threads, 16 elements per thread.  Same rotation formulas, convergence rule and output contract
// as jacobi_fixed_kernel.
template <bool SYM>
__global__ void __launch_bounds__(512) jacobi128_kernel(MatPtrs Ms, const double* __restrict__ Mc,
                                                        double* __restrict__ sigma, double* __restrict__ Vout,
                                                        double* __restrict__ Vg_all) {
  constexpr int D = 128, NT = 512, E = D / JF_G, EH = E / 2, LV = 72;
  extern __shared__ double jf_sm[];
  double* W = jf_sm;
  double* Vs = jf_sm + D * (D + 8);                  // rows 0..63:   Vs[j * LV + i]
  double* Vg = Vg_all + (size_t)blockIdx.x * D * LV;  // rows 64..127: Vg[j * LV + i - 64]
  __shared__ int s_rot;
  __shared__ int s_order[D];
  __shared__ double s_norm[D];
  const double* M = Mc ? Mc + (size_t)blockIdx.x * D * D : Ms.p[blockIdx.x];
  sigma += (size_t)blockIdx.x * D;
  Vout += (size_t)blockIdx.x * D * D;
  const int tid = threadIdx.x;
  for (int e = tid; e < D * D; e += NT) {
    const int i = e / D, j = e % D;
    const double m = SYM ? 0.5 * (M[(size_t)i * D + j] + M[(size_t)j * D + i]) : M[(size_t)i * D + j];
    W[jf_off<D>(j, i)] = m;
    const double id = (i == j) ? 1.0 : 0.0;
    if (i < 64) Vs[j * LV + i] = id; else Vg[j * LV + i - 64] = id;
  }
  __syncthreads();
  const int group = tid / JF_G, lg = tid % JF_G;
  const double tol = 2.0 * D * 2.220446049250313e-16;
  for (int sweep = 0; sweep < 40; sweep++) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int r = 0; r < D - 1; r++) {
      auto player = [&](int pos) {
        int x = pos - 1 + r;
        if (x >= D - 1) x -= D - 1;
        return pos == 0 ? 0 : 1 + x;
      };
      const int p = player(group), q = player(D - 1 - group);
      double x[E], y[E], ug[EH], vg[EH];
      // global half of V first: the longest latency, consumed last
#pragma unroll
      for (int k = 0; k < EH; k++) {
        ug[k] = Vg[p * LV + lg + k * JF_G];
        vg[k] = Vg[q * LV + lg + k * JF_G];
      }
#pragma unroll
      for (int k = 0; k < E; k++) {
        x[k] = W[jf_off<D>(p, lg + k * JF_G)];
        y[k] = W[jf_off<D>(q, lg + k * JF_G)];
      }
      double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
      for (int k = 0; k < E; k++) {
        a = fma(x[k], x[k], a);
        b = fma(y[k], y[k], b);
        c = fma(x[k], y[k], c);
      }
#pragma unroll
      for (int o = JF_G / 2; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
      }
      if (c != 0.0 && a != 0.0 && b != 0.0 && c * c > tol * tol * a * b) {
        const double x2 = b - a, y2 = 2.0 * c;
        const double qq = fma(x2, x2, y2 * y2);
        double rq;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rq) : "d"(qq));
        rq = rq * fma(-0.5 * qq * rq, rq, 1.5);
        const double den = fma(qq, rq, fabs(x2));
        double ri;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(ri) : "d"(den));
        ri = ri * fma(-den, ri, 2.0);
        const double tt = y2 * ri;
        const double t = x2 >= 0.0 ? tt : -tt;
        const double cs = rsqrt(fma(t, t, 1.0));
        const double sn = cs * t;
#pragma unroll
        for (int k = 0; k < E; k++) {
          W[jf_off<D>(p, lg + k * JF_G)] = cs * x[k] - sn * y[k];
          W[jf_off<D>(q, lg + k * JF_G)] = sn * x[k] + cs * y[k];
        }
#pragma unroll
        for (int k = 0; k < EH; k++) {
          const int i = lg + k * JF_G;
          const double u = Vs[p * LV + i], v = Vs[q * LV + i];
          Vs[p * LV + i] = cs * u - sn * v;
          Vs[q * LV + i] = sn * u + cs * v;
        }
#pragma unroll
        for (int k = 0; k < EH; k++) {
          const int i = lg + k * JF_G;
          Vg[p * LV + i] = cs * ug[k] - sn * vg[k];
          Vg[q * LV + i] = sn * ug[k] + cs * vg[k];
        }
        if (lg == 0) s_rot = 1;
      }
      __syncthreads();
    }
    if (tid == 0) g_jacobi_sweeps[blockIdx.x & 7] = sweep + 1;
    if (s_rot == 0) break;
    __syncthreads();
  }
  for (int j = tid; j < D; j += NT) {
    double s2 = 0.0;
    for (int i = 0; i < D; i++) s2 = fma(W[jf_off<D>(j, i)], W[jf_off<D>(j, i)], s2);
    s_norm[j] = sqrt(s2);
  }
  __syncthreads();
  for (int j = tid; j < D; j += NT) {
    int rank = 0;
    // total order even for non-finite input (NaN ranks last): every rank is assigned exactly once
    const double sj = isnan(s_norm[j]) ? -1.0 : s_norm[j];
    for (int k = 0; k < D; k++) {
      const double sk = isnan(s_norm[k]) ? -1.0 : s_norm[k];
      rank += (sk > sj) || (sk == sj && k < j);
    }
    s_order[rank] = j;
  }
  __syncthreads();
  for (int k = tid; k < D; k += NT) sigma[k] = s_norm[s_order[k]];
  for (int e = tid; e < D * D; e += NT) {
    const int i = e / D, k = e % D;
    const int j = s_order[k];
    Vout[e] = i < 64 ? Vs[j * LV + i] : Vg[j * LV + i - 64];
  }
}

template <bool SYM>
static int launch_jacobi128(cudaStream_t st, const MatPtrs& Ms, const double* M, double* sigma, double* V, int batch) {
  Scratch<double> vg((int64_t)batch * 128 * 72, st);
  KS_REQUIRE(vg.p, KS_ECUDA, "scratch allocation failed");
  const int smem = (128 * 136 + 128 * 72) * (int)sizeof(double);
  KS_TRY_CUDA(cudaFuncSetAttribute(jacobi128_kernel<SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  jacobi128_kernel<SYM><<<batch, 512, smem, st>>>(Ms, M, sigma, V, vg.p);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

template <bool SYM>
static bool jacobi_fixed(cudaStream_t st, const MatPtrs& Ms, const double* M, int d, double* sigma, double* V,
                         int batch) {
  if (ks::env(ks::ENV_JACOBI_GENERIC)) return false;
  switch (d) {
    case 16: launch_jacobi_fixed<16, SYM>(st, Ms, M, sigma, V, batch); return true;
    case 32: launch_jacobi_fixed<32, SYM>(st, Ms, M, sigma, V, batch); return true;
    case 64: launch_jacobi_fixed<64, SYM>(st, Ms, M, sigma, V, batch); return true;
    case 128: return launch_jacobi128<SYM>(st, Ms, M, sigma, V, batch) == KS_OK;
    default: return false;
  }
}

int svd_small(cudaStream_t st, const double* M, int d, double* sigma, double* V, int batch) {
  KS_REQUIRE(d >= 1 && d <= 128, KS_ESIZE, "svd_small supports 1 <= d <= 128 (got %d)", d);
  if (batch <= 0) return KS_OK;
  if (jacobi_fixed<false>(st, MatPtrs{}, M, d, sigma, V, batch)) {
    KS_CHECK_LAUNCH();
    return KS_OK;
  }
  const int dp = d + (d & 1);
  const size_t wbytes = (size_t)dp * d * sizeof(double);
  const size_t vbytes = (size_t)dp * dp * sizeof(double);
  const int threads = 512;
  if (wbytes + vbytes <= QR_SMEM_CAP) {
    KS_TRY_CUDA(cudaFuncSetAttribute(jacobi_svd_kernel<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QR_SMEM_CAP));
    jacobi_svd_kernel<true><<<batch, threads, wbytes + vbytes, st>>>(M, d, sigma, V, nullptr);
  } else {
    Scratch<double> vw((int64_t)batch * (d + 1) * (d + 1), st);
    KS_REQUIRE(vw.p, KS_ECUDA, "scratch allocation failed");
    KS_TRY_CUDA(cudaFuncSetAttribute(jacobi_svd_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QR_SMEM_CAP));
    jacobi_svd_kernel<false><<<batch, threads, wbytes, st>>>(M, d, sigma, V, vw.p);
  }
  KS_CHECK_LAUNCH();
  return KS_OK;
}

// Thin SVD of A (n x d) with n >= d: R = qr(A); (sigma, V) = svd(R); U = A V Sigma^-1.
static int thin_svd_tall(cudaStream_t st, const double* A, int64_t n, int d, double rank_tol,
                         double* U, double* sigma, double* V, int32_t* info_dev = nullptr) {
  Scratch<double> R((int64_t)d * d, st);
  KS_REQUIRE(R.p, KS_ECUDA, "scratch allocation failed");
  int rc = qr_r(st, A, n, d, R.p, info_dev);
  if (rc) return rc;
  rc = svd_small(st, R.p, d, sigma, V, 1);
  if (rc) return rc;
  rc = gemm(st, n, d, d, 1.0, A, d, 1, 0, V, d, 1, 0, 0.0, U, d, 1, 0, 1);
  if (rc) return rc;
  scale_cols_kernel<<<ceil_div_u(n * d, 256), 256, 0, st>>>(U, n, d, sigma, rank_tol);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

}  // namespace ks

extern "C" int ks_qr_r(const double* A, int64_t n, int32_t d, double* R, void* stream) {
  return ks::qr_r((cudaStream_t)stream, A, n, d, R);
}

extern "C" int ks_svd_small(const double* M, int32_t d, double* sigma, double* V, void* stream) {
  return ks::svd_small((cudaStream_t)stream, M, d, sigma, V, 1);
}

// Eigen-decomposition of nb symmetric PSD d x d matrices given by separate device pointers,
// symmetrised as 0.5 (M + M^T) on load; same output contract as ks_svd_small_batched.
extern "C" int ks_sym_eig_batched(int32_t nb, const double* const* mats, int32_t d, double* sigma, double* V,
                                  void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_REQUIRE(nb >= 1 && nb <= 8, KS_EINVAL, "1..8 matrices per call");
  KS_REQUIRE(d >= 1 && d <= 128, KS_ESIZE, "d must be in [1, 128] (got %d)", d);
  MatPtrs ps{};
  for (int i = 0; i < nb; i++) ps.p[i] = mats[i];
  if (ks::jacobi_fixed<true>(st, ps, nullptr, d, sigma, V, nb)) {
    KS_CHECK_LAUNCH();
    return KS_OK;
  }
  // generic sizes: symmetrise into a contiguous batch, then the generic kernel
  ks::Scratch<double> sym((int64_t)nb * d * d, st);
  KS_REQUIRE(sym.p, KS_ECUDA, "scratch allocation failed");
  for (int i = 0; i < nb; i++) {
    symmetrize_kernel<<<ceil_div_u((int64_t)d * d, 256), 256, 0, st>>>(mats[i], d, sym.p + (int64_t)i * d * d);
    KS_CHECK_LAUNCH();
  }
  return ks::svd_small(st, sym.p, d, sigma, V, nb);
}

extern "C" int ks_svd_small_batched(const double* M, int32_t batch, int32_t d, double* sigma, double* V,
                                    void* stream) {
  return ks::svd_small((cudaStream_t)stream, M, d, sigma, V, batch);
}

static int compact_svd_impl(const double* A, int64_t n, int32_t d, double rank_tol, double* U, double* sigma,
                            double* V, int32_t* rank, int32_t* info_dev, cudaStream_t st);

// U: n x min(n,d)... to keep the ABI simple the caller provides U (n x k), sigma (k), V (d x k)
// with k = min(n, d); columns past the rank are zero.
extern "C" int ks_compact_svd(const double* A, int64_t n, int32_t d, double rank_tol, double* U,
                              double* sigma, double* V, int32_t* rank, void* stream) {
  return compact_svd_impl(A, n, d, rank_tol, U, sigma, V, rank, nullptr, (cudaStream_t)stream);
}

// Fully asynchronous form (CUDA-graph capturable): no rank read-back, and the QR's CholeskyQR2
// status words go to info_dev (2 x int32 on the device; nonzero = that factorisation declined and
// the result is undefined -- the caller redoes it with ks_compact_svd).
extern "C" int ks_compact_svd_async(const double* A, int64_t n, int32_t d, double rank_tol, double* U,
                                    double* sigma, double* V, int32_t* info_dev, void* stream) {
  KS_REQUIRE(info_dev, KS_EINVAL, "compact_svd_async needs a device status buffer");
  return compact_svd_impl(A, n, d, rank_tol, U, sigma, V, nullptr, info_dev, (cudaStream_t)stream);
}

static int compact_svd_impl(const double* A, int64_t n, int32_t d, double rank_tol, double* U, double* sigma,
                            double* V, int32_t* rank, int32_t* info_dev, cudaStream_t st) {
  KS_REQUIRE(n >= 1 && d >= 1, KS_EINVAL, "compact_svd needs a non-empty matrix");
  KS_REQUIRE(rank_tol >= 0.0 && rank_tol < 1.0, KS_EINVAL, "rank_tol must be in [0, 1)");
  int rc;
  const int k = (int)ks_min64(n, d);
  if (n >= d) {
    rc = ks::thin_svd_tall(st, A, n, d, rank_tol, U, sigma, V, info_dev);
    if (rc) return rc;
  } else {
    // A^T (d x n) = U' S V'^T  =>  A = V' S U'^T: U = V' (n x n), V = U' (d x n)
    ks::Scratch<double> At((int64_t)d * n, st);
    KS_REQUIRE(At.p, KS_ECUDA, "scratch allocation failed");
    transpose_kernel<<<ceil_div_u(n * d, 256), 256, 0, st>>>(A, n, d, At.p);
    KS_CHECK_LAUNCH();
    rc = ks::thin_svd_tall(st, At.p, d, (int)n, rank_tol, V, sigma, U, info_dev);
    if (rc) return rc;
    // U holds V' (n x n) already normalised; zero columns past the rank for consistency
  }
  if (!rank) return KS_OK;  // the caller counts the rank from sigma itself (no synchronisation here)
  std::vector<double> hs(k);
  KS_TRY_CUDA(cudaMemcpyAsync(hs.data(), sigma, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
  KS_TRY_CUDA(cudaStreamSynchronize(st));
  int r = 0;
  if (hs[0] > 0.0)
    for (int j = 0; j < k; j++) r += hs[j] > rank_tol * hs[0];
  *rank = r;
  return KS_OK;
}

extern "C" int ks_inverse_small(const double* M, int32_t d, double* X, int32_t* info, void* stream) {
  KS_REQUIRE(d >= 1 && d <= 128, KS_ESIZE, "inverse_small supports 1 <= d <= 128 (got %d)", d);
  const size_t smem = (size_t)d * d * sizeof(double);
  KS_TRY_CUDA(cudaFuncSetAttribute(inverse_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
  inverse_small_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(M, d, X, info);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

// Profiling aid: sweeps used by the last one-sided Jacobi launch (first 8 problems).
extern "C" int ks_debug_jacobi_sweeps(int32_t* out8) {
  KS_TRY_CUDA(cudaMemcpyFromSymbol(out8, g_jacobi_sweeps, sizeof(int) * 8));
  return KS_OK;
}
