// Leverage scores and the product sampler on device.
//   JL estimator (leverage.py:85-130), exact scores from an SVD (leverage.py:51-64),
//   ProductSampler tables (leverage.py:159-175) with NumPy's exact summation orders,
//   inverse-CDF draws (leverage.py:193-201, Generator.choice) and sketch weights (:208-232).
#include "ks_common.cuh"
#include "ks_pairwise.cuh"
#include "ks_tma.cuh"

namespace {

// ---------------------------------------------------------------- JL scores
// One block = 64 rows: P = A_blk Q^T on FP64 tensor cores (DMMA m16n8k4, 8 warps = 4 row tiles x
// 2 column-tile phases), scores = row sums of P^2 in the accumulator epilogue.  Q (r x d) and the
// rows are staged in padded shared memory with asynchronous copies (zero-filled padding).
constexpr int JL_ROWS = 64;
__global__ void __launch_bounds__(256) jl_scores_kernel(const double* __restrict__ A, int64_t n, int d,
                                                       const double* __restrict__ Q, int r,
                                                       double denom, double* __restrict__ scores) {
  extern __shared__ double sm[];
  const int dp = (d + 3) & ~3, ld = dp + 4, rp = (r + 7) & ~7;
  double* Qs = sm;                    // rp x ld
  double* As = sm + (size_t)rp * ld;  // JL_ROWS x ld
  double* red = As + JL_ROWS * ld;    // 2 x JL_ROWS
  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * JL_ROWS;
  for (int e = tid; e < rp * dp; e += 256) {
    const int j = e / dp, k = e - j * dp;
    const bool ok = j < r && k < d;
    ks_cp_async8(&Qs[j * ld + k], ok ? Q + (size_t)j * d + k : Q, ok);
  }
  for (int e = tid; e < JL_ROWS * dp; e += 256) {
    const int i = e / dp, k = e - i * dp;
    const bool ok = row0 + i < n && k < d;
    ks_cp_async8(&As[i * ld + k], ok ? A + (row0 + i) * d + k : A, ok);
  }
  ks_cp_async_wait_all();
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int m0 = (warp & 3) * 16;
  const double* a_lo = As + (m0 + g) * ld + t;
  const double* a_hi = a_lo + 8 * ld;
  double rs0 = 0.0, rs1 = 0.0;
  for (int n0 = (warp >> 2) * 8; n0 < rp; n0 += 16) {
    const double* q = Qs + (n0 + g) * ld + t;
    double c[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k0 = 0; k0 < dp; k0 += 4) dmma_16x8x4(c, a_lo[k0], a_hi[k0], q[k0]);
    rs0 = fma(c[0], c[0], fma(c[1], c[1], rs0));
    rs1 = fma(c[2], c[2], fma(c[3], c[3], rs1));
  }
  rs0 += __shfl_xor_sync(0xffffffffu, rs0, 1);
  rs0 += __shfl_xor_sync(0xffffffffu, rs0, 2);
  rs1 += __shfl_xor_sync(0xffffffffu, rs1, 1);
  rs1 += __shfl_xor_sync(0xffffffffu, rs1, 2);
  if (t == 0) {
    red[(warp >> 2) * JL_ROWS + m0 + g] = rs0;
    red[(warp >> 2) * JL_ROWS + m0 + g + 8] = rs1;
  }
  __syncthreads();
  if (tid < JL_ROWS && row0 + tid < n) scores[row0 + tid] = (red[tid] + red[JL_ROWS + tid]) / denom;
}

__global__ void row_weighted_sumsq_kernel(const double* __restrict__ U, int64_t n, int d,
                                          const double* __restrict__ w, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int k = 0; k < d; k++) {
    const double u = U[i * d + k];
    s = fma(u * u, w[k], s);
  }
  out[i] = s;
}

__global__ void searchsorted_right_kernel(const double* __restrict__ cdf, int64_t n,
                                          const double* __restrict__ u, int64_t s,
                                          int64_t* __restrict__ idx, int64_t stride, int64_t off) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s) return;
  const double x = u[t];
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cdf[mid] <= x) lo = mid + 1; else hi = mid;
  }
  if (lo > n - 1) lo = n - 1;
  idx[t * stride + off] = lo;
}

struct ProbPtrs {
  const double* p[8];
};

__global__ void sketch_weights_kernel(int nf, ProbPtrs P, const int64_t* __restrict__ idx, int64_t s,
                                      double* __restrict__ w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s) return;
  double prob = 1.0;
  for (int f = 0; f < nf; f++) prob = __dmul_rn(prob, P.p[f][idx[t * nf + f]]);
  w[t] = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(prob, (double)s)));
}

}  // namespace

extern "C" int ks_jl_scores(const double* A, int64_t n, int32_t d, const double* Q, int32_t r,
                            double denom, double* scores, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_REQUIRE(d >= 1 && d <= 128 && r >= 1 && r <= 256, KS_ESIZE, "jl_scores: unsupported d=%d r=%d", d, r);
  if (n <= 0) return KS_OK;
  const size_t smem = sizeof(double) * ((size_t)(((r + 7) & ~7) + JL_ROWS) * (((d + 3) & ~3) + 4) + 2 * JL_ROWS);
  KS_REQUIRE(smem <= 220 * 1024, KS_ESIZE, "jl_scores: shared memory too large");
  KS_TRY_CUDA(cudaFuncSetAttribute(jl_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  jl_scores_kernel<<<ceil_div_u(n, JL_ROWS), 256, smem, st>>>(A, n, d, Q, r, denom, scores);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_row_weighted_sumsq(const double* U, int64_t n, int32_t d, const double* wts,
                                     double* scores, void* stream) {
  if (n <= 0) return KS_OK;
  row_weighted_sumsq_kernel<<<ceil_div_u(n, 256), 256, 0, (cudaStream_t)stream>>>(U, n, d, wts, scores);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_searchsorted_right(const double* cdf, int64_t n, const double* u, int64_t s,
                                     int64_t* idx, int64_t stride, int64_t off, void* stream) {
  if (s <= 0) return KS_OK;
  searchsorted_right_kernel<<<ceil_div_u(s, 256), 256, 0, (cudaStream_t)stream>>>(cdf, n, u, s, idx,
                                                                                stride, off);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_sketch_weights(int32_t nf, const double* const* probs, const int64_t* idx,
                                 int64_t s, double* w, void* stream) {
  KS_REQUIRE(nf >= 1 && nf <= 8, KS_EINVAL, "1..8 factors supported");
  if (s <= 0) return KS_OK;
  ProbPtrs P{};
  for (int f = 0; f < nf; f++) P.p[f] = probs[f];
  sketch_weights_kernel<<<ceil_div_u(s, 256), 256, 0, (cudaStream_t)stream>>>(nf, P, idx, s, w);
  KS_CHECK_LAUNCH();
  return KS_OK;
}
