// Leverage scores and the product sampler on device.
//   JL estimator (leverage.py:85-130), exact scores from an SVD (leverage.py:51-64),
//   ProductSampler tables (leverage.py:159-175) with NumPy's exact summation orders,
//   inverse-CDF draws (leverage.py:193-201, Generator.choice) and sketch weights (:208-232).
#include "ks_common.cuh"
#include "ks_pairwise.cuh"

namespace {

// ---------------------------------------------------------------- JL scores
// One block = 64 rows; Q (r x d) and the rows staged in padded shared memory.
constexpr int JL_ROWS = 64;
__global__ void __launch_bounds__(256) jl_scores_kernel(const double* __restrict__ A, int64_t n, int d,
                                                       const double* __restrict__ Q, int r,
                                                       double denom, double* __restrict__ scores) {
  extern __shared__ double sm[];
  const int ld = d + 1;
  double* Qs = sm;                   // r x ld
  double* As = sm + (size_t)r * ld;  // JL_ROWS x ld
  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * JL_ROWS;
  for (int e = tid; e < r * d; e += 256) {
    const int j = e / d, k = e - j * d;
    Qs[j * ld + k] = Q[e];
  }
  for (int e = tid; e < JL_ROWS * d; e += 256) {
    const int i = e / d, k = e - i * d;
    const int64_t gi = row0 + i;
    As[i * ld + k] = gi < n ? A[gi * d + k] : 0.0;
  }
  __syncthreads();
  const int i = tid >> 2, sub = tid & 3;
  double acc = 0.0;
  const double* a = As + i * ld;
  for (int j = sub; j < r; j += 4) {
    const double* q = Qs + j * ld;
    double z = 0.0;
    for (int k = 0; k < d; k++) z = fma(a[k], q[k], z);
    acc = fma(z, z, acc);
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  const int64_t gi = row0 + i;
  if (sub == 0 && gi < n) scores[gi] = acc / denom;
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
  const size_t smem = sizeof(double) * (size_t)(r + JL_ROWS) * (d + 1);
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
