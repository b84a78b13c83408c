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

// ---------------------------------------------------------------- sampler tables
constexpr int ST_T = 1024;
constexpr int ST_D = 10;  // 2^ST_D = ST_T subtrees

__device__ double pw_combine(const double* slot, int64_t s, int64_t len, int depth, int path) {
  // replay the top levels of the recursion (iterative, depth <= ST_D)
  // evaluate with an explicit stack
  int64_t st_s[ST_D + 1], st_l[ST_D + 1];
  int st_d[ST_D + 1], st_p[ST_D + 1], st_state[ST_D + 1];
  double st_v[ST_D + 1];
  int sp = 0;
  st_s[0] = s; st_l[0] = len; st_d[0] = depth; st_p[0] = path; st_state[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    const int64_t cl = st_l[sp];
    const int dd = st_d[sp];
    if (cl <= PW_BLOCK || dd == ST_D) {
      ret = slot[st_p[sp] << (ST_D - dd)];
      sp--;
      if (sp >= 0) {
        if (st_state[sp] == 1) { st_v[sp] = ret; st_state[sp] = 2; }
        else { ret = st_v[sp] + ret; st_state[sp] = 3; }
      }
      continue;
    }
    int64_t n2;
    pw_split(cl, &n2);
    if (st_state[sp] == 0) {
      st_state[sp] = 1;
      sp++;
      st_s[sp] = st_s[sp - 1]; st_l[sp] = n2; st_d[sp] = dd + 1; st_p[sp] = st_p[sp - 1] * 2;
      st_state[sp] = 0;
    } else if (st_state[sp] == 2) {
      sp++;
      st_s[sp] = st_s[sp - 1] + n2; st_l[sp] = cl - n2; st_d[sp] = dd + 1;
      st_p[sp] = st_p[sp - 1] * 2 + 1; st_state[sp] = 0;
    } else {
      sp--;
      if (sp >= 0) {
        if (st_state[sp] == 1) { st_v[sp] = ret; st_state[sp] = 2; }
        else { ret = st_v[sp] + ret; st_state[sp] = 3; }
      }
    }
  }
  return ret;
}

__device__ __forceinline__ int64_t block_incl_scan_i64(int64_t v, int64_t* wsum) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) wsum[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int64_t t = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    if (lane < nw) wsum[lane] = t;
  }
  __syncthreads();
  if (wid > 0) v += wsum[wid - 1];
  __syncthreads();
  return v;
}

__device__ __forceinline__ double ulp_of(double x) {
  // spacing of doubles at |x| (x > 0, normal range)
  int e;
  frexp(x, &e);          // x = m * 2^e, m in [0.5, 1)
  return ldexp(1.0, e - 53);
}

// One block per factor: total (pairwise), probs, exact sequential cumsum via verified
// speculation.  flags: 1 = negative/non-finite score, 2 = non-positive total.
__global__ void __launch_bounds__(ST_T) sampler_tables_kernel(const double* __restrict__ scores,
                                                             int64_t n, int renorm,
                                                             double* __restrict__ probs,
                                                             double* __restrict__ cdf,
                                                             int32_t* __restrict__ flags) {
  __shared__ double slot[ST_T];
  __shared__ int64_t wsum[32];
  __shared__ double s_total;
  __shared__ int s_bad;
  __shared__ int s_first;
  __shared__ double s_spec[ST_T];
  const int tid = threadIdx.x;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  {
    bool bad = false;
    for (int64_t i = tid; i < n; i += ST_T) {
      const double v = scores[i];
      bad |= !(v >= 0.0) || !isfinite(v);
    }
    if (__syncthreads_or(bad) && tid == 0) s_bad = 1;
  }
  // subtree of thread `tid` at depth ST_D (or the leaf it falls into)
  {
    int64_t s = 0, len = n;
    int depth = 0;
    bool owner = true;
    for (; depth < ST_D; depth++) {
      if (len <= PW_BLOCK) {
        owner = (tid & ((1 << (ST_D - depth)) - 1)) == 0;
        break;
      }
      int64_t n2;
      pw_split(len, &n2);
      const int bit = (tid >> (ST_D - 1 - depth)) & 1;
      if (bit) { s += n2; len -= n2; } else { len = n2; }
    }
    if (owner) {
      auto get = [&](int64_t i) { return scores[i]; };
      slot[tid] = pw_sum_seq(get, s, len);
    }
  }
  __syncthreads();
  if (tid == 0) {
    const double total = pw_combine(slot, 0, n, 0, 0);
    s_total = total;
    int f = s_bad ? 1 : 0;
    if (!(total > 0.0)) f |= 2;
    flags[0] = f;
  }
  __syncthreads();
  const double total = s_total;
  for (int64_t i = tid; i < n; i += ST_T) probs[i] = scores[i] / total;
  __syncthreads();
  if (cdf == nullptr) return;
  // exact cumsum: s_k = fl(s_{k-1} + p_k), verified block speculation
  double prev = 0.0;
  int64_t pos = 0;
  while (pos < n) {
    const int64_t i = pos + tid;
    const bool valid = i < n;
    const double x = valid ? probs[i] : 0.0;
    double ref = prev;
    if (ref == 0.0) ref = (pos < n) ? probs[pos] : 0.0;
    const double u = (ref > 0.0) ? ulp_of(ref) : 0x1.0p-1074;
    long long qi = 0;
    if (valid) {
      const double qd = x / u;
      qi = (qd < 0x1.0p52) ? __double2ll_rn(qd) : (1ll << 52);
    }
    const int64_t Q = block_incl_scan_i64(qi, wsum);
    // spec = prev + Q*u computed exactly when representable
    const double base = prev / u;  // integer-valued when prev is on the grid
    const double spec = (double)((long long)base + Q) * u;
    s_spec[tid] = spec;
    if (tid == 0) s_first = ST_T;
    __syncthreads();
    const double sprev = (tid == 0) ? prev : s_spec[tid - 1];
    const double real = __dadd_rn(sprev, x);
    const bool ok = !valid || (real == spec);
    if (!ok) atomicMin(&s_first, tid);
    __syncthreads();
    const int f = s_first;
    if (valid && tid < f) cdf[i] = spec;
    if (valid && tid == f) cdf[i] = real;
    int64_t adv = (f < ST_T) ? (int64_t)f + 1 : (int64_t)ST_T;
    if (pos + adv > n) adv = n - pos;
    __syncthreads();
    if (tid == 0) s_spec[0] = cdf[pos + adv - 1];
    __syncthreads();
    prev = s_spec[0];
    pos += adv;
    __syncthreads();
  }
  if (renorm) {
    __syncthreads();
    const double last = cdf[n - 1];
    __syncthreads();
    for (int64_t i = tid; i < n; i += ST_T) cdf[i] = cdf[i] / last;
  }
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

extern "C" int ks_sampler_tables(const double* scores, int64_t n, int32_t renormalise,
                                 double* probs, double* cdf, int32_t* flags, void* stream) {
  KS_REQUIRE(n >= 1, KS_EINVAL, "score vector must be nonempty");
  sampler_tables_kernel<<<1, ST_T, 0, (cudaStream_t)stream>>>(scores, n, renormalise, probs, cdf, flags);
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
