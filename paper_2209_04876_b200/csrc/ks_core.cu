// Core runtime + dense FP64 primitives for the kronsolve B200 library.
//   - error / scratch plumbing behind the C-ABI
//   - strided batched DFMA GEMM (building block of the implicit Kronecker multiplies,
//     reference kron.py:44-100)
//   - deterministic split-K A^T B for tall operands (Gram / projection products)
//   - validation, gather, sum-of-squares reductions
#include "ks_common.cuh"

#include <cstdlib>
#include <mutex>
#include <vector>

namespace ks {

int gemm_tn_tall_dmma(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                      int64_t a_ks, int64_t a_ms, const double* B, int64_t b_ks, int64_t b_ns, double* C);

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
  return KS_ECUDA;
}

static std::once_flag g_env_once;
static const char* g_env[ENV_COUNT];

const char* env(EnvSwitch id) {
  static const char* const names[ENV_COUNT] = {"KS_TALL", "KS_KRON2", "KS_RICHARDSON", "KS_NO_EIGBASIS", "KS_GRAM_SCALAR", "KS_GATHER_BLOCKS", "KS_TSQR", "KS_JACOBI_FP32", "KS_JACOBI_GENERIC", "KS_RICH_OLD", "KS_NO_DEFLATE", "KS_NO_OA", "KS_SKETCH_SORT", "KS_TALL_OLD", "KS_TABLES_ONE_CTA"};
  std::call_once(g_env_once, [] {
    for (int i = 0; i < ENV_COUNT; i++) g_env[i] = getenv(names[i]);
  });
  return g_env[id];
}

static std::once_flag g_pool_once;

void* scratch_alloc(size_t bytes, cudaStream_t s) {
  std::call_once(g_pool_once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void scratch_free(void* p, cudaStream_t s) { cudaFreeAsync(p, s); }

}  // namespace ks

extern "C" int ks_abi_version(void) { return KS_ABI_VERSION; }
extern "C" const char* ks_last_error(void) { return ks::g_err; }

// ===========================================================================
// Strided batched GEMM (DFMA, 64x64x16 tiles, 4x4 per thread, conflict-free smem reads)
// ===========================================================================

namespace {

constexpr int GB_M = 64, GB_N = 64, GB_K = 16;

enum GemmEpilogue { EPI_STORE = 0, EPI_RESID_SUMSQ = 1 };

template <int EPI>
__global__ void __launch_bounds__(256) gemm_kernel(
    int64_t M, int64_t N, int64_t K, double alpha,
    const double* __restrict__ A, int64_t a_rs, int64_t a_cs, int64_t a_bs,
    const double* __restrict__ B, int64_t b_rs, int64_t b_cs, int64_t b_bs,
    double beta, double* C, int64_t c_rs, int64_t c_cs, int64_t c_bs,
    double* __restrict__ partial) {
  __shared__ double As[GB_K][GB_M + 1];
  __shared__ double Bs[GB_K][GB_N + 1];
  __shared__ double red[8];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t bz = blockIdx.z;
  const int64_t m0 = (int64_t)blockIdx.y * GB_M, n0 = (int64_t)blockIdx.x * GB_N;
  A += bz * a_bs;
  B += bz * b_bs;
  C += bz * c_bs;
  const bool a_kfast = (a_cs == 1) || (a_rs != 1 && llabs(a_cs) < llabs(a_rs));
  const bool b_nfast = (b_cs == 1) || (b_rs != 1 && llabs(b_cs) < llabs(b_rs));

  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0.0;

  for (int64_t k0 = 0; k0 < K; k0 += GB_K) {
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int e = tid + r * 256;
      int mm, kk;
      if (a_kfast) { mm = e >> 4; kk = e & 15; } else { mm = e & 63; kk = e >> 6; }
      const int64_t gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? A[gm * a_rs + gk * a_cs] : 0.0;
      int nn, kb;
      if (b_nfast) { nn = e & 63; kb = e >> 6; } else { nn = e >> 4; kb = e & 15; }
      const int64_t gn = n0 + nn, gkb = k0 + kb;
      Bs[kb][nn] = (gn < N && gkb < K) ? B[gkb * b_rs + gn * b_cs] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GB_K; kk++) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; i++) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; j++) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

  if (EPI == EPI_STORE) {
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int64_t gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
        if (gm < M && gn < N) {
          double* c = C + gm * c_rs + gn * c_cs;
          const double v = alpha * acc[i][j];
          *c = (beta == 0.0) ? v : v + beta * *c;
        }
      }
  } else {
    double ss = 0.0;
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int64_t gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
        if (gm < M && gn < N) {
          const double r = alpha * acc[i][j] - C[gm * c_rs + gn * c_cs];
          ss = fma(r, r, ss);
        }
      }
    ss = block_sum(ss, red);
    if (tid == 0) {
      const int64_t blk = ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      partial[blk] = ss;
    }
  }
}

// Fixed-order sum of `n` partials into out[0] (single block).
__global__ void sum_partials_kernel(const double* __restrict__ p, int64_t n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += p[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[0] = s;
}

// Split-K A^T B partials: block b covers rows [b*chunk, min(K,(b+1)*chunk)).
constexpr int TT_K = 32;
__global__ void __launch_bounds__(256) gemm_tn_partial_kernel(
    int M, int N, int64_t K, int64_t chunk,
    const double* __restrict__ A, int64_t a_ks, int64_t a_ms,
    const double* __restrict__ B, int64_t b_ks, int64_t b_ns, double* __restrict__ part) {
  extern __shared__ double sm[];
  double* As = sm;                // [TT_K][M]
  double* Bs = sm + TT_K * M;     // [TT_K][N]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t kbeg = (int64_t)blockIdx.x * chunk;
  const int64_t kend = ks_min64(K, kbeg + chunk);
  const int mi = (M + 15) / 16, nj = (N + 15) / 16;  // <= 8 each
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = 0.0;
  const bool a_mfast = (a_ms == 1);
  const bool b_nfast = (b_ns == 1);
  for (int64_t k0 = kbeg; k0 < kend; k0 += TT_K) {
    for (int e = tid; e < TT_K * M; e += 256) {
      int kk, mm;
      if (a_mfast) { kk = e / M; mm = e - kk * M; } else { mm = e / TT_K; kk = e - mm * TT_K; }
      const int64_t gk = k0 + kk;
      As[kk * M + mm] = (gk < kend) ? A[gk * a_ks + (int64_t)mm * a_ms] : 0.0;
    }
    for (int e = tid; e < TT_K * N; e += 256) {
      int kk, nn;
      if (b_nfast) { kk = e / N; nn = e - kk * N; } else { nn = e / TT_K; kk = e - nn * TT_K; }
      const int64_t gk = k0 + kk;
      Bs[kk * N + nn] = (gk < kend) ? B[gk * b_ks + (int64_t)nn * b_ns] : 0.0;
    }
    __syncthreads();
    for (int kk = 0; kk < TT_K; kk++) {
      double a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int m = ty + 16 * i;
        a[i] = (i < mi && m < M) ? As[kk * M + m] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const int n = tx + 16 * j;
        b[j] = (j < nj && n < N) ? Bs[kk * N + n] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* out = part + (int64_t)blockIdx.x * M * N;
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int m = ty + 16 * i, n = tx + 16 * j;
      if (i < mi && j < nj && m < M && n < N) out[m * N + n] = acc[i][j];
    }
}

__global__ void reduce_partials_kernel(const double* __restrict__ part, int64_t nparts,
                                       int64_t count, double alpha, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  double s = 0.0;
  for (int64_t p = 0; p < nparts; p++) s += part[p * count + e];
  out[e] = alpha * s;
}

__global__ void sumsq_diff_partial_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                          int64_t n, double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double r = b ? a[i] - b[i] : a[i];
    s = fma(r, r, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void check_kernel(const double* __restrict__ a, int64_t n, int32_t* flags) {
  bool bad = false, nz = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = a[i];
    bad |= !isfinite(v);
    nz |= (v != 0.0);
  }
  bad = __syncthreads_or(bad);
  nz = __syncthreads_or(nz);
  if (threadIdx.x == 0) {
    if (bad) atomicOr(&flags[0], 1);
    if (nz) atomicOr(&flags[1], 1);
  }
}

__global__ void gather_kernel(const double* __restrict__ b, const int64_t* __restrict__ idx,
                              int64_t n, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = b[idx[i]];
}

}  // namespace

namespace ks {

int gemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t a_rs, int64_t a_cs, int64_t a_bs, const double* B, int64_t b_rs, int64_t b_cs,
         int64_t b_bs, double beta, double* C, int64_t c_rs, int64_t c_cs, int64_t c_bs,
         int64_t batch) {
  if (M <= 0 || N <= 0 || batch <= 0) return KS_OK;
  dim3 grid(ceil_div_u(N, GB_N), ceil_div_u(M, GB_M), (unsigned)batch);
  KS_REQUIRE(grid.y <= 65535 && grid.z <= 65535, KS_ESIZE, "gemm grid too large");
  gemm_kernel<EPI_STORE><<<grid, 256, 0, st>>>(M, N, K, alpha, A, a_rs, a_cs, a_bs, B, b_rs, b_cs,
                                               b_bs, beta, C, c_rs, c_cs, c_bs, nullptr);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

// sum((alpha*A B - C)^2) over an M x N product (single batch)
int gemm_resid_sumsq(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha,
                     const double* A, int64_t a_rs, int64_t a_cs, const double* B, int64_t b_rs,
                     int64_t b_cs, const double* C, int64_t c_rs, int64_t c_cs, double* out) {
  dim3 grid(ceil_div_u(N, GB_N), ceil_div_u(M, GB_M), 1);
  KS_REQUIRE(grid.y <= 65535, KS_ESIZE, "residual grid too large");
  const int64_t nb = (int64_t)grid.x * grid.y;
  Scratch<double> part(nb, st);
  KS_REQUIRE(part.p, KS_ECUDA, "scratch allocation failed");
  gemm_kernel<EPI_RESID_SUMSQ><<<grid, 256, 0, st>>>(M, N, K, alpha, A, a_rs, a_cs, 0, B, b_rs,
                                                     b_cs, 0, 0.0, const_cast<double*>(C), c_rs,
                                                     c_cs, 0, part.p);
  KS_CHECK_LAUNCH();
  sum_partials_kernel<<<1, 1024, 0, st>>>(part.p, nb, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

int gemm_tn_tall(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                 int64_t a_ks, int64_t a_ms, const double* B, int64_t b_ks, int64_t b_ns,
                 double* C) {
  KS_REQUIRE(M >= 1 && N >= 1 && M <= 128 && N <= 128, KS_EINVAL,
             "gemm_tn_tall supports 1 <= M,N <= 128 (got %lld x %lld)", (long long)M, (long long)N);
  if (K <= 0) {
    KS_TRY_CUDA(cudaMemsetAsync(C, 0, sizeof(double) * M * N, st));
    return KS_OK;
  }
  {
    const char* e = ks::env(ks::ENV_TALL);
    if (!(e && e[0] == 'g')) return gemm_tn_tall_dmma(st, M, N, K, alpha, A, a_ks, a_ms, B, b_ks, b_ns, C);
  }
  int64_t nparts = (K + 63) / 64;
  const int64_t cap = 2 * (int64_t)num_sms();
  if (nparts > cap) nparts = cap;
  int64_t chunk = (K + nparts - 1) / nparts;
  chunk = (chunk + TT_K - 1) / TT_K * TT_K;
  nparts = (K + chunk - 1) / chunk;
  Scratch<double> part(nparts * M * N, st);
  KS_REQUIRE(part.p, KS_ECUDA, "scratch allocation failed");
  const size_t smem = sizeof(double) * TT_K * (M + N);
  if (smem > 48 * 1024)
    KS_TRY_CUDA(cudaFuncSetAttribute(gemm_tn_partial_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gemm_tn_partial_kernel<<<(unsigned)nparts, 256, smem, st>>>((int)M, (int)N, K, chunk, A, a_ks,
                                                              a_ms, B, b_ks, b_ns, part.p);
  KS_CHECK_LAUNCH();
  reduce_partials_kernel<<<ceil_div_u(M * N, 256), 256, 0, st>>>(part.p, nparts, M * N, alpha, C);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

int sumsq_diff(cudaStream_t st, const double* a, const double* b, int64_t n, double* out) {
  int nb = (int)ks_min64((n + 1023) / 1024, 4 * (int64_t)num_sms());
  if (nb < 1) nb = 1;
  Scratch<double> part(nb, st);
  KS_REQUIRE(part.p, KS_ECUDA, "scratch allocation failed");
  sumsq_diff_partial_kernel<<<nb, 256, 0, st>>>(a, b, n, part.p);
  KS_CHECK_LAUNCH();
  sum_partials_kernel<<<1, 1024, 0, st>>>(part.p, nb, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

// Mode-n product sequence for (F_0 kron ... kron F_{nf-1}) b, rightmost factor first
// (kron.py:66-77).  Tensor view of b: (J_0, ..., J_{nf-1}, w).
int kron_mat_mul(cudaStream_t st, int nf, const double* const* F, const int64_t* rows,
                 const int64_t* cols, const double* b, int64_t w, double* out) {
  KS_REQUIRE(nf >= 1, KS_EINVAL, "need at least one factor");
  std::vector<int64_t> dims(nf);
  int64_t maxsz = 0, cur = w;
  for (int n = 0; n < nf; n++) dims[n] = cols[n];
  for (int n = 0; n < nf; n++) cur *= cols[n];
  maxsz = cur;
  {
    // running size as factors are applied right to left
    int64_t sz = cur;
    for (int n = nf - 1; n >= 0; n--) {
      sz = sz / cols[n] * rows[n];
      if (sz > maxsz) maxsz = sz;
    }
  }
  if (nf == 1) {
    // out (I x w) = F (I x J) b (J x w)
    return gemm(st, rows[0], w, cols[0], 1.0, F[0], cols[0], 1, 0, b, w, 1, 0, 0.0, out, w, 1, 0, 1);
  }
  Scratch<double> t0(maxsz, st), t1(maxsz, st);
  KS_REQUIRE(t0.p && t1.p, KS_ECUDA, "scratch allocation failed");
  const double* src = b;
  for (int n = nf - 1; n >= 0; n--) {
    int64_t P = 1, Q = w;
    for (int k = 0; k < n; k++) P *= dims[k];
    for (int k = n + 1; k < nf; k++) Q *= dims[k];
    const int64_t J = cols[n], I = rows[n];
    double* dst = (n == 0) ? out : ((src == t0.p) ? t1.p : t0.p);
    int rc;
    if (P >= Q) {
      // batch over q: Y[p, i, q] = sum_j X[p, j, q] F[i, j]
      rc = gemm(st, P, I, J, 1.0, src, J * Q, Q, 1, F[n], 1, J, 0, 0.0, dst, I * Q, Q, 1, Q);
    } else {
      // batch over p: Y_p (I x Q) = F (I x J) X_p (J x Q)
      rc = gemm(st, I, Q, J, 1.0, F[n], J, 1, 0, src, Q, 1, J * Q, 0.0, dst, Q, 1, I * Q, P);
    }
    if (rc) return rc;
    dims[n] = I;
    src = dst;
  }
  return KS_OK;
}

}  // namespace ks

// ---------------------------------------------------------------------------- C-ABI

extern "C" int ks_gemm(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t a_rs,
                       int64_t a_cs, int64_t a_bs, const double* B, int64_t b_rs, int64_t b_cs,
                       int64_t b_bs, double beta, double* C, int64_t c_rs, int64_t c_cs,
                       int64_t c_bs, int64_t batch, void* stream) {
  return ks::gemm((cudaStream_t)stream, M, N, K, alpha, A, a_rs, a_cs, a_bs, B, b_rs, b_cs, b_bs,
                  beta, C, c_rs, c_cs, c_bs, batch);
}

extern "C" int ks_gemm_tn_tall(int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                               int64_t a_ks, int64_t a_ms, const double* B, int64_t b_ks,
                               int64_t b_ns, double* C, void* stream) {
  return ks::gemm_tn_tall((cudaStream_t)stream, M, N, K, alpha, A, a_ks, a_ms, B, b_ks, b_ns, C);
}

extern "C" int ks_kron_mat_mul(int32_t nf, const double* const* factors, const int64_t* rows,
                               const int64_t* cols, const double* b, int64_t ncols, double* out,
                               void* stream) {
  return ks::kron_mat_mul((cudaStream_t)stream, nf, factors, rows, cols, b, ncols, out);
}

extern "C" int ks_sumsq_diff(const double* a, const double* b, int64_t n, double* out,
                             void* stream) {
  return ks::sumsq_diff((cudaStream_t)stream, a, b, n, out);
}

extern "C" int ks_check_finite_nonzero(const double* a, int64_t n, int32_t* flags, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_TRY_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int32_t), st));
  if (n <= 0) return KS_OK;
  int nb = (int)ks_min64((n + 255) / 256, 4 * (int64_t)ks::num_sms());
  check_kernel<<<nb, 256, 0, st>>>(a, n, flags);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

__global__ void gather_count_kernel(const double* __restrict__ b, const int64_t* __restrict__ idx,
                                    const int64_t* __restrict__ count, int64_t cap, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cap || t >= *count) return;
  out[t] = b[idx[t]];
}

extern "C" int ks_gather_count(const double* b, const int64_t* idx, const int64_t* count_dev, int64_t cap,
                               double* out, void* stream) {
  if (cap <= 0) return KS_OK;
  gather_count_kernel<<<ceil_div_u(cap, 256), 256, 0, (cudaStream_t)stream>>>(b, idx, count_dev, cap, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_gather(const double* b, const int64_t* idx, int64_t n, double* out,
                         void* stream) {
  if (n <= 0) return KS_OK;
  gather_kernel<<<ceil_div_u(n, 256), 256, 0, (cudaStream_t)stream>>>(b, idx, n, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}
