// Dense comparison baselines: materialised sketched rows of a Kronecker
// product for sketch_and_solve_ridge (reference kron.py:208-222 sketch_rows_of_kron,
// solvers.py:334-369).  out[t, c] = w[t] * prod_f A_f[j_f(t), c_f] with c unravelled C-order over
// the factor column counts (kron_rows' order: ((1 * a_0) * a_1) * ...).
#include "ks_common.cuh"

namespace {

struct Facs8 {
  const double* A[8];
  int64_t rows[8];
  int32_t cols[8];
};

__global__ void sketch_rows_kernel(Facs8 F, int nf, const int64_t* __restrict__ idx, int flat, const double* __restrict__ w,
                                   int64_t s, int64_t ncols, double* __restrict__ out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= s * ncols) return;
  const int64_t t = q / ncols;
  int64_t c = q - t * ncols;
  // unravel the column index (first factor slowest) and the row multi-index
  int64_t cst = ncols;
  int64_t frem = flat ? idx[t] : 0, fst = 1;
  if (flat)
    for (int f = 0; f < nf; f++) fst *= F.rows[f];
  double prod = 1.0;
  for (int f = 0; f < nf; f++) {
    cst /= F.cols[f];
    const int64_t cf = c / cst;
    c -= cf * cst;
    int64_t jf;
    if (flat) {
      fst /= F.rows[f];
      jf = frem / fst;
      frem -= jf * fst;
    } else {
      jf = idx[t * nf + f];
    }
    prod = prod * F.A[f][jf * F.cols[f] + cf];
  }
  out[q] = w[t] * prod;
}

}  // namespace

extern "C" int ks_sketch_rows(int32_t nf, const double* const* factors, const int64_t* rows, const int32_t* cols,
                              const int64_t* idx, int32_t flat, const double* w, int64_t s, double* out, void* stream) {
  KS_REQUIRE(nf >= 1 && nf <= 8, KS_EINVAL, "1..8 factors supported");
  Facs8 F{};
  int64_t ncols = 1;
  for (int f = 0; f < nf; f++) {
    F.A[f] = factors[f];
    F.rows[f] = rows[f];
    F.cols[f] = cols[f];
    ncols *= cols[f];
  }
  if (s <= 0 || ncols <= 0) return KS_OK;
  sketch_rows_kernel<<<ceil_div_u(s * ncols, 256), 256, 0, (cudaStream_t)stream>>>(F, nf, idx, flat, w, s, ncols, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

// Explicit Kronecker product of two row-major matrices (tensor.py:186-198 for two factors; the
// materialised right group of the three-factor KronMatMul / loss passes, solvers.py:314, :261):
// C[(i k_rows + j), (a q + c)] = A[i, a] B[j, c].  Two consecutive outputs per thread (16-byte
// stores when aligned); A and B are small and stay in L1/L2.
namespace {
__global__ void kron_explicit2_kernel(const double* __restrict__ A, int64_t m, int32_t p, const double* __restrict__ B,
                                      int64_t k, int32_t q, double* __restrict__ C) {
  const int64_t ncols = (int64_t)p * q, total = m * k * ncols;
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (e >= total) return;
  auto at = [&](int64_t f) {  // element f of C
    const int64_t r = f / ncols, col = f - r * ncols;
    const int64_t i = r / k, j = r - i * k;
    const int32_t a = (int32_t)(col / q), c = (int32_t)(col - (int64_t)a * q);
    return __ldg(&A[i * p + a]) * __ldg(&B[j * q + c]);
  };
  const double v0 = at(e);
  if (e + 1 < total) {
    const double v1 = at(e + 1);
    if (((uintptr_t)(C + e) & 15) == 0) *reinterpret_cast<double2*>(C + e) = make_double2(v0, v1);
    else { C[e] = v0; C[e + 1] = v1; }
  } else {
    C[e] = v0;
  }
}

}  // namespace

extern "C" int ks_kron_explicit2(const double* A, int64_t m, int32_t p, const double* B, int64_t k, int32_t q,
                                 double* C, void* stream) {
  KS_REQUIRE(m >= 0 && k >= 0 && p >= 1 && q >= 1, KS_EINVAL, "kron_explicit2: bad shapes");
  const int64_t pairs = (m * k * (int64_t)p * q + 1) / 2;
  if (pairs == 0) return KS_OK;
  kron_explicit2_kernel<<<ceil_div_u(pairs, 256), 256, 0, (cudaStream_t)stream>>>(A, m, p, B, k, q, C);
  KS_CHECK_LAUNCH();
  return KS_OK;
}


// The spectral-row sample of leverage.py:235-252 as used by fast_kronecker_regression
// (solvers.py:424-427): out[t, :] = (w[t] * A[idx[t], :]) / divisor, two roundings in the
// reference's order (the weighted gather, then the division by sqrt(1 - eps_two)).
namespace {
__global__ void scaled_row_gather_kernel(const double* __restrict__ A, int64_t n, int32_t d,
                                         const int64_t* __restrict__ idx, const double* __restrict__ w, int64_t m,
                                         double divisor, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * d) return;
  const int64_t t = e / d;
  const int32_t c = (int32_t)(e - t * d);
  const int64_t r = __ldg(&idx[t]);
  out[e] = __ddiv_rn(__dmul_rn(__ldg(&w[t]), __ldg(&A[r * d + c])), divisor);
}
}  // namespace

extern "C" int ks_scaled_row_gather(const double* A, int64_t n, int32_t d, const int64_t* idx, const double* w,
                                    int64_t m, double divisor, double* out, void* stream) {
  KS_REQUIRE(n >= 0 && m >= 0 && d >= 1 && divisor != 0.0, KS_EINVAL, "scaled_row_gather: bad arguments");
  if (m == 0) return KS_OK;
  scaled_row_gather_kernel<<<ceil_div_u(m * d, 256), 256, 0, (cudaStream_t)stream>>>(A, n, d, idx, w, m, divisor, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}
