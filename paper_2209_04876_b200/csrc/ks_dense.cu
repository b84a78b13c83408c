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
