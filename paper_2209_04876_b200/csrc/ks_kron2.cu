// Two-factor n^2 passes of the exact solver and of the loss (reference kron.py:66-77 through
// solvers.py:314 and solvers.py:261).  The TMA/DMMA kernels of ks_kron2_dmma.cu run whenever
// the layout allows (16-byte aligned rows); the generic DFMA formulation below covers the rest.
#include "ks_common.cuh"

#include <cstdlib>

namespace ks {
int gemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t a_rs, int64_t a_cs, int64_t a_bs, const double* B, int64_t b_rs, int64_t b_cs,
         int64_t b_bs, double beta, double* C, int64_t c_rs, int64_t c_cs, int64_t c_bs,
         int64_t batch);
int gemm_tn_tall(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                 int64_t a_ks, int64_t a_ms, const double* B, int64_t b_ks, int64_t b_ns,
                 double* C);
int gemm_resid_sumsq(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha,
                     const double* A, int64_t a_rs, int64_t a_cs, const double* B, int64_t b_rs,
                     int64_t b_cs, const double* C, int64_t c_rs, int64_t c_cs, double* out);
int kron2_contract_dmma(cudaStream_t st, const double* L, const double* B, int64_t ldb, const double* R,
                        int64_t m, int64_t k, int p, int q, double* T, double* bsq);
int sumsq_diff(cudaStream_t st, const double* a, const double* b, int64_t n, double* out);
int kron2_residual_dmma(cudaStream_t st, const double* L, const double* X, const double* R, const double* B,
                        int64_t ldb, int64_t m, int64_t k, int p, int q, double* out);
}

static bool generic_forced() {
  const char* e = ks::env(ks::ENV_KRON2);
  return e && e[0] == 'g';
}

static int kron2_contract_impl(const double* L, const double* B, int64_t ldb, const double* R, int64_t m,
                               int64_t k, int32_t p, int32_t q, double* T, double* bsq, cudaStream_t st);

// T = L^T (B R)
extern "C" int ks_kron2_contract(const double* L, const double* B, int64_t ldb, const double* R,
                                 int64_t m, int64_t k, int32_t p, int32_t q, double* T,
                                 void* stream) {
  return kron2_contract_impl(L, B, ldb, R, m, k, p, q, T, nullptr, (cudaStream_t)stream);
}

// T = L^T (B R) and bsq[0] = ||B||^2 from the same pass over B
extern "C" int ks_kron2_contract_sumsq(const double* L, const double* B, int64_t ldb, const double* R,
                                       int64_t m, int64_t k, int32_t p, int32_t q, double* T, double* bsq,
                                       void* stream) {
  KS_REQUIRE(bsq, KS_EINVAL, "kron2_contract_sumsq needs an output for ||B||^2");
  return kron2_contract_impl(L, B, ldb, R, m, k, p, q, T, bsq, (cudaStream_t)stream);
}

static int kron2_contract_impl(const double* L, const double* B, int64_t ldb, const double* R, int64_t m,
                               int64_t k, int32_t p, int32_t q, double* T, double* bsq, cudaStream_t st) {
  KS_REQUIRE(p >= 1 && q >= 1 && p <= 128 && q <= 128, KS_ESIZE, "contract widths must be <= 128");
  if (!generic_forced()) {
    const int rc = ks::kron2_contract_dmma(st, L, B, ldb, R, m, k, p, q, T, bsq);
    if (rc >= 0) return rc;
  }
  if (bsq) {  // generic path: a separate pass (contiguous B only)
    KS_REQUIRE(ldb == k, KS_EINVAL, "kron2_contract_sumsq: generic path needs ldb == k");
    const int rc0 = ks::sumsq_diff(st, B, nullptr, m * k, bsq);
    if (rc0) return rc0;
  }
  ks::Scratch<double> P(m * q, st);
  KS_REQUIRE(P.p, KS_ECUDA, "scratch allocation failed");
  int rc = ks::gemm(st, m, q, k, 1.0, B, ldb, 1, 0, R, q, 1, 0, 0.0, P.p, q, 1, 0, 1);
  if (rc) return rc;
  return ks::gemm_tn_tall(st, p, q, m, 1.0, L, p, 1, P.p, q, 1, T);
}

// sum((L X R^T - B)^2)
extern "C" int ks_kron2_residual_sumsq(const double* L, const double* X, const double* R,
                                       const double* B, int64_t ldb, int64_t m, int64_t k, int32_t p,
                                       int32_t q, double* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!generic_forced()) {
    const int rc = ks::kron2_residual_dmma(st, L, X, R, B, ldb, m, k, p, q, out);
    if (rc >= 0) return rc;
  }
  ks::Scratch<double> Zt(k * p, st);
  KS_REQUIRE(Zt.p, KS_ECUDA, "scratch allocation failed");
  // Zt[j, a] = sum_c R[j, c] X[a, c]
  int rc = ks::gemm(st, k, p, q, 1.0, R, q, 1, 0, X, 1, q, 0, 0.0, Zt.p, p, 1, 0, 1);
  if (rc) return rc;
  // E[i, j] = sum_a L[i, a] Zt[j, a] - B[i, j]
  return ks::gemm_resid_sumsq(st, m, k, p, 1.0, L, p, 1, Zt.p, 1, p, B, ldb, 1, out);
}
