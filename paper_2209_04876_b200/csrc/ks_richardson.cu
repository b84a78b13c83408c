// Device-resident preconditioned Richardson iteration of fast_kronecker_regression.
//
// Reference semantics (solvers.py:201-248): x0 = 0; scale = ||P rhs||; tol = residual_tol *
// max(scale, tiny); for it < max_iters: step = P(H x - rhs); history.append(||step||);
// break if ||step|| <= tol; raise if the last 6 norms rise strictly and grow > 10x;
// x -= damping * step.  H x = (SK)^T S (SK) x + lam x (solvers.py:454-456) with the sketched
// operator of kron.py:258-354; P = KronPreconditioner.apply (solvers.py:180-183).
//
// Every iteration runs on the stream without host round trips; the loop state (status,
// iteration count, residual history) lives in device memory and is copied back once.
#include "ks_common.cuh"

#include <cfloat>
#include <cstdlib>

namespace ks {
int sketched_gram_partials(cudaStream_t st, const ks_sketch_view* sk, const double* X,
                           const double* bv, const int64_t* perm, int mode, double* part,
                           int64_t* nparts_out);
int64_t sketched_partials_count(const ks_sketch_view* sk);
bool persistent_supported(int dL, int dR);
int richardson_persistent(cudaStream_t st, const ks_sketch_view* sk, const double* VL, const double* VR,
                          const double* dinv, const double* wL, const double* wR, double* rhs, bool rhs_in_kernel,
                          const double* b_at, const int64_t* perm, double lam, double damping, int max_iters,
                          double residual_tol, double* x, double* hist, int* iters, int* hist_len, int* status,
                          const int64_t* counts_dev, int* state_dev, bool eig_mode, const void* plan_ws);
int64_t richardson_plan_bytes(int64_t ul_cap, int64_t nnz_cap);
int richardson_plan(cudaStream_t st, const ks_sketch_view* sk, const int64_t* counts_dev, void* plan_ws);
}

namespace {

enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_DIVERGED = 2 };

struct LoopState {
  int status;
  int iters;
  int hist_len;
  int pad;
  double tol;
};

// Two-level fixed-order reduction of the block partials (deterministic): split s of gridDim.y sums
// partials [s*per, (s+1)*per) with Neumaier compensation into part2[s]; residual_kernel then sums
// the splits in order.  (One level over ~2000 partials of d^2 = 16384 doubles is a latency-bound
// chain per thread.)
__global__ void partial_split_kernel(const double* __restrict__ part, int64_t nparts, int64_t per, int64_t count,
                                     double* __restrict__ part2, const LoopState* __restrict__ ls) {
  if (ls && ls->status != ST_RUNNING) return;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  const int64_t p0 = (int64_t)blockIdx.y * per, p1 = ks_min64(nparts, p0 + per);
  double s = 0.0, c = 0.0;
  for (int64_t p = p0; p < p1; p++) {
    const double v = part[p * count + e];
    const double t = s + v;
    c += (fabs(s) >= fabs(v)) ? ((s - t) + v) : ((v - t) + s);
    s = t;
  }
  part2[(int64_t)blockIdx.y * count + e] = s + c;
}

// R = sum_p part[p] + lam X - rhs
__global__ void residual_kernel(const double* __restrict__ part, int64_t nparts, int64_t count,
                                const double* __restrict__ X, double lam,
                                const double* __restrict__ rhs, double* __restrict__ R,
                                const LoopState* __restrict__ ls) {
  if (ls && ls->status != ST_RUNNING) return;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  // Neumaier-compensated sum of the block partials (fixed order, deterministic)
  double s = 0.0, c = 0.0;
  for (int64_t p = 0; p < nparts; p++) {
    const double v = part[p * count + e];
    const double t = s + v;
    c += (fabs(s) >= fabs(v)) ? ((s - t) + v) : ((v - t) + s);
    s = t;
  }
  s += c;
  // (G + lam x) - rhs, in the reference's association and rounding
  R[e] = __dsub_rn(__dadd_rn(s, __dmul_rn(lam, X[e])), rhs[e]);
}

// T[r, :] = dinv[r, :] * ((VL^T R)[r, :] VR)     one block per row r
__global__ void precond_a_kernel(const double* __restrict__ VL, const double* __restrict__ VR, int dL,
                                 int dR, const double* __restrict__ dinv, const double* __restrict__ R,
                                 double* __restrict__ T, const LoopState* __restrict__ ls) {
  if (ls && ls->status != ST_RUNNING) return;
  __shared__ double t1[128];
  const int r = blockIdx.x;
  for (int j = threadIdx.x; j < dR; j += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < dL; k++) s = fma(VL[k * dL + r], R[k * dR + j], s);
    t1[j] = s;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < dR; c += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < dR; j++) s = fma(t1[j], VR[j * dR + c], s);
    T[r * dR + c] = s * dinv[r * dR + c];
  }
}

// Y[r, :] = (VL T)[r, :] VR^T; rowsq[r] = ||Y[r, :]||^2       one block per row r
__global__ void precond_b_kernel(const double* __restrict__ VL, const double* __restrict__ VRt, int dL,
                                 int dR, const double* __restrict__ T, double* __restrict__ Y,
                                 double* __restrict__ rowsq, const LoopState* __restrict__ ls) {
  if (ls && ls->status != ST_RUNNING) return;
  __shared__ double s1[128];
  __shared__ double red[32];
  const int r = blockIdx.x;
  for (int j = threadIdx.x; j < dR; j += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < dL; k++) s = fma(VL[r * dL + k], T[k * dR + j], s);
    s1[j] = s;
  }
  __syncthreads();
  double sq = 0.0;
  for (int c = threadIdx.x; c < dR; c += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < dR; j++) s = fma(s1[j], VRt[j * dR + c], s);
    Y[r * dR + c] = s;
    sq = fma(s, s, sq);
  }
  sq = block_sum(sq, red);
  if (threadIdx.x == 0 && rowsq) rowsq[r] = sq;
}

__global__ void transpose_sq_kernel(const double* __restrict__ a, int d, double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d * d) return;
  const int i = e / d, j = e - i * d;
  out[j * d + i] = a[e];
}

__global__ void init_state_kernel(LoopState* ls, const double* __restrict__ rowsq, int dL,
                                  double residual_tol, double* __restrict__ x, int64_t count) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < count) x[e] = 0.0;
  if (e == 0) {
    double s = 0.0;
    for (int r = 0; r < dL; r++) s += rowsq[r];
    const double scale = sqrt(s);
    ls->status = ST_RUNNING;
    ls->iters = 0;
    ls->hist_len = 0;
    ls->tol = residual_tol * fmax(scale, DBL_MIN);
  }
}

// norm, history, stopping rules, x update (one block)
__global__ void update_kernel(LoopState* ls, const double* __restrict__ rowsq, int dL, int it,
                              double* __restrict__ hist, const double* __restrict__ step,
                              double damping, double* __restrict__ x, int64_t count) {
  __shared__ int s_go;
  if (threadIdx.x == 0) {
    s_go = 0;
    if (ls->status == ST_RUNNING) {
      double s = 0.0;
      for (int r = 0; r < dL; r++) s += rowsq[r];
      const double nrm = sqrt(s);
      hist[it] = nrm;
      ls->hist_len = it + 1;
      const int h = it + 1;
      if (nrm <= ls->tol) {
        ls->status = ST_CONVERGED;
      } else {
        bool diverged = false;
        if (h > 5) {
          bool inc = true;
          for (int i = h - 6; i < h - 1; i++) inc &= hist[i + 1] > hist[i];
          diverged = inc && (hist[h - 1] > 10.0 * hist[h - 6]);
        }
        if (diverged) {
          ls->status = ST_DIVERGED;
        } else {
          s_go = 1;
          ls->iters = it + 1;
        }
      }
    }
  }
  __syncthreads();
  if (!s_go) return;
  for (int64_t e = threadIdx.x; e < count; e += blockDim.x) x[e] = __dsub_rn(x[e], __dmul_rn(damping, step[e]));
}

}  // namespace

namespace ks {

int precond_apply(cudaStream_t st, const double* VL, const double* VR, const double* VRt, int dL,
                  int dR, const double* dinv, const double* r, double* tmp, double* y,
                  double* rowsq, const void* ls) {
  const int thr = dR >= 128 ? 128 : (dR >= 64 ? 64 : 32);
  precond_a_kernel<<<dL, thr, 0, st>>>(VL, VR, dL, dR, dinv, r, tmp, (const LoopState*)ls);
  KS_CHECK_LAUNCH();
  precond_b_kernel<<<dL, thr, 0, st>>>(VL, VRt, dL, dR, tmp, y, rowsq, (const LoopState*)ls);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

}  // namespace ks

extern "C" int ks_kron_precond_apply(const double* VL, const double* VR, int32_t dL, int32_t dR,
                                     const double* dinv, const double* r, double* y, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_REQUIRE(dL >= 1 && dR >= 1 && dL <= 128 && dR <= 128, KS_ESIZE, "preconditioner dims must be <= 128");
  ks::Scratch<double> VRt((int64_t)dR * dR, st), tmp((int64_t)dL * dR, st);
  KS_REQUIRE(VRt.p && tmp.p, KS_ECUDA, "scratch allocation failed");
  transpose_sq_kernel<<<ceil_div_u((int64_t)dR * dR, 256), 256, 0, st>>>(VR, dR, VRt.p);
  KS_CHECK_LAUNCH();
  return ks::precond_apply(st, VL, VR, VRt.p, dL, dR, dinv, r, tmp.p, y, nullptr, nullptr);
}

extern "C" int ks_richardson_sketched(const ks_sketch_view* sk, const double* VL, const double* VR,
                                      const double* dinv, const double* rhs, double lam,
                                      double damping, int32_t max_iters, double residual_tol,
                                      double* x, double* hist, int32_t* iters, int32_t* hist_len,
                                      void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int dL = sk->dL, dR = sk->dR;
  KS_REQUIRE(dL >= 1 && dR >= 1 && dL <= 128 && dR <= 128, KS_ESIZE, "group widths must be <= 128");
  const char* mode = ks::env(ks::ENV_RICHARDSON);
  const bool force_multi = mode && mode[0] == 'm';
  if (!force_multi && sk->nnz > 0 && ks::persistent_supported(dL, dR) && max_iters <= 1024) {
    int status = 0;
    int it = 0, hl = 0;
    int rc = ks::richardson_persistent(st, sk, VL, VR, dinv, nullptr, nullptr, const_cast<double*>(rhs), false,
                                       nullptr, nullptr, lam, damping, max_iters, residual_tol, x, hist, &it, &hl,
                                       &status, nullptr, nullptr, false, nullptr);
    if (rc) return rc;
    *iters = it;
    *hist_len = hl;
    if (status == 2) {
      ks::set_error("Richardson iteration diverged");
      return KS_EDIVERGED;
    }
    return KS_OK;
  }
  const int64_t count = (int64_t)dL * dR;
  const int64_t np = ks::sketched_partials_count(sk);
  ks::Scratch<double> part(np * count + 1, st), part2(32 * count, st), R(count, st), T(count, st), step(count, st);
  ks::Scratch<double> rowsq(dL, st), VRt((int64_t)dR * dR, st);
  ks::Scratch<LoopState> ls(1, st);
  KS_REQUIRE(part.p && part2.p && R.p && T.p && step.p && rowsq.p && VRt.p && ls.p, KS_ECUDA,
             "scratch allocation failed");
  transpose_sq_kernel<<<ceil_div_u((int64_t)dR * dR, 256), 256, 0, st>>>(VR, dR, VRt.p);
  KS_CHECK_LAUNCH();
  // scale = ||P rhs||
  int rc = ks::precond_apply(st, VL, VR, VRt.p, dL, dR, dinv, rhs, T.p, step.p, rowsq.p, nullptr);
  if (rc) return rc;
  init_state_kernel<<<ceil_div_u(count, 256), 256, 0, st>>>(ls.p, rowsq.p, dL, residual_tol, x, count);
  KS_CHECK_LAUNCH();
  for (int it = 0; it < max_iters; it++) {
    int64_t nb = 0;
    rc = ks::sketched_gram_partials(st, sk, x, nullptr, nullptr, 1, part.p, &nb);
    if (rc) return rc;
    if (nb > 64) {  // two levels: 32 splits, then the splits in order
      const int64_t per = (nb + 31) / 32, ns = (nb + per - 1) / per;
      partial_split_kernel<<<dim3(ceil_div_u(count, 256), (unsigned)ns), 256, 0, st>>>(part.p, nb, per, count,
                                                                                       part2.p, ls.p);
      KS_CHECK_LAUNCH();
      residual_kernel<<<ceil_div_u(count, 256), 256, 0, st>>>(part2.p, ns, count, x, lam, rhs, R.p, ls.p);
    } else {
      residual_kernel<<<ceil_div_u(count, 256), 256, 0, st>>>(part.p, nb, count, x, lam, rhs, R.p, ls.p);
    }
    KS_CHECK_LAUNCH();
    rc = ks::precond_apply(st, VL, VR, VRt.p, dL, dR, dinv, R.p, T.p, step.p, rowsq.p, ls.p);
    if (rc) return rc;
    update_kernel<<<1, 1024, 0, st>>>(ls.p, rowsq.p, dL, it, hist, step.p, damping, x, count);
    KS_CHECK_LAUNCH();
  }
  LoopState h{};
  KS_TRY_CUDA(cudaMemcpyAsync(&h, ls.p, sizeof(LoopState), cudaMemcpyDeviceToHost, st));
  KS_TRY_CUDA(cudaStreamSynchronize(st));
  *iters = h.iters;
  *hist_len = h.hist_len;
  if (h.status == ST_DIVERGED) {
    ks::set_error("Richardson iteration diverged");
    return KS_EDIVERGED;
  }
  return KS_OK;
}

// Fused form for single-factor groups on the persistent path: the right-hand side
// (SK)^T S b (solvers.py:455) is built inside the loop kernel from b_at (b at the sparse-diagonal
// rows) and returned in rhs_out; dinv (may be null) defaults to pseudo-reciprocal(wL x wR + lam).
extern "C" int ks_richardson_fused(const ks_sketch_view* sk, const int64_t* perm, const double* b_at,
                                   const double* VL, const double* wL, const double* VR, const double* wR,
                                   const double* dinv, double lam, double damping, int32_t max_iters,
                                   double residual_tol, double* x, double* hist, double* rhs_out, int32_t* iters,
                                   int32_t* hist_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int dL = sk->dL, dR = sk->dR;
  KS_REQUIRE(sk->nnz > 0 && ks::persistent_supported(dL, dR) && max_iters <= 1024, KS_ESIZE,
             "fused Richardson needs dL, dR in {16, 32, 64}, nnz > 0 and <= 1024 iterations");
  KS_REQUIRE(dinv || (wL && wR), KS_EINVAL, "need dinv or both eigenvalue vectors");
  int status = 0, it = 0, hl = 0;
  int rc = ks::richardson_persistent(st, sk, VL, VR, dinv, wL, wR, rhs_out, true, b_at, perm, lam, damping,
                                     max_iters, residual_tol, x, hist, &it, &hl, &status, nullptr, nullptr,
                                     !ks::env(ks::ENV_NO_EIGBASIS), nullptr);
  if (rc) return rc;
  *iters = it;
  *hist_len = hl;
  if (status == 2) {
    ks::set_error("Richardson iteration diverged");
    return KS_EDIVERGED;
  }
  return KS_OK;
}

// Asynchronous fused form for CUDA-graph capture: the view's nnz / u_left are capacities and the
// real counts are read on the device from counts_dev ([nnz, u_left]); the loop state
// [status (1 converged, 2 diverged), iterations, history length] goes to state_dev.  No host
// synchronisation.
extern "C" int64_t ks_richardson_plan_bytes(int64_t u_left_cap, int64_t nnz_cap) {
  return ks::richardson_plan_bytes(u_left_cap, nnz_cap);
}

extern "C" int ks_richardson_plan_async(const ks_sketch_view* sk, const int64_t* counts_dev, void* plan_ws,
                                        void* stream) {
  KS_REQUIRE(plan_ws && sk->nnz > 0, KS_EINVAL, "need a plan workspace and a nonempty sketch");
  return ks::richardson_plan((cudaStream_t)stream, sk, counts_dev, plan_ws);
}

extern "C" int ks_richardson_fused_async(const ks_sketch_view* sk, const int64_t* counts_dev, const int64_t* perm,
                                         const double* b_at, const double* VL, const double* wL, const double* VR,
                                         const double* wR, const double* dinv, double lam, double damping,
                                         int32_t max_iters, double residual_tol, double* x, double* hist,
                                         double* rhs_out, int32_t* state_dev, const void* plan_ws, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int dL = sk->dL, dR = sk->dR;
  KS_REQUIRE(sk->nnz > 0 && ks::persistent_supported(dL, dR) && max_iters <= 1024, KS_ESIZE,
             "fused Richardson needs dL, dR in {16, 32, 64}, nnz > 0 and <= 1024 iterations");
  KS_REQUIRE(dinv || (wL && wR), KS_EINVAL, "need dinv or both eigenvalue vectors");
  KS_REQUIRE(counts_dev && state_dev, KS_EINVAL, "need device counts and a device state buffer");
  int status = 0, it = 0, hl = 0;
  return ks::richardson_persistent(st, sk, VL, VR, dinv, wL, wR, rhs_out, true, b_at, perm, lam, damping, max_iters,
                                   residual_tol, x, hist, &it, &hl, &status, counts_dev, state_dev,
                                   !ks::env(ks::ENV_NO_EIGBASIS), plan_ws);
}
