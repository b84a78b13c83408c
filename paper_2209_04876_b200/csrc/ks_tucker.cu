// Tucker-ALS factor-matrix updates on the device.
//
// Reference: pkg/src/kronsolve/tucker.py
//   * build_factor_workspace (:217-280) + _power_iteration (:283-313)  -> factor_workspace_kernel
//     (one CTA: 100-step power iteration on the constrained Gram, penalty weight, Kronecker-
//     diagonal base inverse, Woodbury correction matrices; the R_n x R_n core inverse is
//     ks_inverse_small)
//   * fast_factor_matrix_update (:316-379)                               -> factor_rows_kernel
//     (one CTA per factor row: gathers its sampled entries of the unfolding, builds the sketched
//     right-hand side and runs the whole preconditioned Richardson solve of the penalised
//     constrained row problem in shared memory, then projects and maps through (G^T)^+)
//   * FactorUpdateWorkspace.apply / apply_base / apply_penalized_normal (:185-214) -> ws_apply_kernel
//   * initial_model's np.linalg.qr (:400-409)                            -> qr_explicit_kernel
//     (Householder QR with LAPACK's dgeqrf/dorg2r sign convention, explicit thin Q)
//   * per-row random streams (SeedSequence(seed).spawn(I_n), :361-369) -> draws_rows_kernel turns
//     the per-row PCG64 uniforms into product-sampler draws + weights (leverage.py:196-231) with
//     the row index prepended, so ks_sketch_diag dedups every row's sketch in one sort.
//
// Layout: the other factors' row-major matrices A_m (I_m x R_m); a vector over the leftover
// Kronecker columns is indexed C-order by (r_0, ..., r_{M-1}) (first other factor slowest), as
// in kron.py.  Inside a CTA the sketched operator uses the two-group scheme of kron.py:258-354
// with the left group = the first other factor: the row's samples (sorted by flat index) form
// contiguous groups of equal first-factor row, so K_S x = {v_t (Y_g . R_t)} with
// Y_g = A_0[j_g]^T X and K_S^T c = sum_g A_0[j_g] (x) (sum_{t in g} c_t R_t).
#include "ks_common.cuh"

namespace {

constexpr int FT = 256;   // threads per CTA
constexpr int MAXM = 4;   // other factors (model order <= 5)

struct Others {
  const double* A[MAXM];  // I_m x R_m
  const double* V[MAXM];  // Gram eigenvectors, R_m x R_m (column j = vector j)
  const double* G[MAXM];  // Gram matrices, R_m x R_m
  const double* E[MAXM];  // Gram eigenvalues, R_m
  int64_t I[MAXM];
  int32_t R[MAXM];
  int32_t M;
  int32_t Rrest, Rright;
  int64_t Irest, Iright;
};

__device__ __forceinline__ int64_t mode_stride(const Others& o, int m) {
  int64_t st = 1;
  for (int k = m + 1; k < o.M; k++) st *= o.R[k];
  return st;
}

// Sum over k < n of f(k, acc) with 8 independent accumulators (memory-level parallelism for the
// L2-latency-bound gathers), combined in a fixed order.
template <class F>
__device__ __forceinline__ double sum8(int n, F f) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0, s5 = 0.0, s6 = 0.0, s7 = 0.0;
  int k = 0;
  for (; k + 8 <= n; k += 8) {
    s0 = f(k, s0); s1 = f(k + 1, s1); s2 = f(k + 2, s2); s3 = f(k + 3, s3);
    s4 = f(k + 4, s4); s5 = f(k + 5, s5); s6 = f(k + 6, s6); s7 = f(k + 7, s7);
  }
  for (; k < n; k++) s0 = f(k, s0);
  return ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7));
}

// dst = (I (x) .. (x) F (x) .. (x) I) src along mode m; F(i,k) = trans ? F[k*R+i] : F[i*R+k].
__device__ void mode_product(const double* __restrict__ F, int R, int64_t st, bool trans,
                             const double* src, double* dst, int n) {
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const int im = (int)((r / st) % R);
    const int64_t base = r - (int64_t)im * st;
    dst[r] = sum8(R, [&](int k, double acc) {
      const double f = trans ? __ldg(F + (int64_t)k * R + im) : __ldg(F + (int64_t)im * R + k);
      return fma(f, src[base + (int64_t)k * st], acc);
    });
  }
}

// (F_0 (x) ... (x) F_{M-1}) src with F_m = mats[m] (or its transpose); ping-pong through p0/p1
// (src may be p0 or p1 or neither).  Returns the buffer holding the result.  Ends synced.
__device__ double* kron_apply(const Others& o, const double* const* mats, bool trans, const double* src,
                              double* p0, double* p1) {
  const double* cur = src;
  double* dst = nullptr;
  for (int m = o.M - 1; m >= 0; m--) {  // rightmost factor first, like kron_vec_square
    dst = (cur == p0) ? p1 : p0;
    mode_product(mats[m], o.R[m], mode_stride(o, m), trans, cur, dst, o.Rrest);
    __syncthreads();
    cur = dst;
  }
  return dst;
}

// y[k] = sum_l P[k*sk + l*sl] x[l] for k < K (one warp per output, fixed order).  No sync.
__device__ void warp_dots(int K, int L, const double* __restrict__ P, int64_t sk, int64_t sl,
                          const double* x, double* y) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = wid; k < K; k += nw) {
    double acc = 0.0;
    for (int l = lane; l < L; l += 32) acc = fma(__ldg(P + (int64_t)k * sk + (int64_t)l * sl), x[l], acc);
    acc = warp_sum(acc);
    if (lane == 0) y[k] = acc;
  }
}

__device__ __forceinline__ double thread_dot(int L, const double* __restrict__ P, int64_t sl, const double* x) {
  return sum8(L, [&](int l, double acc) { return fma(__ldg(P + (int64_t)l * sl), x[l], acc); });
}

__device__ double block_sumsq(const double* v, int n, double* red) {
  double a = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) a = fma(v[r], v[r], a);
  return block_sum(a, red);
}

__device__ double block_dot(const double* u, const double* v, int n, double* red) {
  double a = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) a = fma(u[r], v[r], a);
  return block_sum(a, red);
}

// ------------------------------------------------------------------ workspace (one CTA)

struct WsArgs {
  Others o;
  int32_t Rn;
  const double* gn;   // R_n x R_rest  (core unfolding G)
  const double* gnp;  // R_rest x R_n  (G^+)
  double lam, eps;
  const double* v0;   // R_rest standard normals (default_rng(0), tucker.py:298)
  double* wout;       // [0] = w, [1] = power-iteration estimate ||.||^2
  double* bdiag;      // R_rest
  double* right;      // R_n x R_rest
  double* cm;         // R_n x R_n  (I + right p0), inverted by the caller
  int32_t* flags;     // [0] |= 1: non-finite power iterate
};

__global__ void __launch_bounds__(FT) factor_workspace_kernel(WsArgs a) {
  extern __shared__ double sm[];
  const Others& o = a.o;
  const int n = o.Rrest, Rn = a.Rn;
  double* v = sm;
  double* u = v + n;
  double* t = u + n;
  double* p0 = t + n;
  double* p1 = p0 + n;
  double* s0 = p1 + n;      // R_n
  double* s1 = s0 + Rn;     // R_n
  double* red = s1 + Rn;    // 32
  __shared__ int s_stop;

  // v = v0 / ||v0||
  for (int r = threadIdx.x; r < n; r += blockDim.x) v[r] = a.v0[r];
  __syncthreads();
  const double n0 = sqrt(block_sumsq(v, n, red));
  for (int r = threadIdx.x; r < n; r += blockDim.x) v[r] = v[r] / n0;
  __syncthreads();

  double est = 0.0, best = 0.0;
  for (int it = 0; it < 100; it++) {
    // u = v - G^T (G^T)^+ v
    warp_dots(Rn, n, a.gnp, 1, Rn, v, s0);
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x) u[r] = v[r] - thread_dot(Rn, a.gn + r, n, s0);
    __syncthreads();
    // t = (kron of Grams) u + lam G^+ (G^+^T u)
    double* ku = kron_apply(o, o.G, false, u, p0, p1);
    warp_dots(Rn, n, a.gnp, 1, Rn, u, s1);
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x) t[r] = ku[r] + a.lam * thread_dot(Rn, a.gnp + (int64_t)r * Rn, 1, s1);
    __syncthreads();
    // out = t - G^T (G^T)^+ t  (into u)
    warp_dots(Rn, n, a.gnp, 1, Rn, t, s0);
    __syncthreads();
    int bad = 0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      const double y = t[r] - thread_dot(Rn, a.gn + r, n, s0);
      u[r] = y;
      bad |= !isfinite(y);
    }
    bad = __syncthreads_or(bad);
    if (bad) {
      if (threadIdx.x == 0) a.flags[0] |= 1;
      return;
    }
    const double nrm = sqrt(block_sumsq(u, n, red));
    if (nrm <= 1e-300) {
      best = 0.0;
      break;
    }
    const double nw = block_dot(v, u, n, red);
    best = fmax(best, nw);
    for (int r = threadIdx.x; r < n; r += blockDim.x) v[r] = u[r] / nrm;
    if (threadIdx.x == 0) s_stop = fabs(nw - est) <= 1e-6 * fmax(1e-30, fabs(nw));
    __syncthreads();
    if (s_stop) break;
    est = nw;
  }
  const double w = (1.0 + 12.0 / a.eps) * best * 1.05;
  if (threadIdx.x == 0) {
    a.wout[0] = w;
    a.wout[1] = best;
  }
  // base_diag = pseudo_reciprocal(kron(eigenvalues) + w)
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    // kron(e_0, e_1, ...)[r] = ((e_0[r_0] e_1[r_1]) e_2[r_2]) ...
    double e = 1.0;
    int64_t st = n, rem = r;
    for (int m = 0; m < o.M; m++) {
      st /= o.R[m];
      const int rm = (int)(rem / st);
      rem -= (int64_t)rm * st;
      e = (m == 0) ? o.E[0][rm] : e * o.E[m][rm];
    }
    const double d = e + w;
    a.bdiag[r] = d > 0.0 ? 1.0 / d : 0.0;
  }
  // correction_right = lam (G^T)^+ - w G
  for (int64_t q = threadIdx.x; q < (int64_t)Rn * n; q += blockDim.x) {
    const int k = (int)(q / n), r = (int)(q % n);
    a.right[q] = a.lam * a.gnp[(int64_t)r * Rn + k] - w * a.gn[q];
  }
  __syncthreads();
  // cm = I + right . (V diag V^T) G^+, one column of G^+ at a time
  for (int c = 0; c < Rn; c++) {
    for (int r = threadIdx.x; r < n; r += blockDim.x) t[r] = a.gnp[(int64_t)r * Rn + c];
    __syncthreads();
    double* q = kron_apply(o, o.V, true, t, p0, p1);
    for (int r = threadIdx.x; r < n; r += blockDim.x) q[r] = a.bdiag[r] * q[r];
    __syncthreads();
    double* pc = kron_apply(o, o.V, false, q, p0, p1);
    warp_dots(Rn, n, a.right, n, 1, pc, s0);
    __syncthreads();
    if (threadIdx.x < Rn) a.cm[(int64_t)threadIdx.x * Rn + c] = (threadIdx.x == c ? 1.0 : 0.0) + s0[threadIdx.x];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ shared operator pieces

struct Ws {
  const double* gn;     // R_n x R_rest
  const double* gnp;    // R_rest x R_n
  const double* mid;    // R_n x R_n
  const double* right;  // R_n x R_rest
  const double* bdiag;  // R_rest
  const double* wdev;   // [0] = w
  double lam;
  int32_t Rn;
};

// out = apply_base(src) = V diag(bdiag) V^T src.  Uses p0/p1; returns the result buffer.
__device__ double* apply_base(const Others& o, const Ws& ws, const double* src, double* p0, double* p1) {
  double* q = kron_apply(o, o.V, true, src, p0, p1);
  for (int r = threadIdx.x; r < o.Rrest; r += blockDim.x) q[r] = q[r] * ws.bdiag[r];
  __syncthreads();
  return kron_apply(o, o.V, false, q, p0, p1);
}

// dst = workspace.apply(src) (tucker.py:194-200).  src must not alias base/tmp/p0/p1/dst.
__device__ void ws_apply(const Others& o, const Ws& ws, const double* src, double* base, double* tmp,
                         double* p0, double* p1, double* s0, double* s1, double* dst) {
  const int n = o.Rrest, Rn = ws.Rn;
  double* b = apply_base(o, ws, src, p0, p1);
  for (int r = threadIdx.x; r < n; r += blockDim.x) base[r] = b[r];
  __syncthreads();
  warp_dots(Rn, n, ws.right, n, 1, base, s0);  // corr = right @ base
  __syncthreads();
  if (threadIdx.x < Rn) s1[threadIdx.x] = thread_dot(Rn, ws.mid + (int64_t)threadIdx.x * Rn, 1, s0);
  __syncthreads();
  for (int r = threadIdx.x; r < n; r += blockDim.x) tmp[r] = thread_dot(Rn, ws.gnp + (int64_t)r * Rn, 1, s1);
  __syncthreads();
  double* c = apply_base(o, ws, tmp, p0, p1);
  for (int r = threadIdx.x; r < n; r += blockDim.x) dst[r] = base[r] - c[r];
  __syncthreads();
}

// t += w z + lam G^+ ((G^T)^+ z) - w G^+ (G z), in the reference's order (tucker.py:371-376).
__device__ void penalty_terms(const Others& o, const Ws& ws, double w, const double* z, double* t,
                              double* s0, double* s1) {
  const int n = o.Rrest, Rn = ws.Rn;
  warp_dots(Rn, n, ws.gnp, 1, Rn, z, s0);  // (G^T)^+ z
  warp_dots(Rn, n, ws.gn, n, 1, z, s1);    // G z
  __syncthreads();
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const double* row = ws.gnp + (int64_t)r * Rn;
    const double pu = thread_dot(Rn, row, 1, s0), pq = thread_dot(Rn, row, 1, s1);
    t[r] = ((t[r] + w * z[r]) + ws.lam * pu) - w * pq;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ per-row Richardson (one CTA/row)

struct RowArgs {
  Others o;
  Ws ws;
  const int64_t* sd_idx;  // composite keys row*I_rest + flat (or flat only when shared)
  const double* sd_val;
  int64_t nnz;
  int32_t shared;
  const double* x;        // data tensor
  int64_t xs_n;           // stride of mode n
  int64_t xs[MAXM];       // strides of the other modes
  double* kr;             // Khatri-Rao right rows (nnz x R_right) when M >= 3
  double damping;
  int32_t max_iters;
  double residual_tol;
  int32_t cap;            // max samples per row
  int32_t ucap;           // max groups per row
  double* out;            // I_n x R_n
  int32_t* iters;         // I_n
  int32_t* flags;         // I_n: 1 = diverged, 2 = too many samples
  double* hist;           // I_n x max_iters (may be null)
};

// Right-group row element rr of sample t: A_1[j_t] (M = 2), a Khatri-Rao row (M >= 3), 1 (M = 1).
struct RightRows {
  const double* base;  // A_1 (M = 2) or kr + lo * R_right (M >= 3)
  int M, RR, R1;
  __device__ __forceinline__ double at(const int32_t* jr, int t, int rr) const {
    if (M == 1) return 1.0;
    if (M == 2) return __ldg(base + (int64_t)jr[t] * R1 + rr);
    return base[(int64_t)t * RR + rr];
  }
};

__device__ __forceinline__ RightRows right_rows(const RowArgs& a, int64_t lo) {
  const Others& o = a.o;
  RightRows r;
  r.M = o.M;
  r.RR = o.Rright;
  r.R1 = o.M >= 2 ? o.R[1] : 1;
  r.base = o.M == 2 ? o.A[1] : (o.M >= 3 ? a.kr + lo * o.Rright : nullptr);
  return r;
}

// c -> dst = K_S^T c (grouped); Z: u x R_right scratch, part: partial sums.
__device__ void sk_transpose(const RowArgs& a, const RightRows& rw, int u, const int32_t* jr,
                             const int32_t* gstart, const int32_t* gj, const double* c, double* Z, double* part,
                             double* dst) {
  const int RR = a.o.Rright, R0 = a.o.R[0], n = a.o.Rrest;
  const double* A0 = a.o.A[0];
  for (int task = threadIdx.x; task < u * RR; task += blockDim.x) {
    const int g = task / RR, rr = task - g * RR;
    const int t0 = gstart[g];
    Z[task] = sum8(gstart[g + 1] - t0, [&](int k, double acc) { return fma(c[t0 + k], rw.at(jr, t0 + k, rr), acc); });
  }
  __syncthreads();
  const int P = n >= (int)blockDim.x ? 1 : (int)blockDim.x / n;
  for (int task = threadIdx.x; task < n * P; task += blockDim.x) {
    const int pp = task / n, oo = task - pp * n;
    const int r0 = oo / RR, rr = oo - r0 * RR;
    const int cnt = u > pp ? (u - pp + P - 1) / P : 0;
    part[task] = sum8(cnt, [&](int k, double acc) {
      const int g = pp + k * P;
      return fma(__ldg(A0 + (int64_t)gj[g] * R0 + r0), Z[g * RR + rr], acc);
    });
  }
  __syncthreads();
  for (int oo = threadIdx.x; oo < n; oo += blockDim.x) {
    double sacc = part[oo];
    for (int pp = 1; pp < P; pp++) sacc += part[pp * n + oo];
    dst[oo] = sacc;
  }
  __syncthreads();
}

// c_t = v_t (v_t (K x)_t) for the row's samples (kron.py:258-300 then the scaling of :345).
__device__ void sk_forward(const RowArgs& a, const RightRows& rw, int nt, int u, const int32_t* jr,
                           const int32_t* gid, const int32_t* gj, const double* v, const double* xv, double* Y,
                           double* c) {
  const int RR = a.o.Rright, R0 = a.o.R[0];
  const double* A0 = a.o.A[0];
  for (int task = threadIdx.x; task < u * RR; task += blockDim.x) {
    const int g = task / RR, rr = task - g * RR;
    const double* arow = A0 + (int64_t)gj[g] * R0;
    Y[task] = sum8(R0, [&](int r0, double acc) { return fma(__ldg(arow + r0), xv[r0 * RR + rr], acc); });
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    const double* y = Y + (int64_t)gid[t] * RR;
    const double val = sum8(RR, [&](int rr, double acc) { return fma(y[rr], rw.at(jr, t, rr), acc); });
    c[t] = v[t] * (v[t] * val);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024) factor_rows_kernel(RowArgs a) {
  const int NT = blockDim.x;
  extern __shared__ double sm[];
  const Others& o = a.o;
  const int n = o.Rrest, Rn = a.ws.Rn, cap = a.cap, ucap = a.ucap;
  const int row = blockIdx.x;
  const int P = n >= NT ? 1 : NT / n;
  double* xv = sm;
  double* rhs = xv + n;
  double* tv = rhs + n;
  double* bv = tv + n;
  double* sv = bv + n;
  double* p0 = sv + n;
  double* p1 = p0 + n;
  double* tmp = p1 + n;
  double* part = tmp + n;                     // P * n
  double* s0 = part + (int64_t)P * n;         // R_n
  double* s1 = s0 + Rn;                       // R_n
  double* red = s1 + Rn;                      // 32
  double* hs = red + 32;                      // max_iters
  double* vv = hs + a.max_iters;              // cap
  double* vb = vv + cap;                      // cap
  double* cc = vb + cap;                      // cap
  double* YZ = cc + cap;                      // ucap * R_right
  int32_t* jr = (int32_t*)(YZ + (int64_t)ucap * o.Rright);  // cap
  int32_t* gid = jr + cap;                    // cap
  int32_t* gj = gid + cap;                    // ucap
  int32_t* gstart = gj + ucap;                // ucap + 1
  __shared__ int64_t s_lo, s_hi;
  __shared__ int s_stop, s_wtot[32];

  // ---- this row's segment of the (sorted) sparse diagonal
  if (threadIdx.x == 0) {
    int64_t lo = 0, hi = a.nnz;
    if (!a.shared) {
      const int64_t k0 = (int64_t)row * o.Irest, k1 = k0 + o.Irest;
      int64_t l = 0, h = a.nnz;
      while (l < h) { const int64_t m = (l + h) >> 1; if (a.sd_idx[m] < k0) l = m + 1; else h = m; }
      lo = l;
      h = a.nnz;
      while (l < h) { const int64_t m = (l + h) >> 1; if (a.sd_idx[m] < k1) l = m + 1; else h = m; }
      hi = l;
    }
    s_lo = lo;
    s_hi = hi;
  }
  __syncthreads();
  const int64_t lo = s_lo;
  const int nt = (int)(s_hi - s_lo);
  if (nt > cap) {
    if (threadIdx.x == 0) a.flags[row] = 2;
    return;
  }
  const int64_t kbase = a.shared ? 0 : (int64_t)row * o.Irest;
  // ---- samples: right-group flat index, value, v * b_at, first-factor groups
  int running = 0;
  for (int base = 0; base < nt; base += NT) {
    const int t = base + threadIdx.x;
    int head = 0;
    int64_t j0 = 0;
    if (t < nt) {
      const int64_t f = a.sd_idx[lo + t] - kbase;
      j0 = f / o.Iright;
      const int64_t jrt = f - j0 * o.Iright;
      jr[t] = (int32_t)jrt;
      const double val = a.sd_val[lo + t];
      vv[t] = val;
      // b[row, f] of the mode-n unfolding, read in place from the tensor
      int64_t off = (int64_t)row * a.xs_n + j0 * a.xs[0];
      int64_t rem = jrt, st = o.Iright;
      for (int m = 1; m < o.M; m++) {
        st /= o.I[m];
        const int64_t jm = rem / st;
        rem -= jm * st;
        off += jm * a.xs[m];
      }
      vb[t] = val * a.x[off];
      if (o.M >= 3) {  // Khatri-Rao row of the right group (kron.py:193-205 order)
        for (int rr = 0; rr < o.Rright; rr++) {
          int64_t rrem = rr, rst = o.Rright, jrem = jrt, jst = o.Iright;
          double prod = 1.0;
          for (int m = 1; m < o.M; m++) {
            rst /= o.R[m];
            jst /= o.I[m];
            const int64_t rm = rrem / rst, jm = jrem / jst;
            rrem -= rm * rst;
            jrem -= jm * jst;
            prod = prod * __ldg(o.A[m] + jm * o.R[m] + rm);
          }
          a.kr[(lo + t) * o.Rright + rr] = prod;
        }
      }
      head = (t == 0) || ((a.sd_idx[lo + t - 1] - kbase) / o.Iright != j0);
    }
    // block-wide exclusive scan of the head flags -> group ids
    const unsigned bal = __ballot_sync(0xffffffffu, head);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) s_wtot[wid] = __popc(bal);
    __syncthreads();
    int before = running;
    for (int w = 0; w < wid; w++) before += s_wtot[w];
    int tot = 0;
    for (int w = 0; w < NT / 32; w++) tot += s_wtot[w];
    const int incl = before + __popc(bal & ((2u << lane) - 1u));  // heads up to and including t
    if (t < nt) {
      const int g = incl - 1;
      gid[t] = g;
      if (head) {
        if (g < ucap) {
          gj[g] = (int32_t)j0;
          gstart[g] = t;
        }
      }
    }
    running += tot;
    __syncthreads();
  }
  const int u = running;
  if (u > ucap) {
    if (threadIdx.x == 0) a.flags[row] = 2;
    return;
  }
  if (threadIdx.x == 0) gstart[u] = nt;
  for (int t = threadIdx.x; t < nt; t += NT) cc[t] = vv[t] * vb[t];
  __syncthreads();
  const double w = a.ws.wdev[0];

  // ---- rhs = K_S^T (v * (v * b_at))
  const RightRows rw = right_rows(a, lo);
  sk_transpose(a, rw, u, jr, gstart, gj, cc, YZ, part, rhs);
  // ---- Richardson (solvers.py:201-248)
  for (int r = threadIdx.x; r < n; r += NT) xv[r] = 0.0;
  ws_apply(o, a.ws, rhs, bv, tmp, p0, p1, s0, s1, sv);
  const double scale = sqrt(block_sumsq(sv, n, red));
  const double tol = a.residual_tol * fmax(scale, 2.2250738585072014e-308);
  int done = 0, nh = 0, diverged = 0;
  for (int it = 0; it < a.max_iters; it++) {
    // tv = normal(x) - rhs
    sk_forward(a, rw, nt, u, jr, gid, gj, vv, xv, YZ, cc);
    sk_transpose(a, rw, u, jr, gstart, gj, cc, YZ, part, tv);
    penalty_terms(o, a.ws, w, xv, tv, s0, s1);
    for (int r = threadIdx.x; r < n; r += NT) tv[r] = tv[r] - rhs[r];
    __syncthreads();
    ws_apply(o, a.ws, tv, bv, tmp, p0, p1, s0, s1, sv);
    const double nrm = sqrt(block_sumsq(sv, n, red));
    if (threadIdx.x == 0) hs[nh] = nrm;
    nh++;
    if (nrm <= tol) break;
    if (nh > 5) {
      bool inc = true;
      for (int k = nh - 6; k < nh - 1; k++) inc = inc && (hs[k + 1] > hs[k]);
      if (threadIdx.x == 0) s_stop = inc && hs[nh - 1] > 10.0 * hs[nh - 6];
      __syncthreads();
      if (s_stop) {
        diverged = 1;
        break;
      }
    }
    for (int r = threadIdx.x; r < n; r += NT) xv[r] = xv[r] - a.damping * sv[r];
    __syncthreads();
    done++;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a.iters[row] = done;
    a.flags[row] = diverged;
  }
  if (a.hist)
    for (int k = threadIdx.x; k < a.max_iters; k += NT) a.hist[(int64_t)row * a.max_iters + k] = k < nh ? hs[k] : 0.0;
  // ---- z = G^T ((G^T)^+ x); new row = (G^T)^+ z  (tucker.py:377-378)
  warp_dots(Rn, n, a.ws.gnp, 1, Rn, xv, s0);
  __syncthreads();
  for (int r = threadIdx.x; r < n; r += NT) tv[r] = thread_dot(Rn, a.ws.gn + r, n, s0);
  __syncthreads();
  warp_dots(Rn, n, a.ws.gnp, 1, Rn, tv, s1);
  __syncthreads();
  if (threadIdx.x < Rn) a.out[(int64_t)row * Rn + threadIdx.x] = s1[threadIdx.x];
}

// ------------------------------------------------------------------ workspace apply (tests / API)

__global__ void __launch_bounds__(FT) ws_apply_kernel(Others o, Ws ws, const double* z, int32_t which, double* out) {
  extern __shared__ double sm[];
  const int n = o.Rrest, Rn = ws.Rn;
  double* src = sm;
  double* base = src + n;
  double* tmp = base + n;
  double* p0 = tmp + n;
  double* p1 = p0 + n;
  double* dst = p1 + n;
  double* s0 = dst + n;
  double* s1 = s0 + Rn;
  for (int r = threadIdx.x; r < n; r += FT) src[r] = z[r];
  __syncthreads();
  if (which == 0) {
    ws_apply(o, ws, src, base, tmp, p0, p1, s0, s1, dst);
  } else if (which == 1) {
    double* b = apply_base(o, ws, src, p0, p1);
    for (int r = threadIdx.x; r < n; r += FT) dst[r] = b[r];
  } else {
    // apply_penalized_normal: kron(Grams) z + w z + G^+ (right z)  (tucker.py:208-214)
    double* kz = kron_apply(o, o.G, false, src, p0, p1);
    warp_dots(Rn, n, ws.right, n, 1, src, s0);
    __syncthreads();
    const double w = ws.wdev[0];
    for (int r = threadIdx.x; r < n; r += FT)
      dst[r] = (kz[r] + w * src[r]) + thread_dot(Rn, ws.gnp + (int64_t)r * Rn, 1, s0);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < n; r += FT) out[r] = dst[r];
}

// ------------------------------------------------------------------ per-row draws

struct CdfPtrs {
  const double* cdf[MAXM];
  const double* prob[MAXM];
  int64_t n[MAXM];
};

// u: [m][row][t] uniforms; idx: (rows*s) x (M+1) with column 0 = row; w = 1/sqrt(prob * s).
__global__ void draws_rows_kernel(CdfPtrs c, int M, const double* __restrict__ u, int64_t rows, int64_t s,
                                  int64_t* __restrict__ idx, double* __restrict__ w) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = rows * s;
  if (q >= total) return;
  const int64_t row = q / s;
  idx[q * (M + 1)] = row;
  double prob = 1.0;
  for (int m = 0; m < M; m++) {
    const double x = u[(int64_t)m * total + q];
    const double* cdf = c.cdf[m];
    int64_t lo = 0, hi = c.n[m];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cdf[mid] <= x) lo = mid + 1; else hi = mid;
    }
    if (lo > c.n[m] - 1) lo = c.n[m] - 1;
    idx[q * (M + 1) + 1 + m] = lo;
    prob = __dmul_rn(prob, c.prob[m][lo]);
  }
  w[q] = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(prob, (double)s)));
}

// ------------------------------------------------------------------ explicit thin QR (LAPACK signs)

// Q (n x k) of A = QR by Householder reflections with dlarfg's convention
// (beta = -sign(alpha) |(alpha, x)|, tau = (beta - alpha) / beta, v = x / (alpha - beta)),
// then Q = H_0 ... H_{k-1} [I; 0] accumulated backwards as dorg2r does.  W: n x k scratch.
__global__ void __launch_bounds__(FT) qr_explicit_kernel(const double* __restrict__ A, int64_t n, int k,
                                                         double* __restrict__ W, double* __restrict__ Q) {
  __shared__ double red[32];
  __shared__ double tau[128];
  for (int64_t q = threadIdx.x; q < n * k; q += FT) W[q] = A[q];
  __syncthreads();
  for (int j = 0; j < k; j++) {
    double a2 = 0.0;
    for (int64_t r = j + 1 + threadIdx.x; r < n; r += FT) a2 = fma(W[r * k + j], W[r * k + j], a2);
    const double xnorm = sqrt(block_sum(a2, red));
    const double alpha = W[(int64_t)j * k + j];
    double tj = 0.0, beta = alpha;
    if (xnorm != 0.0) {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tj = (beta - alpha) / beta;
      const double sc = 1.0 / (alpha - beta);
      for (int64_t r = j + 1 + threadIdx.x; r < n; r += FT) W[r * k + j] *= sc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      tau[j] = tj;
      W[(int64_t)j * k + j] = beta;
    }
    __syncthreads();
    // apply H_j to the trailing columns
    for (int c = j + 1; c < k; c++) {
      double s = 0.0;
      for (int64_t r = j + 1 + threadIdx.x; r < n; r += FT) s = fma(W[r * k + j], W[r * k + c], s);
      s = block_sum(s, red) + W[(int64_t)j * k + c];
      __syncthreads();
      const double f = tj * s;
      if (threadIdx.x == 0) W[(int64_t)j * k + c] -= f;
      for (int64_t r = j + 1 + threadIdx.x; r < n; r += FT) W[r * k + c] -= f * W[r * k + j];
      __syncthreads();
    }
  }
  // Q = H_0 ... H_{k-1} [I; 0]
  for (int64_t q = threadIdx.x; q < n * k; q += FT) {
    const int64_t r = q / k, c = q % k;
    Q[q] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = k - 1; j >= 0; j--) {
    const double tj = tau[j];
    for (int c = j; c < k; c++) {
      double s = 0.0;
      for (int64_t r = j + 1 + threadIdx.x; r < n; r += FT) s = fma(W[r * k + j], Q[r * k + c], s);
      s = block_sum(s, red) + Q[(int64_t)j * k + c];
      const double f = tj * s;
      __syncthreads();
      if (threadIdx.x == 0) Q[(int64_t)j * k + c] -= f;
      for (int64_t r = j + 1 + threadIdx.x; r < n; r += FT) Q[r * k + c] -= f * W[r * k + j];
      __syncthreads();
    }
  }
}

// X (d x n) = sum_k (V[i][k] / sigma_k) U[j][k]  -- pseudo_inverse's (v / sigma) @ u.T (tensor.py:110-115)
__global__ void pinv_compose_kernel(const double* __restrict__ U, int64_t n, const double* __restrict__ sigma,
                                    const double* __restrict__ V, int64_t d, int k, double* __restrict__ X) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= d * n) return;
  const int64_t i = q / n, j = q % n;
  double acc = 0.0;
  for (int kk = 0; kk < k; kk++) acc = fma(V[i * k + kk] / sigma[kk], U[j * k + kk], acc);
  X[q] = acc;
}

int fill_others(Others& o, int32_t M, const double* const* A, const int64_t* I, const int32_t* R,
                const double* const* V, const double* const* G, const double* const* E) {
  KS_REQUIRE(M >= 1 && M <= MAXM, KS_EINVAL, "factor updates support 1..%d other factors (got %d)", MAXM, M);
  o = Others{};
  o.M = M;
  int64_t rr = 1, ii = 1, rright = 1, iright = 1;
  for (int m = 0; m < M; m++) {
    o.A[m] = A ? A[m] : nullptr;
    o.V[m] = V ? V[m] : nullptr;
    o.G[m] = G ? G[m] : nullptr;
    o.E[m] = E ? E[m] : nullptr;
    o.I[m] = I ? I[m] : 1;
    o.R[m] = R[m];
    KS_REQUIRE(R[m] >= 1 && R[m] <= 1024, KS_ESIZE, "rank %d out of range", R[m]);
    rr *= R[m];
    ii *= o.I[m];
    if (m >= 1) {
      rright *= R[m];
      iright *= o.I[m];
    }
  }
  KS_REQUIRE(rr <= 4096, KS_ESIZE, "leftover Kronecker rank %lld > 4096 unsupported", (long long)rr);
  KS_REQUIRE(iright < (1LL << 31), KS_ESIZE, "leftover row space too large");
  o.Rrest = (int32_t)rr;
  o.Rright = (int32_t)rright;
  o.Irest = ii;
  o.Iright = iright;
  return KS_OK;
}

}  // namespace

extern "C" int ks_factor_workspace(int32_t M, const int32_t* R, const double* const* V, const double* const* G,
                                   const double* const* E, int32_t Rn, const double* gn, const double* gnp,
                                   double lam, double eps, const double* v0, double* wout, double* bdiag,
                                   double* right, double* cm, int32_t* flags, void* stream) {
  Others o;
  int rc = fill_others(o, M, nullptr, nullptr, R, V, G, E);
  if (rc) return rc;
  KS_REQUIRE(Rn >= 1 && Rn <= 64, KS_ESIZE, "core rank %d out of range [1, 64]", Rn);
  WsArgs a{o, Rn, gn, gnp, lam, eps, v0, wout, bdiag, right, cm, flags};
  const size_t smem = sizeof(double) * ((size_t)5 * o.Rrest + 2 * Rn + 32);
  KS_TRY_CUDA(cudaFuncSetAttribute(factor_workspace_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  factor_workspace_kernel<<<1, FT, smem, (cudaStream_t)stream>>>(a);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_factor_ws_apply(int32_t M, const int32_t* R, const double* const* V, const double* const* G,
                                  int32_t Rn, const double* gn, const double* gnp, const double* mid,
                                  const double* right, const double* bdiag, const double* wdev, double lam,
                                  const double* z, int32_t which, double* out, void* stream) {
  Others o;
  int rc = fill_others(o, M, nullptr, nullptr, R, V, G, nullptr);
  if (rc) return rc;
  KS_REQUIRE(Rn >= 1 && Rn <= 64, KS_ESIZE, "core rank %d out of range [1, 64]", Rn);
  KS_REQUIRE(which >= 0 && which <= 2, KS_EINVAL, "which must be 0 (apply), 1 (apply_base) or 2 (penalised normal)");
  Ws ws{gn, gnp, mid, right, bdiag, wdev, lam, Rn};
  const size_t smem = sizeof(double) * ((size_t)6 * o.Rrest + 2 * Rn);
  KS_TRY_CUDA(cudaFuncSetAttribute(ws_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ws_apply_kernel<<<1, FT, smem, (cudaStream_t)stream>>>(o, ws, z, which, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_factor_draws_rows(int32_t M, const double* const* cdf, const double* const* prob,
                                    const int64_t* n, const double* u, int64_t rows, int64_t s, int64_t* idx,
                                    double* w, void* stream) {
  KS_REQUIRE(M >= 1 && M <= MAXM, KS_EINVAL, "1..%d factors supported", MAXM);
  if (rows <= 0 || s <= 0) return KS_OK;
  CdfPtrs c{};
  for (int m = 0; m < M; m++) {
    c.cdf[m] = cdf[m];
    c.prob[m] = prob[m];
    c.n[m] = n[m];
  }
  draws_rows_kernel<<<ceil_div_u(rows * s, 256), 256, 0, (cudaStream_t)stream>>>(c, M, u, rows, s, idx, w);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int64_t ks_factor_rows_smem(int32_t Rrest, int32_t Rright, int32_t Rn, int32_t max_iters, int32_t cap,
                                       int32_t ucap, int32_t threads) {
  const int P = Rrest >= threads ? 1 : threads / Rrest;
  return (int64_t)sizeof(double) * ((int64_t)8 * Rrest + (int64_t)P * Rrest + 2 * Rn + 32 + max_iters + 3LL * cap +
                                    (int64_t)ucap * Rright) +
         (int64_t)sizeof(int32_t) * (2LL * cap + 2LL * ucap + 1);
}

extern "C" int ks_factor_rows_richardson(int32_t M, const double* const* A, const int64_t* I, const int32_t* R,
                                         const double* const* V, int32_t Rn, const double* gn, const double* gnp,
                                         const double* mid, const double* right, const double* bdiag,
                                         const double* wdev, double lam, const int64_t* sd_idx, const double* sd_val,
                                         int64_t nnz, int32_t shared, int64_t rows, const double* x, int64_t xs_n,
                                         const int64_t* xs, double* kr, double damping, int32_t max_iters,
                                         double residual_tol, int32_t cap, double* out, int32_t* iters,
                                         int32_t* flags, double* hist, void* stream) {
  Others o;
  int rc = fill_others(o, M, A, I, R, V, nullptr, nullptr);
  if (rc) return rc;
  KS_REQUIRE(Rn >= 1 && Rn <= 64, KS_ESIZE, "core rank %d out of range [1, 64]", Rn);
  KS_REQUIRE(max_iters >= 0 && max_iters <= 4096, KS_EINVAL, "max_iters out of range");
  KS_REQUIRE(M < 3 || kr != nullptr, KS_EINVAL, "Khatri-Rao scratch required for >= 3 other factors");
  if (rows <= 0) return KS_OK;
  cap = (int32_t)ks_max64(1, cap);
  const int32_t ucap = (int32_t)ks_min64(cap, o.I[0]);
  // few heavy rows: 32 warps per row to hide the L2 latency of the factor-row gathers
  // (measured at c5: 1024 threads for the 64 mode-2 rows, 256 for the 512 rows of modes 0/1)
  const int threads = rows <= 2 * (int64_t)ks::num_sms() ? 1024 : 256;
  const int64_t smem = ks_factor_rows_smem(o.Rrest, o.Rright, Rn, max_iters, cap, ucap, threads);
  KS_REQUIRE(smem <= 227 * 1024, KS_ESIZE, "factor row solve needs %lld bytes of shared memory (> 227 KB)",
             (long long)smem);
  RowArgs a{};
  a.o = o;
  a.ws = Ws{gn, gnp, mid, right, bdiag, wdev, lam, Rn};
  a.sd_idx = sd_idx;
  a.sd_val = sd_val;
  a.nnz = nnz;
  a.shared = shared;
  a.x = x;
  a.xs_n = xs_n;
  for (int m = 0; m < M; m++) a.xs[m] = xs[m];
  a.kr = kr;
  a.damping = damping;
  a.max_iters = max_iters;
  a.residual_tol = residual_tol;
  a.cap = cap;
  a.ucap = ucap;
  a.out = out;
  a.iters = iters;
  a.flags = flags;
  a.hist = hist;
  KS_TRY_CUDA(cudaFuncSetAttribute(factor_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  factor_rows_kernel<<<(unsigned)rows, threads, (size_t)smem, (cudaStream_t)stream>>>(a);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_qr_explicit(const double* A, int64_t n, int32_t k, double* Q, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_REQUIRE(k >= 1 && k <= 128 && n >= k, KS_ESIZE, "qr_explicit needs 1 <= k <= min(n, 128)");
  ks::Scratch<double> W(n * k, st);
  KS_REQUIRE(W.p, KS_ECUDA, "scratch allocation failed");
  qr_explicit_kernel<<<1, FT, 0, st>>>(A, n, k, W.p, Q);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_pinv_compose(const double* U, int64_t n, const double* sigma, const double* V, int64_t d,
                               int32_t k, double* X, void* stream) {
  if (n <= 0 || d <= 0) return KS_OK;
  pinv_compose_kernel<<<ceil_div_u(n * d, 256), 256, 0, (cudaStream_t)stream>>>(U, n, sigma, V, d, k, X);
  KS_CHECK_LAUNCH();
  return KS_OK;
}
