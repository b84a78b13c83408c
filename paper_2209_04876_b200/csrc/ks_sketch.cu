// Row-sketch plumbing and the sketched Kronecker operator.
//   sparse_diagonal_from_sketch (kron.py:173-190)
//   two-group view of the sketched rows (kron.py:117-144, :225-255, :303-309)
//   sketched_kron_apply / sketched_kron_transpose_apply (kron.py:258-354)
// The reference recomputes np.unique/argsort on every apply; here the grouping is built once
// per sketch and every apply is a gathered-row contraction over the distinct left-group rows.
#include <cstdlib>

#include "ks_common.cuh"
#include "ks_tma.cuh"
#include "ks_pairwise.cuh"

#include <vector>

namespace ks {
int radix_sort_pairs(cudaStream_t st, uint64_t* keys, int64_t* vals, int64_t n, int bits);
int scan_exclusive_i32(cudaStream_t st, const int32_t* in, int64_t n, int64_t* out);
}

namespace {

struct Shape8 {
  int64_t v[8];
};

__global__ void ravel_kernel(const int64_t* __restrict__ idx, int nf, Shape8 rs, int64_t s,
                             uint64_t* __restrict__ keys, int64_t* __restrict__ vals) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s) return;
  int64_t f = 0;
  for (int k = 0; k < nf; k++) f = f * rs.v[k] + idx[t * nf + k];
  keys[t] = (uint64_t)f;
  vals[t] = t;
}

__global__ void head_flags_kernel(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ head) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// One thread per segment start: value = sqrt(w2[first] + pairwise(w2[rest])) -- np.add.reduceat
// copies the first element and reduces the remainder with the pairwise inner loop.
__global__ void seg_sqrt_sum_kernel(const uint64_t* __restrict__ keys, const int64_t* __restrict__ perm,
                                    const int32_t* __restrict__ head, const int64_t* __restrict__ segid,
                                    int64_t n, const double* __restrict__ w,
                                    int64_t* __restrict__ sd_idx, double* __restrict__ sd_val) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !head[i]) return;
  int64_t e = i + 1;
  while (e < n && !head[e]) e++;
  const double w0 = w[perm[i]];
  double acc = __dmul_rn(w0, w0);
  if (e - i > 1) {
    auto get = [&](int64_t j) {
      const double x = w[perm[j]];
      return __dmul_rn(x, x);
    };
    acc = acc + pw_sum_seq(get, i + 1, e - i - 1);
  }
  const int64_t g = segid[i];
  sd_idx[g] = (int64_t)keys[i];
  sd_val[g] = __dsqrt_rn(acc);
}

__global__ void nnz_kernel(const int32_t* __restrict__ head, const int64_t* __restrict__ segid, int64_t n,
                           int64_t* __restrict__ out) {
  out[0] = segid[n - 1] + head[n - 1];
}

// Two-factor fused path: unique-key heads and left-row heads of the sorted keys in one pass
// (a unique key starts a new left row when its first factor's index differs from the
// previous element's).
__global__ void heads2_kernel(const uint64_t* __restrict__ keys, int64_t n, uint64_t n1,
                              int32_t* __restrict__ head, int32_t* __restrict__ lhead) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool h = i == 0 || keys[i] != keys[i - 1];
  head[i] = h ? 1 : 0;
  lhead[i] = (h && (i == 0 || keys[i] / n1 != keys[i - 1] / n1)) ? 1 : 0;
}

// Segment values (as seg_sqrt_sum_kernel) plus the two-group view of the sparse diagonal:
// right row = i1, left rows / segment starts at the left heads.
__global__ void seg_sqrt_group2_kernel(const uint64_t* __restrict__ keys, const int64_t* __restrict__ perm,
                                       const int32_t* __restrict__ head, const int64_t* __restrict__ segid,
                                       const int32_t* __restrict__ lhead, const int64_t* __restrict__ lsegid,
                                       int64_t n, uint64_t n1, const double* __restrict__ w,
                                       int64_t* __restrict__ sd_idx, double* __restrict__ sd_val,
                                       int64_t* __restrict__ seg, int64_t* __restrict__ lrow,
                                       int64_t* __restrict__ rrow, int64_t* __restrict__ counts,
                                       int64_t* __restrict__ first_raw) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == n - 1) {
    const int64_t nnz = segid[i] + head[i], ul = lsegid[i] + lhead[i];
    counts[0] = nnz;
    counts[1] = ul;
    seg[ul] = nnz;
  }
  if (!head[i]) return;
  int64_t e = i + 1;
  while (e < n && !head[e]) e++;
  const double w0 = w[perm[i]];
  double acc = __dmul_rn(w0, w0);
  if (e - i > 1) {
    auto get = [&](int64_t j) {
      const double x = w[perm[j]];
      return __dmul_rn(x, x);
    };
    acc = acc + pw_sum_seq(get, i + 1, e - i - 1);
  }
  const int64_t g = segid[i];
  const uint64_t key = keys[i];
  sd_idx[g] = (int64_t)key;
  sd_val[g] = __dsqrt_rn(acc);
  rrow[g] = (int64_t)(key % n1);
  if (first_raw) first_raw[g] = perm[i];  // the first draw (in draw order) of this entry
  if (lhead[i]) {
    const int64_t u = lsegid[i];
    seg[u] = g;
    lrow[u] = (int64_t)(key / n1);
  }
}

// ---- grouping of the sketched rows into (left group, right group) --------------------------

struct GroupSpec {
  int nf;
  int64_t rows[8];
  int nl, nr;
  int lpos[8], rpos[8];
};

__device__ __forceinline__ void unravel(int64_t flat, const GroupSpec& g, int64_t* multi) {
  for (int k = g.nf - 1; k >= 0; k--) {
    multi[k] = flat % g.rows[k];
    flat /= g.rows[k];
  }
}

// key = left_key * right_rows + right_key, val = sample position in the sparse diagonal
__global__ void group_keys_kernel(const int64_t* __restrict__ sd_idx, int64_t nnz, GroupSpec g,
                                  int64_t right_rows, uint64_t* __restrict__ keys,
                                  int64_t* __restrict__ vals) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  int64_t m[8];
  unravel(sd_idx[t], g, m);
  int64_t lk = 0, rk = 0;
  for (int k = 0; k < g.nl; k++) lk = lk * g.rows[g.lpos[k]] + m[g.lpos[k]];
  for (int k = 0; k < g.nr; k++) rk = rk * g.rows[g.rpos[k]] + m[g.rpos[k]];
  keys[t] = (uint64_t)(lk * right_rows + rk);
  vals[t] = t;
}

__global__ void left_head_kernel(const uint64_t* __restrict__ keys, int64_t n, int64_t right_rows,
                                 int32_t* __restrict__ head) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  head[i] = (i == 0 || keys[i] / right_rows != keys[i - 1] / right_rows) ? 1 : 0;
}

struct FacPtrs {
  const double* f[8];
  int64_t cols[8];
};

// Column c of the Khatri-Rao row of a factor group (kron.py:193-205: first factor slowest,
// product accumulated left to right starting from 1.0).
__device__ double kr_entry(const FacPtrs& F, const int64_t* m, const int* pos, int np, int c) {
  int64_t digit[8];
  int64_t rem = c;
  for (int k = np - 1; k >= 0; k--) {
    const int64_t cols = F.cols[pos[k]];
    digit[k] = rem % cols;
    rem /= cols;
  }
  double prod = 1.0;
  for (int k = 0; k < np; k++) {
    const int f = pos[k];
    prod = __dmul_rn(prod, F.f[f][m[f] * F.cols[f] + digit[k]]);
  }
  return prod;
}

// Per grouped sample t: v[t], perm[t], rrow[t] (row in Rmat), and for each left segment start
// the segment offset and left row; materialises Khatri-Rao rows of multi-factor groups.
__global__ void group_fill_kernel(const uint64_t* __restrict__ keys, const int64_t* __restrict__ pos,
                                  const int32_t* __restrict__ head, const int64_t* __restrict__ segid,
                                  int64_t nnz, int64_t right_rows, GroupSpec g, FacPtrs F,
                                  const int64_t* __restrict__ sd_idx, const double* __restrict__ sd_val,
                                  int64_t* __restrict__ seg, int64_t* __restrict__ lrow,
                                  int64_t* __restrict__ rrow, double* __restrict__ v,
                                  int64_t* __restrict__ perm, double* __restrict__ Lbuf, int dL,
                                  double* __restrict__ Rbuf, int dR) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  const int64_t p = pos[t];
  perm[t] = p;
  v[t] = sd_val[p];
  int64_t m[8];
  unravel(sd_idx[p], g, m);
  const uint64_t key = keys[t];
  const int64_t rk = (int64_t)(key % (uint64_t)right_rows);
  if (Rbuf) {
    // Khatri-Rao row of the right group, natural (row-major) column order of the group
    rrow[t] = t;
    for (int c = 0; c < dR; c++) Rbuf[t * dR + c] = kr_entry(F, m, g.rpos, g.nr, c);
  } else {
    rrow[t] = (g.nr == 1) ? m[g.rpos[0]] : rk;
  }
  if (head[t]) {
    const int64_t u = segid[t];
    seg[u] = t;
    if (Lbuf) {
      lrow[u] = u;
      for (int c = 0; c < dL; c++) Lbuf[u * dL + c] = kr_entry(F, m, g.lpos, g.nl, c);
    } else {
      lrow[u] = m[g.lpos[0]];
    }
  }
  if (t == nnz - 1) seg[segid[t] + head[t]] = nnz;
}

// ---- applies --------------------------------------------------------------------------------
// One warp per distinct left row u: y = X^T L_u (dR), then over the segment's samples.
constexpr int AP_WARPS = 8;
constexpr int MAXD = 128;

__global__ void __launch_bounds__(AP_WARPS * 32) forward_kernel(ks_sketch_view sk, const double* __restrict__ X,
                                                               const int64_t* __restrict__ perm,
                                                               double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * AP_WARPS + (threadIdx.x >> 5);
  if (u >= sk.u_left) return;
  const int dL = sk.dL, dR = sk.dR;
  const double* L = sk.Lmat + sk.lrow[u] * sk.ldl;
  double y[MAXD / 32];
#pragma unroll
  for (int j = 0; j < MAXD / 32; j++) y[j] = 0.0;
  for (int i = 0; i < dL; i++) {
    const double li = L[i];
#pragma unroll
    for (int j = 0; j < MAXD / 32; j++) {
      const int k = lane + 32 * j;
      if (k < dR) y[j] = fma(li, X[(int64_t)i * dR + k], y[j]);
    }
  }
  for (int64_t t = sk.seg[u]; t < sk.seg[u + 1]; t++) {
    const double* R = sk.Rmat + sk.rrow[t] * sk.ldr;
    double d = 0.0;
#pragma unroll
    for (int j = 0; j < MAXD / 32; j++) {
      const int k = lane + 32 * j;
      if (k < dR) d = fma(y[j], R[k], d);
    }
    d = warp_sum(d);
    if (lane == 0) out[perm ? perm[t] : t] = sk.v[t] * d;
  }
}

// MODE 0: s_t = v_t * bv[perm[t]]  (transpose apply)
// MODE 1: s_t = v_t * (v_t * L_u^T X R_t)  (fused normal operator)
// Each block handles AP_WARPS*CHW distinct left rows; block partial G_b = L_chunk^T Z_chunk.
constexpr int CHW = 4;  // left rows per warp per block
template <int MODE>
__global__ void __launch_bounds__(AP_WARPS * 32) gram_apply_kernel(ks_sketch_view sk, const double* __restrict__ X,
                                                                  const double* __restrict__ bv,
                                                                  const int64_t* __restrict__ perm,
                                                                  double* __restrict__ part) {
  extern __shared__ double sm[];
  const int dL = sk.dL, dR = sk.dR;
  const int CH = AP_WARPS * CHW;
  double* Ls = sm;                       // CH x dL
  double* Zs = sm + (size_t)CH * dL;     // CH x dR
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t u0 = (int64_t)blockIdx.x * CH;
  for (int e = tid; e < CH * dL; e += blockDim.x) {
    const int c = e / dL, i = e - c * dL;
    const int64_t u = u0 + c;
    Ls[e] = (u < sk.u_left) ? sk.Lmat[sk.lrow[u] * sk.ldl + i] : 0.0;
  }
  __syncthreads();
  for (int cc = 0; cc < CHW; cc++) {
    const int c = w * CHW + cc;
    const int64_t u = u0 + c;
    double z[MAXD / 32];
#pragma unroll
    for (int j = 0; j < MAXD / 32; j++) z[j] = 0.0;
    if (u < sk.u_left) {
      double y[MAXD / 32];
      if (MODE == 1) {
#pragma unroll
        for (int j = 0; j < MAXD / 32; j++) y[j] = 0.0;
        const double* L = Ls + (size_t)c * dL;
        for (int i = 0; i < dL; i++) {
          const double li = L[i];
#pragma unroll
          for (int j = 0; j < MAXD / 32; j++) {
            const int k = lane + 32 * j;
            if (k < dR) y[j] = fma(li, X[(int64_t)i * dR + k], y[j]);
          }
        }
      }
      for (int64_t t = sk.seg[u]; t < sk.seg[u + 1]; t++) {
        const double* R = sk.Rmat + sk.rrow[t] * sk.ldr;
        double r[MAXD / 32];
#pragma unroll
        for (int j = 0; j < MAXD / 32; j++) {
          const int k = lane + 32 * j;
          r[j] = (k < dR) ? R[k] : 0.0;
        }
        const double vt = sk.v[t];
        double s;
        if (MODE == 1) {
          double d = 0.0;
#pragma unroll
          for (int j = 0; j < MAXD / 32; j++) d = fma(y[j], r[j], d);
          d = warp_sum(d);
          s = vt * (vt * d);
        } else {
          s = vt * bv[perm ? perm[t] : t];
        }
#pragma unroll
        for (int j = 0; j < MAXD / 32; j++) z[j] = fma(s, r[j], z[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < MAXD / 32; j++) {
      const int k = lane + 32 * j;
      if (k < dR) Zs[(size_t)c * dR + k] = z[j];
    }
  }
  __syncthreads();
  // G_b[i][k] = sum_c Ls[c][i] Zs[c][k]
  double* G = part + (int64_t)blockIdx.x * dL * dR;
  for (int e = tid; e < dL * dR; e += blockDim.x) {
    const int i = e / dR, k = e - i * dR;
    double g = 0.0;
    for (int c = 0; c < CH; c++) g = fma(Ls[c * dL + i], Zs[c * dR + k], g);
    G[e] = g;
  }
}


// Fused normal-operator partials for d_L = d_R = 128 on the FP64 tensor cores (the generic path's
// widest case: the persistent loop kernel's X does not fit shared memory at 128 x 128).  Grid-stride
// over chunks of 32 left rows; per chunk Y = L_c X (DMMA, X resident in shared memory), the
// samples' values and Z_c = sum_t c_t R_t (one warp per left row), then G_b += L_c^T Z_c (DMMA) into
// register accumulators (warp w owns rows 16w..16w+15 of G_b).  One d^2 partial per block.
constexpr int G128_CH = 32, G128_LDX = 136, G128_LDL = 132, G128_LDZ = 136;
__global__ void __launch_bounds__(256) gram_apply_dmma128_kernel(ks_sketch_view sk, const double* __restrict__ X,
                                                                 double* __restrict__ part) {
  extern __shared__ double sm[];
  double* Xs = sm;                             // 128 x LDX
  double* Ls = Xs + 128 * G128_LDX;            // CH x LDL
  double* Ys = Ls + G128_CH * G128_LDL;        // CH x LDZ: Y, then Z
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  for (int e = tid; e < 128 * 128; e += 256) Xs[(e >> 7) * G128_LDX + (e & 127)] = X[e];
  double acc[16][4];
#pragma unroll
  for (int q = 0; q < 16; q++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[q][j] = 0.0;
  const int64_t nchunks = (sk.u_left + G128_CH - 1) / G128_CH;
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int64_t u0 = chunk * G128_CH;
    const int rows = (int)ks_min64(G128_CH, sk.u_left - u0);
    __syncthreads();  // the previous chunk's G phase is done with Ls / Ys
    for (int e = tid; e < G128_CH * 128; e += 256) {
      const int r = e >> 7, k = e & 127;
      Ls[r * G128_LDL + k] = (r < rows) ? sk.Lmat[sk.lrow[u0 + r] * sk.ldl + k] : 0.0;
    }
    __syncthreads();
    {  // Y = L_c X: 2 m-tiles x 16 n-tiles; warp w: m-tile w & 1, n-tiles 4 (w >> 1) .. + 3
      const int mt = w & 1, nt0 = (w >> 1) * 4;
      double c[4][4];
#pragma unroll
      for (int q = 0; q < 4; q++)
#pragma unroll
        for (int j = 0; j < 4; j++) c[q][j] = 0.0;
#pragma unroll 4
      for (int k0 = 0; k0 < 128; k0 += 4) {
        const double a0 = Ls[(mt * 16 + g) * G128_LDL + k0 + t];
        const double a1 = Ls[(mt * 16 + g + 8) * G128_LDL + k0 + t];
#pragma unroll
        for (int q = 0; q < 4; q++) dmma_16x8x4(c[q], a0, a1, Xs[(k0 + t) * G128_LDX + (nt0 + q) * 8 + g]);
      }
#pragma unroll
      for (int q = 0; q < 4; q++) {
        double* y0 = Ys + (mt * 16 + g) * G128_LDZ + (nt0 + q) * 8 + 2 * t;
        double* y1 = y0 + 8 * G128_LDZ;
        y0[0] = c[q][0];
        y0[1] = c[q][1];
        y1[0] = c[q][2];
        y1[1] = c[q][3];
      }
    }
    __syncthreads();
    // samples of each left row (warp per row): c_t = v_t (v_t Y_u . R_t), Z_u = sum c_t R_t
    for (int rr = w; rr < G128_CH; rr += 8) {
      double z[4] = {0.0, 0.0, 0.0, 0.0};
      if (rr < rows) {
        const int64_t u = u0 + rr;
        double y[4];
#pragma unroll
        for (int j = 0; j < 4; j++) y[j] = Ys[rr * G128_LDZ + lane + 32 * j];
        for (int64_t tt = sk.seg[u]; tt < sk.seg[u + 1]; tt++) {
          const double* R = sk.Rmat + sk.rrow[tt] * sk.ldr;
          double r[4];
#pragma unroll
          for (int j = 0; j < 4; j++) r[j] = R[lane + 32 * j];
          double d = 0.0;
#pragma unroll
          for (int j = 0; j < 4; j++) d = fma(y[j], r[j], d);
          d = warp_sum(d);
          const double vt = sk.v[tt];
          const double cf = vt * (vt * d);
#pragma unroll
          for (int j = 0; j < 4; j++) z[j] = fma(cf, r[j], z[j]);
        }
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 4; j++) Ys[rr * G128_LDZ + lane + 32 * j] = z[j];
    }
    __syncthreads();
    // G_b += L_c^T Z_c: warp w owns m-tile w (rows 16w..), all 16 n-tiles; k over the chunk rows
#pragma unroll 2
    for (int k0 = 0; k0 < G128_CH; k0 += 4) {
      const double a0 = Ls[(k0 + t) * G128_LDL + w * 16 + g];
      const double a1 = Ls[(k0 + t) * G128_LDL + w * 16 + g + 8];
#pragma unroll
      for (int q = 0; q < 16; q++) dmma_16x8x4(acc[q], a0, a1, Ys[(k0 + t) * G128_LDZ + q * 8 + g]);
    }
  }
  double* G = part + (int64_t)blockIdx.x * 128 * 128;
#pragma unroll
  for (int q = 0; q < 16; q++) {
    const int row = w * 16 + g, col = q * 8 + 2 * t;
    G[row * 128 + col] = acc[q][0];
    G[row * 128 + col + 1] = acc[q][1];
    G[(row + 8) * 128 + col] = acc[q][2];
    G[(row + 8) * 128 + col + 1] = acc[q][3];
  }
}

__global__ void reduce_cols_kernel(const double* __restrict__ part, int64_t nparts, int64_t count,
                                   double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  double s = 0.0, c = 0.0;
  for (int64_t p = 0; p < nparts; p++) {
    const double v = part[p * count + e];
    const double t = s + v;
    c += (fabs(s) >= fabs(v)) ? ((s - t) + v) : ((v - t) + s);
    s = t;
  }
  out[e] = s + c;
}


// ---- two-factor sketch by left-row buckets --------------------------------------------------
// The same outputs as the sort path (ravel, stable radix sort of the flat indices, run heads,
// scans, seg_sqrt_group2) from a counting sort on the left row: draws are counted and scattered
// into left-row buckets (atomics: arbitrary order inside a bucket), each bucket is sorted by
// (right row, draw index) -- i.e. into the stable order of the flat sort -- and reduced into its
// unique entries by one warp, and two block scans place the entries.  Six small launches instead
// of ~20 (c3: 86 -> 44 us in a graph, tools/bench_sketch.py).
constexpr int BK_T = 1024;  // threads of the single-block scans

__global__ void bk_count_kernel(const int64_t* __restrict__ idx, int64_t s, int32_t* __restrict__ cnt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < s) atomicAdd(&cnt[idx[2 * t]], 1);
}

// exclusive scans (one block) of NS int32 arrays of n counts: out_k[0..n]; cur (optional) gets a
// copy of out_0[0..n).  Tiles of BK_T x 8 counts: every thread loads 8 consecutive counts (two
// 16-byte loads, all in flight), a block scan of the thread totals, the tile total carried over.
// (Several CTAs: CTA c scans [c chunk, (c + 1) chunk) starting from the sum of the chunks before it,
// part[q nb + c'] from bk_partsum_kernel; chunk is a multiple of the tile.)
template <int NS>
__global__ void __launch_bounds__(BK_T) bk_scan_kernel(const int32_t* __restrict__ in0, const int32_t* __restrict__ in1,
                                                       int64_t n, int32_t* __restrict__ out0,
                                                       int32_t* __restrict__ out1, int32_t* __restrict__ cur,
                                                       const int32_t* __restrict__ part = nullptr, int64_t chunk = 0) {
  constexpr int PT = 8, TILE = BK_T * PT;
  __shared__ int32_t wsum[NS][BK_T / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int c = blockIdx.x, nb = gridDim.x;
  const int64_t lo = part ? (int64_t)c * chunk : 0, hi = part ? min(n, lo + chunk) : n;
  int32_t carry[NS];
#pragma unroll
  for (int q = 0; q < NS; q++) {
    carry[q] = 0;
    if (part)
      for (int i = 0; i < c; i++) carry[q] += part[q * nb + i];
  }
  for (int64_t t0 = lo; t0 < hi; t0 += TILE) {
    const int64_t b = t0 + (int64_t)tid * PT;
    int32_t v[NS][PT], inc[NS], loc[NS];
#pragma unroll
    for (int q = 0; q < NS; q++) {
      const int32_t* src = q ? in1 : in0;
      if (b + PT <= n && (((uintptr_t)(src + b)) & 15) == 0) {
        const int4 x0 = *reinterpret_cast<const int4*>(src + b), x1 = *reinterpret_cast<const int4*>(src + b + 4);
        v[q][0] = x0.x; v[q][1] = x0.y; v[q][2] = x0.z; v[q][3] = x0.w;
        v[q][4] = x1.x; v[q][5] = x1.y; v[q][6] = x1.z; v[q][7] = x1.w;
      } else {
#pragma unroll
        for (int k = 0; k < PT; k++) v[q][k] = b + k < n ? src[b + k] : 0;
      }
      loc[q] = 0;
#pragma unroll
      for (int k = 0; k < PT; k++) loc[q] += v[q][k];
      inc[q] = loc[q];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xffffffffu, inc[q], o);
        if (lane >= o) inc[q] += u;
      }
      if (lane == 31) wsum[q][wid] = inc[q];
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
      for (int q = 0; q < NS; q++) {
        int32_t x = wsum[q][lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t u = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += u;
        }
        wsum[q][lane] = x;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NS; q++) {
      int32_t* out = q ? out1 : out0;
      int32_t run = carry[q] + inc[q] - loc[q] + (wid ? wsum[q][wid - 1] : 0);
      int32_t o[PT];
#pragma unroll
      for (int k = 0; k < PT; k++) {
        o[k] = run;
        run += v[q][k];
      }
      // 16-byte stores (scalar 4-byte stores from one SM throttle on the L1 store queue)
      if (b + PT <= n && (((uintptr_t)(out + b)) & 15) == 0 && (q || !cur || (((uintptr_t)(cur + b)) & 15) == 0)) {
        *reinterpret_cast<int4*>(out + b) = make_int4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<int4*>(out + b + 4) = make_int4(o[4], o[5], o[6], o[7]);
        if (q == 0 && cur) {
          *reinterpret_cast<int4*>(cur + b) = make_int4(o[0], o[1], o[2], o[3]);
          *reinterpret_cast<int4*>(cur + b + 4) = make_int4(o[4], o[5], o[6], o[7]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < PT; k++)
          if (b + k < n) {
            out[b + k] = o[k];
            if (q == 0 && cur) cur[b + k] = o[k];
          }
      }
      carry[q] += wsum[q][BK_T / 32 - 1];
    }
    __syncthreads();
  }
  if (tid == 0 && hi == n) {
    out0[n] = carry[0];
    if (NS > 1) out1[n] = carry[NS - 1];
  }
}

// per-chunk sums for the multi-CTA form of bk_scan_kernel
template <int NS>
__global__ void __launch_bounds__(BK_T) bk_partsum_kernel(const int32_t* __restrict__ in0,
                                                          const int32_t* __restrict__ in1, int64_t n, int64_t chunk,
                                                          int32_t* __restrict__ part) {
  __shared__ int32_t ws[NS][BK_T / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, c = blockIdx.x;
  const int64_t lo = (int64_t)c * chunk, hi = min(n, lo + chunk);
#pragma unroll
  for (int q = 0; q < NS; q++) {
    const int32_t* src = q ? in1 : in0;
    int32_t v = 0;
    for (int64_t i = lo + tid; i < hi; i += BK_T) v += src[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) ws[q][wid] = v;
  }
  __syncthreads();
  if (tid < NS) {
    int32_t t = 0;
    for (int w = 0; w < BK_T / 32; w++) t += ws[tid][w];
    part[tid * gridDim.x + c] = t;
  }
}

// exclusive scan(s) of n counts, one block for small n, else one tile-multiple chunk per CTA
template <int NS>
static int bk_scan(cudaStream_t st, const int32_t* in0, const int32_t* in1, int64_t n, int32_t* out0, int32_t* out1,
                   int32_t* cur) {
  constexpr int64_t TILE = (int64_t)BK_T * 8;
  const int64_t nt = (n + TILE - 1) / TILE;
  if (nt <= 2) {
    bk_scan_kernel<NS><<<1, BK_T, 0, st>>>(in0, in1, n, out0, out1, cur);
    KS_CHECK_LAUNCH();
    return KS_OK;
  }
  const int nb = (int)std::min<int64_t>(nt, 64);
  const int64_t chunk = ((nt + nb - 1) / nb) * TILE;
  const int nbu = (int)((n + chunk - 1) / chunk);
  ks::Scratch<int32_t> part((size_t)NS * nbu, st);
  KS_REQUIRE(part.p, KS_ECUDA, "scratch allocation failed");
  bk_partsum_kernel<NS><<<nbu, BK_T, 0, st>>>(in0, in1, n, chunk, part.p);
  KS_CHECK_LAUNCH();
  bk_scan_kernel<NS><<<nbu, BK_T, 0, st>>>(in0, in1, n, out0, out1, cur, part.p, chunk);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

__global__ void bk_scatter_kernel(const int64_t* __restrict__ idx, int64_t s, int32_t* __restrict__ cur,
                                  int32_t* __restrict__ slot) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < s) slot[atomicAdd(&cur[idx[2 * t]], 1)] = (int32_t)t;
}

// One warp per left-row bucket: sort its draws by key (right row << 32 | draw index) -- a warp
// bitonic sort up to 32 draws, ranks by counting beyond -- then reduce the runs of equal right
// rows into entries (values as seg_sqrt_group2_kernel: w0^2 + pairwise sum of the others'
// squares, in draw order), staged at the bucket's draw offset; ucnt = entries of the bucket.
__global__ void bk_bucket_kernel(const int64_t* __restrict__ idx, const double* __restrict__ w,
                                 const int32_t* __restrict__ off, int64_t n0, int32_t* __restrict__ slot,
                                 int32_t* __restrict__ tmp, double* __restrict__ st_val,
                                 int32_t* __restrict__ st_r, int32_t* __restrict__ st_first,
                                 int32_t* __restrict__ ucnt, int32_t* __restrict__ nonempty) {
  const int64_t l = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (l >= n0) return;
  const int32_t b = off[l], m = off[l + 1] - b;
  if (lane == 0) nonempty[l] = m > 0 ? 1 : 0;
  if (m == 0) {
    if (lane == 0) ucnt[l] = 0;
    return;
  }
  auto key_of = [&](int32_t t) { return ((uint64_t)(uint32_t)idx[2 * (int64_t)t + 1] << 32) | (uint32_t)t; };
  if (m <= 32) {
    uint64_t k = lane < m ? key_of(slot[b + lane]) : ~0ull;
#pragma unroll
    for (int sz = 2; sz <= 32; sz <<= 1) {
#pragma unroll
      for (int j = sz >> 1; j > 0; j >>= 1) {
        const uint64_t o = __shfl_xor_sync(0xffffffffu, k, j);
        const bool up = (lane & sz) == 0, lower = (lane & j) == 0;
        k = (lower == up) ? (k < o ? k : o) : (k < o ? o : k);
      }
    }
    if (lane < m) slot[b + lane] = (int32_t)(uint32_t)k;
  } else {  // rank by counting (keys are unique): O(m^2 / 32) per warp, for rare large buckets
    for (int32_t i = lane; i < m; i += 32) {
      const uint64_t ki = key_of(slot[b + i]);
      int32_t r = 0;
      for (int32_t j = 0; j < m; j++) r += key_of(slot[b + j]) < ki;
      tmp[b + r] = (int32_t)(uint32_t)ki;
    }
    __syncwarp();
    for (int32_t i = lane; i < m; i += 32) slot[b + i] = tmp[b + i];
  }
  __syncwarp();
  if (m <= 32) {  // runs of equal right rows, one lane per draw: heads, entry ranks by ballot
    const int32_t t = lane < m ? slot[b + lane] : 0;
    const int64_t r = lane < m ? idx[2 * (int64_t)t + 1] : -1;
    const int64_t rp = __shfl_up_sync(0xffffffffu, r, 1);
    const bool head = lane < m && (lane == 0 || rp != r);
    const unsigned hm = __ballot_sync(0xffffffffu, head);
    if (head) {
      const int32_t u = __popc(hm & ((1u << lane) - 1));
      const unsigned later = hm & ~((2u << lane) - 1);  // heads after this one
      const int32_t e = later ? __ffs(later) - 1 : m;
      const double w0 = w[t];
      double acc = __dmul_rn(w0, w0);
      if (e - lane > 1) {
        auto get = [&](int64_t j) {
          const double x = w[slot[b + j]];
          return __dmul_rn(x, x);
        };
        acc = acc + pw_sum_seq(get, lane + 1, e - lane - 1);
      }
      st_val[b + u] = __dsqrt_rn(acc);
      st_r[b + u] = (int32_t)r;
      st_first[b + u] = t;
    }
    if (lane == 0) ucnt[l] = __popc(hm);
    return;
  }
  if (lane != 0) return;
  int32_t u = 0;
  for (int32_t i = 0; i < m;) {
    const int32_t t0 = slot[b + i];
    const int64_t r = idx[2 * (int64_t)t0 + 1];
    int32_t e = i + 1;
    while (e < m && idx[2 * (int64_t)slot[b + e] + 1] == r) e++;
    const double w0 = w[t0];
    double acc = __dmul_rn(w0, w0);
    if (e - i > 1) {
      auto get = [&](int64_t j) {
        const double x = w[slot[b + j]];
        return __dmul_rn(x, x);
      };
      acc = acc + pw_sum_seq(get, i + 1, e - i - 1);
    }
    st_val[b + u] = __dsqrt_rn(acc);
    st_r[b + u] = (int32_t)r;
    st_first[b + u] = t0;
    u++;
    i = e;
  }
  ucnt[l] = u;
}

// Final placement: entry g = uoff[l] + k of bucket l; left group u = goff[l] (non-empty buckets)
__global__ void bk_place_kernel(const int32_t* __restrict__ off, const int32_t* __restrict__ ucnt,
                                const int32_t* __restrict__ uoff, const int32_t* __restrict__ goff, int64_t n0,
                                uint64_t n1, const double* __restrict__ st_val, const int32_t* __restrict__ st_r,
                                const int32_t* __restrict__ st_first, int64_t* __restrict__ sd_idx,
                                double* __restrict__ sd_val, int64_t* __restrict__ seg, int64_t* __restrict__ lrow,
                                int64_t* __restrict__ rrow, int64_t* __restrict__ counts,
                                int64_t* __restrict__ first_raw) {
  const int64_t l = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int sub = threadIdx.x & 7;
  if (l >= n0) return;
  const int32_t u = ucnt[l], b = off[l], g0 = uoff[l];
  if (l == n0 - 1 && sub == 0) {
    counts[0] = uoff[n0];
    counts[1] = goff[n0];
    seg[goff[n0]] = uoff[n0];
  }
  if (u == 0) return;
  if (sub == 0) {
    seg[goff[l]] = g0;
    lrow[goff[l]] = l;
  }
  for (int32_t k = sub; k < u; k += 8) {
    const int64_t g = g0 + k;
    const int64_t r = st_r[b + k];
    sd_idx[g] = (int64_t)((uint64_t)l * n1 + (uint64_t)r);
    sd_val[g] = st_val[b + k];
    rrow[g] = r;
    if (first_raw) first_raw[g] = st_first[b + k];
  }
}


}  // namespace

namespace ks {

int sketched_gram_partials(cudaStream_t st, const ks_sketch_view* sk, const double* X,
                           const double* bv, const int64_t* perm, int mode, double* part,
                           int64_t* nparts_out) {
  const int CH = AP_WARPS * CHW;
  const int64_t nb = (sk->u_left + CH - 1) / CH;
  *nparts_out = nb;
  if (nb == 0) return KS_OK;
  const size_t smem = sizeof(double) * (size_t)CH * (sk->dL + sk->dR);
  if (mode == 1 && sk->dL == 128 && sk->dR == 128 && !ks::env(ks::ENV_GRAM_SCALAR)) {
    const int64_t nchunks = (sk->u_left + G128_CH - 1) / G128_CH;
    const int64_t nb128 = ks_min64(nchunks, (int64_t)num_sms());
    *nparts_out = nb128;
    const size_t sm128 = sizeof(double) * (size_t)(128 * G128_LDX + G128_CH * G128_LDL + G128_CH * G128_LDZ);
    KS_TRY_CUDA(cudaFuncSetAttribute(gram_apply_dmma128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm128));
    gram_apply_dmma128_kernel<<<(unsigned)nb128, 256, sm128, st>>>(*sk, X, part);
    KS_CHECK_LAUNCH();
    return KS_OK;
  }
  if (mode == 1) {
    KS_TRY_CUDA(cudaFuncSetAttribute(gram_apply_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    gram_apply_kernel<1><<<(unsigned)nb, AP_WARPS * 32, smem, st>>>(*sk, X, bv, perm, part);
  } else {
    KS_TRY_CUDA(cudaFuncSetAttribute(gram_apply_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    gram_apply_kernel<0><<<(unsigned)nb, AP_WARPS * 32, smem, st>>>(*sk, X, bv, perm, part);
  }
  KS_CHECK_LAUNCH();
  return KS_OK;
}

int64_t sketched_partials_count(const ks_sketch_view* sk) {
  const int CH = AP_WARPS * CHW;
  return (sk->u_left + CH - 1) / CH;
}

int reduce_partials(cudaStream_t st, const double* part, int64_t nparts, int64_t count, double* out) {
  if (nparts == 0) {
    KS_TRY_CUDA(cudaMemsetAsync(out, 0, count * sizeof(double), st));
    return KS_OK;
  }
  reduce_cols_kernel<<<ceil_div_u(count, 256), 256, 0, st>>>(part, nparts, count, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

}  // namespace ks

// ------------------------------------------------------------------------------------ C-ABI

extern "C" int ks_sketch_diag(int32_t nf, const int64_t* idx, const int64_t* row_shape,
                              const double* w, int64_t s, int64_t* sd_idx, double* sd_val,
                              int64_t* nnz, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_REQUIRE(nf >= 1 && nf <= 8, KS_EINVAL, "1..8 factors supported");
  if (s <= 0) { *nnz = 0; return KS_OK; }
  Shape8 rs{};
  uint64_t rows = 1;
  for (int k = 0; k < nf; k++) { rs.v[k] = row_shape[k]; rows *= (uint64_t)row_shape[k]; }
  int bits = 0;
  while (bits < 64 && ((rows - 1) >> bits) != 0) bits++;
  ks::Scratch<uint64_t> keys(s, st);
  ks::Scratch<int64_t> perm(s, st);
  ks::Scratch<int32_t> head(s, st);
  ks::Scratch<int64_t> segid(s + 1, st);
  KS_REQUIRE(keys.p && perm.p && head.p && segid.p, KS_ECUDA, "scratch allocation failed");
  ravel_kernel<<<ceil_div_u(s, 256), 256, 0, st>>>(idx, nf, rs, s, keys.p, perm.p);
  KS_CHECK_LAUNCH();
  int rc = ks::radix_sort_pairs(st, keys.p, perm.p, s, bits);
  if (rc) return rc;
  head_flags_kernel<<<ceil_div_u(s, 256), 256, 0, st>>>(keys.p, s, head.p);
  KS_CHECK_LAUNCH();
  rc = ks::scan_exclusive_i32(st, head.p, s, segid.p);
  if (rc) return rc;
  seg_sqrt_sum_kernel<<<ceil_div_u(s, 128), 128, 0, st>>>(keys.p, perm.p, head.p, segid.p, s, w,
                                                          sd_idx, sd_val);
  KS_CHECK_LAUNCH();
  nnz_kernel<<<1, 1, 0, st>>>(head.p, segid.p, s, segid.p + s);
  KS_CHECK_LAUNCH();
  KS_TRY_CUDA(cudaMemcpyAsync(nnz, segid.p + s, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  KS_TRY_CUDA(cudaStreamSynchronize(st));
  return KS_OK;
}

extern "C" int ks_sketch_diag_grouped2_ex(const int64_t* idx, const int64_t* row_shape, const double* w, int64_t s,
                                          int64_t* sd_idx, double* sd_val, int64_t* seg, int64_t* lrow, int64_t* rrow,
                                          int64_t* counts, int64_t* counts_dev, int64_t* first_raw, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_REQUIRE(counts || counts_dev, KS_EINVAL, "need a host or a device counts buffer");
  if (s <= 0) {
    if (counts) counts[0] = counts[1] = 0;
    if (counts_dev) KS_TRY_CUDA(cudaMemsetAsync(counts_dev, 0, 2 * sizeof(int64_t), st));
    return KS_OK;
  }
  Shape8 rs{};
  rs.v[0] = row_shape[0];
  rs.v[1] = row_shape[1];
  const uint64_t n1 = (uint64_t)row_shape[1];
  const uint64_t rows = (uint64_t)row_shape[0] * n1;
  const int64_t n0 = row_shape[0];
  if (!ks::env(ks::ENV_SKETCH_SORT) && n0 >= 1 && n0 <= (1 << 24) && n1 <= (1ull << 31) && s < (1ll << 31) &&
      s <= 64 * n0) {
    // left-row buckets (at most 64 draws per left row on average: the warps' sorts stay short)
    int64_t* dcounts_b = counts_dev;
    ks::Scratch<int64_t> dcb(counts_dev ? 0 : 2, st);
    if (!dcounts_b) dcounts_b = dcb.p;
    ks::Scratch<int32_t> cnt(n0 + 1, st), off(n0 + 1, st), cur(n0 + 1, st), slot(s, st), tmp(s, st), sr(s, st),
        sf(s, st), ucnt(n0 + 1, st), uoff(n0 + 1, st), ne(n0 + 1, st), goff(n0 + 1, st);
    ks::Scratch<double> sv(s, st);
    KS_REQUIRE(dcounts_b && cnt.p && off.p && cur.p && slot.p && tmp.p && sr.p && sf.p && ucnt.p && uoff.p && ne.p &&
                   goff.p && sv.p,
               KS_ECUDA, "scratch allocation failed");
    KS_TRY_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (size_t)n0, st));
    bk_count_kernel<<<ceil_div_u(s, 256), 256, 0, st>>>(idx, s, cnt.p);
    if (int rc = bk_scan<1>(st, cnt.p, nullptr, n0, off.p, nullptr, cur.p)) return rc;
    bk_scatter_kernel<<<ceil_div_u(s, 256), 256, 0, st>>>(idx, s, cur.p, slot.p);
    bk_bucket_kernel<<<ceil_div_u(n0 * 32, 256), 256, 0, st>>>(idx, w, off.p, n0, slot.p, tmp.p, sv.p, sr.p, sf.p,
                                                               ucnt.p, ne.p);
    if (int rc = bk_scan<2>(st, ucnt.p, ne.p, n0, uoff.p, goff.p, nullptr)) return rc;
    bk_place_kernel<<<ceil_div_u(n0 * 8, 256), 256, 0, st>>>(off.p, ucnt.p, uoff.p, goff.p, n0, n1, sv.p, sr.p, sf.p,
                                                             sd_idx, sd_val, seg, lrow, rrow, dcounts_b, first_raw);
    KS_CHECK_LAUNCH();
    if (counts) {
      KS_TRY_CUDA(cudaMemcpyAsync(counts, dcounts_b, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      KS_TRY_CUDA(cudaStreamSynchronize(st));
    }
    return KS_OK;
  }
  int bits = 0;
  while (bits < 64 && ((rows - 1) >> bits) != 0) bits++;
  ks::Scratch<uint64_t> keys(s, st);
  ks::Scratch<int64_t> perm(s, st);
  ks::Scratch<int32_t> head(2 * s, st);
  ks::Scratch<int64_t> segid(2 * s, st);
  ks::Scratch<int64_t> dcounts_s(counts_dev ? 0 : 2, st);
  int64_t* dcounts = counts_dev ? counts_dev : dcounts_s.p;
  KS_REQUIRE(keys.p && perm.p && head.p && segid.p && dcounts, KS_ECUDA, "scratch allocation failed");
  int32_t* lhead = head.p + s;
  int64_t* lsegid = segid.p + s;
  ravel_kernel<<<ceil_div_u(s, 256), 256, 0, st>>>(idx, 2, rs, s, keys.p, perm.p);
  KS_CHECK_LAUNCH();
  int rc = ks::radix_sort_pairs(st, keys.p, perm.p, s, bits);
  if (rc) return rc;
  heads2_kernel<<<ceil_div_u(s, 256), 256, 0, st>>>(keys.p, s, n1, head.p, lhead);
  KS_CHECK_LAUNCH();
  rc = ks::scan_exclusive_i32(st, head.p, s, segid.p);
  if (rc) return rc;
  rc = ks::scan_exclusive_i32(st, lhead, s, lsegid);
  if (rc) return rc;
  seg_sqrt_group2_kernel<<<ceil_div_u(s, 128), 128, 0, st>>>(keys.p, perm.p, head.p, segid.p, lhead, lsegid, s, n1, w,
                                                             sd_idx, sd_val, seg, lrow, rrow, dcounts, first_raw);
  KS_CHECK_LAUNCH();
  if (counts) {
    KS_TRY_CUDA(cudaMemcpyAsync(counts, dcounts, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KS_TRY_CUDA(cudaStreamSynchronize(st));
  }
  return KS_OK;
}

extern "C" int ks_sketch_group(int32_t nf, const double* const* factors, const int64_t* rows,
                               const int64_t* cols, int32_t nleft, const int32_t* left_pos,
                               int32_t nright, const int32_t* right_pos, const int64_t* sd_idx,
                               const double* sd_val, int64_t nnz, int64_t* seg, int64_t* lrow,
                               int64_t* rrow, double* v, int64_t* perm, double* Lbuf,
                               double* Rbuf, int64_t* u_left, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_REQUIRE(nf >= 1 && nf <= 8 && nleft + nright == nf, KS_EINVAL, "bad group specification");
  if (nnz <= 0) { *u_left = 0; return KS_OK; }
  GroupSpec g{};
  g.nf = nf;
  g.nl = nleft;
  g.nr = nright;
  FacPtrs F{};
  for (int k = 0; k < nf; k++) { g.rows[k] = rows[k]; F.f[k] = factors[k]; F.cols[k] = cols[k]; }
  int64_t right_rows = 1, left_rows = 1, dL = 1, dR = 1;
  for (int k = 0; k < nleft; k++) { g.lpos[k] = left_pos[k]; left_rows *= rows[left_pos[k]]; dL *= cols[left_pos[k]]; }
  for (int k = 0; k < nright; k++) { g.rpos[k] = right_pos[k]; right_rows *= rows[right_pos[k]]; dR *= cols[right_pos[k]]; }
  KS_REQUIRE(dL <= MAXD && dR <= MAXD, KS_ESIZE, "group column products must be <= %d (got %lld, %lld)", MAXD,
             (long long)dL, (long long)dR);
  KS_REQUIRE((Lbuf != nullptr) == (nleft != 1), KS_EINVAL, "Lbuf required iff the left group is not a single factor");
  KS_REQUIRE((Rbuf != nullptr) == (nright != 1), KS_EINVAL, "Rbuf required iff the right group is not a single factor");
  ks::Scratch<uint64_t> keys(nnz, st);
  ks::Scratch<int64_t> pos(nnz, st);
  ks::Scratch<int32_t> head(nnz, st);
  ks::Scratch<int64_t> segid(nnz + 1, st);
  KS_REQUIRE(keys.p && pos.p && head.p && segid.p, KS_ECUDA, "scratch allocation failed");
  group_keys_kernel<<<ceil_div_u(nnz, 256), 256, 0, st>>>(sd_idx, nnz, g, right_rows, keys.p, pos.p);
  KS_CHECK_LAUNCH();
  // left group a prefix of the factor order => sorted flat order is already grouped
  bool prefix = true;
  for (int k = 0; k < nleft; k++) prefix &= (left_pos[k] == k);
  if (!prefix) {
    uint64_t total = (uint64_t)left_rows * (uint64_t)right_rows;
    int bits = 0;
    while (bits < 64 && ((total - 1) >> bits) != 0) bits++;
    int rc = ks::radix_sort_pairs(st, keys.p, pos.p, nnz, bits);
    if (rc) return rc;
  }
  left_head_kernel<<<ceil_div_u(nnz, 256), 256, 0, st>>>(keys.p, nnz, right_rows, head.p);
  KS_CHECK_LAUNCH();
  int rc = ks::scan_exclusive_i32(st, head.p, nnz, segid.p);
  if (rc) return rc;
  group_fill_kernel<<<ceil_div_u(nnz, 128), 128, 0, st>>>(keys.p, pos.p, head.p, segid.p, nnz, right_rows, g, F,
                                                          sd_idx, sd_val, seg, lrow, rrow, v, perm, Lbuf,
                                                          (int)dL, Rbuf, (int)dR);
  KS_CHECK_LAUNCH();
  nnz_kernel<<<1, 1, 0, st>>>(head.p, segid.p, nnz, segid.p + nnz);
  KS_CHECK_LAUNCH();
  KS_TRY_CUDA(cudaMemcpyAsync(u_left, segid.p + nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  KS_TRY_CUDA(cudaStreamSynchronize(st));
  return KS_OK;
}

extern "C" int ks_sketched_apply(const ks_sketch_view* sk, const double* X, const int64_t* perm,
                                 double* vals, void* stream) {
  KS_REQUIRE(sk->dR <= MAXD, KS_ESIZE, "right group width must be <= %d", MAXD);
  if (sk->u_left <= 0) return KS_OK;
  forward_kernel<<<ceil_div_u(sk->u_left, AP_WARPS), AP_WARPS * 32, 0, (cudaStream_t)stream>>>(*sk, X, perm, vals);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_sketched_transpose_apply(const ks_sketch_view* sk, const double* bv,
                                           const int64_t* perm, double* G, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  KS_REQUIRE(sk->dR <= MAXD && sk->dL <= MAXD, KS_ESIZE, "group widths must be <= %d", MAXD);
  const int64_t count = (int64_t)sk->dL * sk->dR;
  const int64_t np = ks::sketched_partials_count(sk);
  ks::Scratch<double> part(np * count + 1, st);
  KS_REQUIRE(part.p, KS_ECUDA, "scratch allocation failed");
  int64_t nb = 0;
  int rc = ks::sketched_gram_partials(st, sk, nullptr, bv, perm, 0, part.p, &nb);
  if (rc) return rc;
  return ks::reduce_partials(st, part.p, nb, count, G);
}

extern "C" int ks_sketch_diag_grouped2(const int64_t* idx, const int64_t* row_shape, const double* w, int64_t s,
                                       int64_t* sd_idx, double* sd_val, int64_t* seg, int64_t* lrow, int64_t* rrow,
                                       int64_t* counts, int64_t* counts_dev, void* stream) {
  return ks_sketch_diag_grouped2_ex(idx, row_shape, w, s, sd_idx, sd_val, seg, lrow, rrow, counts, counts_dev, nullptr,
                                    stream);
}

namespace {
// Gather of the sampled b entries.  Default launch: ceil(s / 256) blocks, one read per thread (the
// loop below runs once).  With page-locked host b every read is one PCIe request and the gather is
// request-rate bound (~3.8 ns per read on the B200 boxes, tools/hostgather_bench.cu).  The gather
// runs after the sketch in the solve graph (KS_GATHER_BESIDE_SKETCH=1, part of the graph key through
// solvers._switches, moves it beside the sketch: measured slower).  KS_GATHER_BLOCKS=<n> (A/B only)
// caps the grid, each thread then keeping GATHER_ILP independent reads in flight per pass.
constexpr int GATHER_ILP = 8;
__global__ void gather_draws2_kernel(const double* __restrict__ b, const int64_t* __restrict__ draws, int64_t n1,
                                     int64_t s, double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q0 < s; q0 += stride * GATHER_ILP) {
    double v[GATHER_ILP];
#pragma unroll
    for (int k = 0; k < GATHER_ILP; k++) {
      const int64_t q = q0 + k * stride;
      v[k] = q < s ? b[draws[2 * q] * n1 + draws[2 * q + 1]] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < GATHER_ILP; k++) {
      const int64_t q = q0 + k * stride;
      if (q < s) out[q] = v[k];
    }
  }
}
}  // namespace

extern "C" int ks_gather_draws2(const double* b, const int64_t* draws, int64_t n1, int64_t s, double* out,
                                void* stream) {
  if (s <= 0) return KS_OK;
  static const int max_blocks = [] {
    const char* e = ks::env(ks::ENV_GATHER_BLOCKS);  // diagnostic switch (A/B of the grid size)
    return e ? atoi(e) : 0;
  }();
  // default: one read per thread over the whole grid, all ~s reads in flight at once (measured
  // fastest for page-locked host b, where every read is one PCIe request; KS_GATHER_BLOCKS caps
  // the grid for A/B runs, each thread then reading GATHER_ILP entries per pass)
  int64_t nb = max_blocks > 0 ? ceil_div_u(s, 256 * GATHER_ILP) : ceil_div_u(s, 256);
  if (max_blocks > 0 && nb > max_blocks) nb = max_blocks;
  gather_draws2_kernel<<<(int)nb, 256, 0, (cudaStream_t)stream>>>(b, draws, n1, s, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}
