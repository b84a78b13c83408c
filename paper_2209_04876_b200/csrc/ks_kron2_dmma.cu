// KronMatMul n^2 pass on the FP64 tensor pipe (sm_100a):  T (p x q) = L^T (m x p) . B (m x k) . R (k x q)
//
// This is kron_mat_mul([U1^T, U2^T], b) of the exact solver (reference solvers.py:314 via
// kron.py:66-77), the pass that dominates kronmatmul_svd_solve at n^2 = 2.7e8 (c3) ... 4.3e9 (c4).
//
// Design (persistent, stream-K, warp-specialised):
//   * B is streamed from HBM exactly once in 128-row x 16-column tiles by TMA
//     (cp.async.bulk.tensor, SWIZZLE_128B) into a 6-stage shared-memory ring guarded by
//     full/empty mbarriers; R^T tiles (q x 16, L2 resident) ride along in the same stage.
//   * One producer warp issues TMA; four consumer warps run DMMA m16n8k4 (FP64 tensor cores),
//     each owning a 32 x q block of P = B[I, :] R in registers.
//   * The (row-block, k-step) space is split evenly over one CTA per SM (stream-K); at every
//     row-block boundary the CTA folds its P into T_part = L[I]^T P (DMMA, P staged in padded
//     smem) and stores it to a private slot; a fixed-order reduction sums the slots
//     (deterministic, independent of timing).
#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace ks {
int gemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t a_rs, int64_t a_cs, int64_t a_bs, const double* B, int64_t b_rs, int64_t b_cs,
         int64_t b_bs, double beta, double* C, int64_t c_rs, int64_t c_cs, int64_t c_bs,
         int64_t batch);
}

namespace {

constexpr int KS_STAGES = 6;
// KronMatMul: 8 consumer warps (4 row groups x 2 column halves) = 2 per SM sub-partition
constexpr int K1_CW = 8;
constexpr int K1_THREADS = (K1_CW + 1) * 32;

template <int Q, int WM>
struct K1Cfg {
  static constexpr int BM = 4 * WM;
  static constexpr int B_TILE = BM * 16;                  // doubles
  static constexpr int R_TILE = Q * 16;                   // doubles
  static constexpr int STAGE = B_TILE + R_TILE;           // doubles (multiple of 128 -> 1 KB aligned)
  static constexpr int QP = Q + 4;                        // padded P row
  static constexpr int P_OFF = KS_STAGES * STAGE;         // doubles
  static constexpr int BAR_OFF = P_OFF + BM * QP;         // doubles
  static constexpr size_t BYTES = (size_t)BAR_OFF * 8 + 2 * KS_STAGES * 8 + 1024;
};

template <int Q, int WM, bool SQ>
__global__ void __launch_bounds__(K1_THREADS, 1)
    kron2_contract_kernel(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmR,
                          const double* __restrict__ L, int64_t m, int p, int q, int64_t nKS,
                          int64_t total_steps, int64_t per_cta, int max_seg, double* __restrict__ part,
                          double* __restrict__ sqpart) {
  using C = K1Cfg<Q, WM>;
  constexpr int BM = C::BM;
  constexpr int MT = WM / 16, NT = Q / 16;
  extern __shared__ unsigned char dyn_raw[];
  double* sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(dyn_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
  uint64_t* empty = full + KS_STAGES;
  double* Ps = sm + C::P_OFF;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t s0 = (int64_t)blockIdx.x * per_cta;
  const int64_t s1 = (s0 + per_cta < total_steps) ? s0 + per_cta : total_steps;
  if (s0 >= s1) return;
  if (tid == 0) {
    for (int s = 0; s < KS_STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], K1_CW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t rb_first = s0 / nKS;

  if (warp == K1_CW) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      tma_prefetch(&tmB);
      tma_prefetch(&tmR);
      // ring slot, phase and (row block, k-step) advanced incrementally (no 64-bit divisions)
      int st = 0;
      uint32_t ph = 1u;
      int64_t rb = s0 / nKS, kk = s0 - rb * nKS;
      for (int64_t s = s0; s < s1; s++) {
        mbar_wait(&empty[st], ph);
        double* stage = sm + st * C::STAGE;
        mbar_arrive_expect_tx(&full[st], (uint32_t)(C::STAGE * 8));
        tma_load_2d(stage, &tmB, (int)(kk * 16), (int)(rb * BM), &full[st]);
        tma_load_2d(stage + C::B_TILE, &tmR, (int)(kk * 16), 0, &full[st]);
        if (++kk == nKS) {
          kk = 0;
          rb++;
        }
        if (++st == KS_STAGES) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }

  // ------------------------------ consumers ------------------------------
  double acc[MT][NT][4];
#pragma unroll
  for (int a = 0; a < MT; a++)
#pragma unroll
    for (int b = 0; b < NT; b++)
#pragma unroll
      for (int c = 0; c < 4; c++) acc[a][b][c] = 0.0;

  const int row_w = (warp & 3) * WM, col_w = (warp >> 2) * (Q / 2);
  // ||B||^2 on the side (sqpart != null): the column-half-0 warps see every element of B exactly once
  // in their A fragments
  const bool sq_on = SQ && col_w == 0;
  double sq = 0.0;
  int st = 0;
  uint32_t ph = 0u;
  int64_t rb = s0 / nKS, kk = s0 - rb * nKS;  // advanced incrementally below
  for (int64_t s = s0; s < s1; s++) {
    mbar_wait(&full[st], ph);
    const double* Bs = sm + st * C::STAGE;
    const double* Rs = Bs + C::B_TILE;
#pragma unroll
    for (int k0 = 0; k0 < 16; k0 += 4) {
      double af[MT][2], bf[NT];
#pragma unroll
      for (int a = 0; a < MT; a++) {
        af[a][0] = Bs[swz128(row_w + a * 16 + g, k0 + t4)];
        af[a][1] = Bs[swz128(row_w + a * 16 + g + 8, k0 + t4)];
      }
      if constexpr (SQ) {
        if (sq_on) {
#pragma unroll
          for (int a = 0; a < MT; a++) sq = fma(af[a][1], af[a][1], fma(af[a][0], af[a][0], sq));
        }
      }
#pragma unroll
      for (int b = 0; b < NT; b++) bf[b] = Rs[swz128(col_w + b * 8 + g, k0 + t4)];
#pragma unroll
      for (int a = 0; a < MT; a++)
#pragma unroll
        for (int b = 0; b < NT; b++) dmma_16x8x4(acc[a][b], af[a][0], af[a][1], bf[b]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (++st == KS_STAGES) {
      st = 0;
      ph ^= 1u;
    }
    const bool row_end = ++kk == nKS;
    const bool seg_end = row_end || (s + 1 == s1);
    if (row_end) kk = 0;
    if (seg_end) {
      // ---- epilogue: T_part = L[I]^T P_I (row block rb) ----
#pragma unroll
      for (int a = 0; a < MT; a++)
#pragma unroll
        for (int b = 0; b < NT; b++) {
          const int r0 = row_w + a * 16 + g, c0 = col_w + b * 8 + 2 * t4;
          Ps[r0 * C::QP + c0] = acc[a][b][0];
          Ps[r0 * C::QP + c0 + 1] = acc[a][b][1];
          Ps[(r0 + 8) * C::QP + c0] = acc[a][b][2];
          Ps[(r0 + 8) * C::QP + c0 + 1] = acc[a][b][3];
          acc[a][b][0] = acc[a][b][1] = acc[a][b][2] = acc[a][b][3] = 0.0;
        }
      named_bar_sync(1, K1_CW * 32);
      const int64_t row0 = rb * BM;
      double* out = part + ((int64_t)blockIdx.x * max_seg + (rb - rb_first)) * p * q;
      for (int a0 = warp * 16; a0 < p; a0 += K1_CW * 16) {
        double t[Q / 8][4];
#pragma unroll
        for (int b = 0; b < Q / 8; b++) t[b][0] = t[b][1] = t[b][2] = t[b][3] = 0.0;
        for (int k0 = 0; k0 < BM; k0 += 4) {
          const int64_t gi = row0 + k0 + t4;
          const bool rok = gi < m;
          const double* Lr = L + gi * p;
          const double la0 = (rok && a0 + g < p) ? __ldg(Lr + a0 + g) : 0.0;
          const double la1 = (rok && a0 + g + 8 < p) ? __ldg(Lr + a0 + g + 8) : 0.0;
#pragma unroll
          for (int b = 0; b < Q / 8; b++) {
            const double pb = Ps[(k0 + t4) * C::QP + b * 8 + g];
            dmma_16x8x4(t[b], la0, la1, pb);
          }
        }
#pragma unroll
        for (int b = 0; b < Q / 8; b++) {
          const int c0 = b * 8 + 2 * t4;
          const int r0 = a0 + g;
          if (r0 < p) {
            if (c0 < q) out[r0 * q + c0] = t[b][0];
            if (c0 + 1 < q) out[r0 * q + c0 + 1] = t[b][1];
          }
          if (r0 + 8 < p) {
            if (c0 < q) out[(r0 + 8) * q + c0] = t[b][2];
            if (c0 + 1 < q) out[(r0 + 8) * q + c0 + 1] = t[b][3];
          }
        }
      }
      named_bar_sync(1, K1_CW * 32);
    }
    if (row_end) rb++;
  }
  if constexpr (SQ) {  // this CTA's share of ||B||^2: fixed-order warp and CTA sums
    __shared__ double sqs[K1_CW];
    sq = warp_sum(sq);
    if (lane == 0) sqs[warp] = sq;
    named_bar_sync(1, K1_CW * 32);
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < K1_CW; w++) t += sqs[w];
      sqpart[blockIdx.x] = t;
    }
  }
}

// T[e] = sum over slots (fixed order), warp per output element
__global__ void reduce_slots_kernel(const double* __restrict__ part, int64_t nslots, int64_t count,
                                    double* __restrict__ out) {
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= count) return;
  double s = 0.0;
  for (int64_t k = lane; k < nslots; k += 32) s += part[k * count + e];
  s = warp_sum(s);
  if (lane == 0) out[e] = s;
}

__global__ void transpose_kernel_rq(const double* __restrict__ a, int64_t rows, int cols, double* __restrict__ out) {
  // out (cols x rows) = a^T, a: rows x cols
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t j = e / rows, i = e - j * rows;
  out[e] = a[i * cols + j];
}

template <int Q, int WM>
int launch_k1(cudaStream_t st, const CUtensorMap& tmB, const CUtensorMap& tmR, const double* L, int64_t m,
              int p, int q, int64_t k, double* T, double* bsq) {
  using C = K1Cfg<Q, WM>;
  const int64_t nRB = (m + C::BM - 1) / C::BM;
  const int64_t nKS = (k + 15) / 16;
  const int64_t total = nRB * nKS;
  int grid = ks::num_sms();
  if (total < grid) grid = (int)total;
  const int64_t per = (total + grid - 1) / grid;
  grid = (int)((total + per - 1) / per);
  const int max_seg = (int)((per + nKS - 1) / nKS) + 1;
  const int64_t nslots = (int64_t)grid * max_seg;
  ks::Scratch<double> part(nslots * p * q, st);
  KS_REQUIRE(part.p, KS_ECUDA, "scratch allocation failed");
  KS_TRY_CUDA(cudaMemsetAsync(part.p, 0, sizeof(double) * nslots * p * q, st));
  ks::Scratch<double> sqp(bsq ? grid : 0, st);
  if (bsq) {
    KS_REQUIRE(sqp.p, KS_ECUDA, "scratch allocation failed");
    KS_TRY_CUDA(cudaMemsetAsync(sqp.p, 0, sizeof(double) * grid, st));
  }
  // the ||B||^2 side sum is its own instantiation: the plain contraction's kernel is untouched by it
  auto kern = bsq ? kron2_contract_kernel<Q, WM, true> : kron2_contract_kernel<Q, WM, false>;
  KS_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES));
  kern<<<grid, K1_THREADS, C::BYTES, st>>>(tmB, tmR, L, m, p, q, nKS, total, per, max_seg, part.p, sqp.p);
  KS_CHECK_LAUNCH();
  const int64_t count = (int64_t)p * q;
  reduce_slots_kernel<<<ceil_div_u(count * 32, 256), 256, 0, st>>>(part.p, nslots, count, T);
  KS_CHECK_LAUNCH();
  if (bsq) {
    reduce_slots_kernel<<<1, 32, 0, st>>>(sqp.p, grid, 1, bsq);
    KS_CHECK_LAUNCH();
  }
  return KS_OK;
}

}  // namespace

namespace ks {

// Returns KS_OK if the TMA/DMMA path ran, -1 if the shapes/layout need the generic path.
int kron2_contract_dmma(cudaStream_t st, const double* L, const double* B, int64_t ldb, const double* R,
                        int64_t m, int64_t k, int p, int q, double* T, double* bsq) {
  if (p < 1 || p > 128 || q < 1 || q > 128 || m < 1 || k < 16) return -1;
  if (((uintptr_t)B & 15) || (ldb & 1)) return -1;
  int Qp = q <= 16 ? 16 : q <= 32 ? 32 : q <= 64 ? 64 : 128;
  Scratch<double> Rt((int64_t)Qp * k, st);
  KS_REQUIRE(Rt.p, KS_ECUDA, "scratch allocation failed");
  transpose_kernel_rq<<<ceil_div_u(k * q, 256), 256, 0, st>>>(R, k, q, Rt.p);
  KS_CHECK_LAUNCH();
  CUtensorMap tmB, tmR;
  const int WM = (Qp == 128) ? 16 : 32;
  const uint32_t BM = 4 * WM;
  if (!make_tmap_f64(&tmB, B, (uint64_t)m, (uint64_t)k, (uint64_t)ldb, BM)) return -1;
  if (!make_tmap_f64(&tmR, Rt.p, (uint64_t)q, (uint64_t)k, (uint64_t)k, (uint32_t)Qp)) return -1;
  switch (Qp) {
    case 16: return launch_k1<16, 32>(st, tmB, tmR, L, m, p, q, k, T, bsq);
    case 32: return launch_k1<32, 32>(st, tmB, tmR, L, m, p, q, k, T, bsq);
    case 64: return launch_k1<64, 32>(st, tmB, tmR, L, m, p, q, k, T, bsq);
    default: return launch_k1<128, 16>(st, tmB, tmR, L, m, p, q, k, T, bsq);
  }
}

}  // namespace ks

// =============================================================================================
// Loss pass on the FP64 tensor pipe:  sum_{i,j} ((L Zt^T)[i,j] - B[i,j])^2,  Zt = R X^T (k x p)
// (ridge_loss's ||K x - b||^2 for two factor groups, reference solvers.py:251-262; never
//  materialises K x).  Persistent CTAs sweep (BM x BN) tiles of B in row-major order; TMA
//  streams B tiles and Zt tiles through a 3-stage ring; L[I] (BM x P) is reloaded once per row
//  block through its own full/empty barrier pair; DMMA forms the tile of K x, the epilogue
//  subtracts the B tile from shared memory and accumulates squares (Kahan) in registers.
// =============================================================================================
namespace {

constexpr int K2_BN = 32;

template <int P, int BM>
struct K2Cfg {
  // ring depth: the narrow widths are HBM-bound and need more of b in flight per SM
  static constexpr int STAGES = P == 16 ? 5 : P == 32 ? 4 : 3;
  static constexpr int CW = BM / 16;                      // consumer warps: one m16 row tile each
  static constexpr int THREADS = (CW + 1) * 32;           // + the producer warp
  static constexpr int WM = 16;                           // rows per consumer warp
  static constexpr int B_TILE = BM * K2_BN;               // doubles: BN/16 boxes of (16 x BM)
  static constexpr int Z_TILE = K2_BN * P;                // doubles: P/16 boxes of (16 x BN)
  static constexpr int STAGE = B_TILE + Z_TILE;
  static constexpr int L_OFF = STAGES * STAGE;         // BM x P: P/16 boxes of (16 x BM)
  static constexpr int BAR_OFF = L_OFF + BM * P;
  static constexpr size_t BYTES = (size_t)BAR_OFF * 8 + 2 * (STAGES + 1) * 8 + 1024 + 64;
  static_assert(BYTES <= 232448, "K2 ring fits shared memory");
};

template <int P, int BM>
__global__ void __launch_bounds__(K2Cfg<P, BM>::THREADS, 1)
    kron2_resid_kernel(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmZ,
                       const __grid_constant__ CUtensorMap tmL, int64_t nCB, int64_t total_tiles,
                       int64_t per_cta, double* __restrict__ part) {
  using C = K2Cfg<P, BM>;
  constexpr int WM = C::WM, MT = WM / 16, NT = K2_BN / 8;
  extern __shared__ unsigned char dyn_raw[];
  double* sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(dyn_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
  uint64_t* empty = full + C::STAGES;
  uint64_t* lfull = empty + C::STAGES;
  uint64_t* lempty = lfull + 1;
  __shared__ double red[8];
  double* Ls = sm + C::L_OFF;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t s0 = (int64_t)blockIdx.x * per_cta;
  const int64_t s1 = (s0 + per_cta < total_tiles) ? s0 + per_cta : total_tiles;
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::CW);
    }
    mbar_init(lfull, 1);
    mbar_init(lempty, C::CW);
    fence_barrier_init();
  }
  __syncthreads();
  double ssum = 0.0, scomp = 0.0;
  if (s0 < s1) {
    if (warp == C::CW) {
      if (lane == 0) {
        tma_prefetch(&tmB);
        tma_prefetch(&tmZ);
        tma_prefetch(&tmL);
        int64_t cur_rb = -1;
        uint32_t lphase = 0;
        int64_t rb = s0 / nCB, cb = s0 - rb * nCB;  // advanced incrementally (no 64-bit divisions)
        int st = 0;
        uint32_t sph = 1u;
        for (int64_t s = s0; s < s1; s++) {
          if (rb != cur_rb) {
            mbar_wait(lempty, lphase ^ 1u);
            lphase ^= 1u;
            mbar_arrive_expect_tx(lfull, (uint32_t)(BM * P * 8));
#pragma unroll
            for (int j = 0; j < P / 16; j++) tma_load_2d(Ls + j * BM * 16, &tmL, j * 16, (int)(rb * BM), lfull);
            cur_rb = rb;
          }
          mbar_wait(&empty[st], sph);
          double* stage = sm + st * C::STAGE;
          mbar_arrive_expect_tx(&full[st], (uint32_t)(C::STAGE * 8));
#pragma unroll
          for (int j = 0; j < K2_BN / 16; j++)
            tma_load_2d(stage + j * BM * 16, &tmB, (int)(cb * K2_BN + j * 16), (int)(rb * BM), &full[st]);
#pragma unroll
          for (int j = 0; j < P / 16; j++)
            tma_load_2d(stage + C::B_TILE + j * K2_BN * 16, &tmZ, j * 16, (int)(cb * K2_BN), &full[st]);
          if (++cb == nCB) {
            cb = 0;
            rb++;
          }
          if (++st == C::STAGES) {
            st = 0;
            sph ^= 1u;
          }
        }
      }
    } else {
      int64_t cur_rb = -1;
      uint32_t lphase = 0;
      const int row_w = warp * WM;
      int64_t rb = s0 / nCB, cb = s0 - rb * nCB;
      int st = 0;
      uint32_t sph = 0u;
      for (int64_t s = s0; s < s1; s++) {
        if (rb != cur_rb) {
          if (cur_rb >= 0) {
            __syncwarp();
            if (lane == 0) mbar_arrive(lempty);
          }
          mbar_wait(lfull, lphase);
          lphase ^= 1u;
          cur_rb = rb;
        }
        mbar_wait(&full[st], sph);
        const double* Bs = sm + st * C::STAGE;
        const double* Zs = Bs + C::B_TILE;
        double acc[MT][NT][4];
#pragma unroll
        for (int a = 0; a < MT; a++)
#pragma unroll
          for (int b = 0; b < NT; b++) acc[a][b][0] = acc[a][b][1] = acc[a][b][2] = acc[a][b][3] = 0.0;
#pragma unroll
        for (int k0 = 0; k0 < P; k0 += 4) {
          const int box = k0 >> 4, kc = (k0 & 15) + t4;
          double af[MT][2], bf[NT];
#pragma unroll
          for (int a = 0; a < MT; a++) {
            af[a][0] = Ls[box * BM * 16 + swz128(row_w + a * 16 + g, kc)];
            af[a][1] = Ls[box * BM * 16 + swz128(row_w + a * 16 + g + 8, kc)];
          }
#pragma unroll
          for (int b = 0; b < NT; b++) bf[b] = Zs[box * K2_BN * 16 + swz128(b * 8 + g, kc)];
#pragma unroll
          for (int a = 0; a < MT; a++)
#pragma unroll
            for (int b = 0; b < NT; b++) dmma_16x8x4(acc[a][b], af[a][0], af[a][1], bf[b]);
        }
        // epilogue: subtract the B tile, accumulate squares
#pragma unroll
        for (int a = 0; a < MT; a++)
#pragma unroll
          for (int b = 0; b < NT; b++) {
            const int r0 = row_w + a * 16 + g, c0 = b * 8 + 2 * t4;
            const int box = c0 >> 4, cc = c0 & 15;
            const double e0 = acc[a][b][0] - Bs[box * BM * 16 + swz128(r0, cc)];
            const double e1 = acc[a][b][1] - Bs[box * BM * 16 + swz128(r0, cc + 1)];
            const double e2 = acc[a][b][2] - Bs[box * BM * 16 + swz128(r0 + 8, cc)];
            const double e3 = acc[a][b][3] - Bs[box * BM * 16 + swz128(r0 + 8, cc + 1)];
            // squares only (no cancellation): plain fixed-order sums, two chains per lane
            if (b & 1) scomp = fma(e0, e0, fma(e1, e1, fma(e2, e2, fma(e3, e3, scomp))));
            else ssum = fma(e0, e0, fma(e1, e1, fma(e2, e2, fma(e3, e3, ssum))));
          }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == C::STAGES) {
          st = 0;
          sph ^= 1u;
        }
        if (++cb == nCB) {
          cb = 0;
          rb++;
        }
      }
    }
  }
  // CTA partial (consumers only contribute)
  ssum = warp_sum(ssum + scomp);
  if (lane == 0) red[warp] = ssum;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < C::CW; w++) s += red[w];
    part[blockIdx.x] = s;
  }
}

template <int P, int BM>
int launch_k2(cudaStream_t st, const CUtensorMap& tmB, const CUtensorMap& tmZ, const CUtensorMap& tmL, int64_t m,
              int64_t k, double* out) {
  using C = K2Cfg<P, BM>;
  const int64_t nRB = (m + BM - 1) / BM, nCB = (k + K2_BN - 1) / K2_BN;
  const int64_t total = nRB * nCB;
  int grid = ks::num_sms();
  if (total < grid) grid = (int)total;
  const int64_t per = (total + grid - 1) / grid;
  grid = (int)((total + per - 1) / per);
  ks::Scratch<double> part(grid, st);
  KS_REQUIRE(part.p, KS_ECUDA, "scratch allocation failed");
  auto kern = kron2_resid_kernel<P, BM>;
  KS_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES));
  kern<<<grid, C::THREADS, C::BYTES, st>>>(tmB, tmZ, tmL, nCB, total, per, part.p);
  KS_CHECK_LAUNCH();
  reduce_slots_kernel<<<1, 32, 0, st>>>(part.p, grid, 1, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

}  // namespace

namespace ks {

// sum((L X R^T - B)^2) on the TMA/DMMA path; -1 if the layout needs the generic path.
int kron2_residual_dmma(cudaStream_t st, const double* L, const double* X, const double* R, const double* B,
                        int64_t ldb, int64_t m, int64_t k, int p, int q, double* out) {
  if (!(p == 16 || p == 32 || p == 64 || p == 128) || q < 1 || m < 1 || k < 1) return -1;
  if (((uintptr_t)B & 15) || (ldb & 1) || ((uintptr_t)L & 15)) return -1;
  Scratch<double> Zt(k * p, st);
  KS_REQUIRE(Zt.p, KS_ECUDA, "scratch allocation failed");
  // Zt[j, a] = sum_c R[j, c] X[a, c]
  int rc = gemm(st, k, p, q, 1.0, R, q, 1, 0, X, 1, q, 0, 0.0, Zt.p, p, 1, 0, 1);
  if (rc) return rc;
  const uint32_t BM = (p == 128) ? 64 : 128;
  CUtensorMap tmB, tmZ, tmL;
  if (!make_tmap_f64(&tmB, B, (uint64_t)m, (uint64_t)k, (uint64_t)ldb, BM)) return -1;
  if (!make_tmap_f64(&tmZ, Zt.p, (uint64_t)k, (uint64_t)p, (uint64_t)p, K2_BN)) return -1;
  if (!make_tmap_f64(&tmL, L, (uint64_t)m, (uint64_t)p, (uint64_t)p, BM)) return -1;
  switch (p) {
    case 16: return launch_k2<16, 128>(st, tmB, tmZ, tmL, m, k, out);
    case 32: return launch_k2<32, 128>(st, tmB, tmZ, tmL, m, k, out);
    case 64: return launch_k2<64, 128>(st, tmB, tmZ, tmL, m, k, out);
    default: return launch_k2<128, 64>(st, tmB, tmZ, tmL, m, k, out);
  }
}

}  // namespace ks
