// K13: the three-factor n-pass of the Tucker exact core update (tucker.py:120 -> solvers.py:314 ->
// kron.py:66-77 at N = 3): T = (U0 kron U1 kron U2)^T b, b the n0 x n1 x n2 data tensor, as ONE
// streaming pass over b in the reference's own rightmost-first order.
//
// b is cut into units of up to 128 consecutive (i0, i1) rows of n2 doubles (a unit never crosses an
// i0 slab).  Every CTA streams a contiguous range of units through a ring of stages filled by TMA
// (stages of one 16-column box of a unit's rows, 128-byte swizzle, so the DMMA fragment reads are
// conflict free; the last warp to release a stage refills it); each of the 8 warps owns one m16
// row tile of every unit and, per unit,
//   step 1   M[i1, r2]  = sum_i2 b[i0, i1, i2] U2[i2, r2]          (rows x R2, the only n-sized work;
//                                                                   FP64 DMMA, U2 fragments in registers)
//   step 2   S[r1, r2]  = sum_i1 U1[i1, r1] M[i1, r2]              (R1 x R2, DMMA)
//   step 3   P[r0, r1, r2] += U0[i0, r0] S[r1, r2]                 (at the end of every i0 slab:
//                                                                   the warps' S tiles summed in order)
// M never leaves the warp: step 2 takes its B fragments from step 1's accumulators by shuffles, and
// S accumulates in registers across the units of a slab.
// Each CTA's P goes to its slot of a partial buffer; a second launch sums the slots in CTA order
// (deterministic).  b is read once from HBM and nothing of size n is written: the pass is bound by
// HBM bandwidth (8 n0 n1 n2 bytes) -- 2 n0 n1 n2 R2 flops.
#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace {

constexpr int K3_CW = 8;                 // compute warps (one m16 row tile each)
constexpr int K3_T = K3_CW * 32;         // lane 0 of warp 0 also issues the copies
constexpr int K3_SMEM = 227 * 1024;
constexpr int K3_ROWS = K3_CW * 16;      // (i0, i1) rows per unit at most: 128
constexpr int K3_PMAX = 8;               // core entries per compute thread: R0 R1 R2 <= 2048

struct K3Args {
  const double* U0;
  const double* U1;
  const double* U2;
  const double* B;
  double* part;  // grid x (R0 R1 R2)
  double* sqpart;  // register-streaming kernel, may be null: per-CTA ||b||^2
  int64_t n0, n1, n2;
  int R0, R1, R2;
  int rows;      // (i0, i1) rows per unit (the TMA box height, a multiple of 16)
  int nb1;       // units per i0 slab
  int stages;
  int stage_doubles;
  int stream_only;  // profiling aid: consume the boxes without computing
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void compute_bar() { __syncthreads(); }

// a warp's release of a ring stage (acq_rel: its reads of the stage are ordered before the refill
// that the last releaser issues); true for the last of the K3_CW warps
__device__ __forceinline__ bool release_last(unsigned* cnt) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(cnt)) : "memory");
  return old == K3_CW - 1;
}

template <int NBOX>
__global__ void __launch_bounds__(K3_T, 1)
    kron3_contract_kernel(const __grid_constant__ CUtensorMap tmB, K3Args a) {
  constexpr int KS = NBOX * 4;  // k-steps of step 1 (16 columns per box)
  extern __shared__ __align__(16) unsigned char k3_raw[];
  // 1 KB aligned base (SWIZZLE_128B destinations), kept in the shared window so loads stay LDS
  double* sm = reinterpret_cast<double*>(k3_raw + ((1024u - (smem_u32(k3_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int R0 = a.R0, R1 = a.R1, R2 = a.R2, R12 = R1 * R2, NP = R0 * R12;
  const int ROWS = a.rows, NS = a.stages, SD = a.stage_doubles, MT1 = (R1 + 15) / 16;
  // shared memory: NS stages of one box (ROWS x 16, SWIZZLE_128B), the per-warp S tiles
  // (K3_CW x MT1 x 16 x 8), S (MT1 x 16 x 8), then the stage mbarriers and release counters
  double* Sp = sm + (size_t)NS * SD;
  double* Ss = Sp + K3_CW * MT1 * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(Ss + MT1 * 128);
  unsigned* rel = reinterpret_cast<unsigned*>(full + NS);  // per stage: warps done with its box
  const int64_t units = a.n0 * a.nb1;
  const int64_t u_beg = units * blockIdx.x / gridDim.x, u_end = units * (blockIdx.x + 1) / gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < NS; s++) {
      mbar_init(&full[s], 1);
      rel[s] = 0u;
    }
    fence_barrier_init();
  }
  __syncthreads();

  // the ring: stage q % NS holds box q of the CTA's sequence (box q % NBOX of unit u_beg + q / NBOX).
  // Every warp counts itself out of a stage after its reads; the LAST warp to release a stage issues
  // the box NS later into it at once (no producer warp, no waiting on the slowest consumer's turn).
  const int64_t q_end = (u_end - u_beg) * NBOX;
  auto issue_box = [&](int64_t qq, int slot) {
    const int64_t u = u_beg + qq / NBOX, ui0 = u / a.nb1;
    const int k = (int)(qq % NBOX), row = (int)(ui0 * a.n1 + (u - ui0 * a.nb1) * ROWS);
    mbar_arrive_expect_tx(&full[slot], (uint32_t)(ROWS * 128));
    if (a.stream_only == 2)  // bandwidth probe: the same bytes as one contiguous 1-D bulk copy
      bulk_g2s(sm + (size_t)slot * SD, a.B + ((int64_t)row * a.n2 + k * ROWS * 16), (uint32_t)(ROWS * 128),
               &full[slot]);
    else
      tma_load_2d(sm + (size_t)slot * SD, &tmB, 16 * k, row, &full[slot]);
  };
  if (tid == 0) {
    tma_prefetch(&tmB);
    for (int64_t qq = 0; qq < min(q_end, (int64_t)NS); qq++) issue_box(qq, (int)qq);
  }

  // ------------------------------ every warp computes ------------------------------
  const int m0 = warp * 16;  // this warp's row tile of every unit
  const bool rows_on = m0 < ROWS;
  double u2f[KS];  // b0 = U2[k = 4 ks + t4][n = g] (zero past n2 / R2)
#pragma unroll
  for (int j = 0; j < KS; j++) {
    const int k = j * 4 + t4;
    u2f[j] = (k < a.n2 && g < R2) ? __ldg(&a.U2[(size_t)k * R2 + g]) : 0.0;
  }
  double P[K3_PMAX];  // P entries tid + 256 k
#pragma unroll
  for (int k = 0; k < K3_PMAX; k++) P[k] = 0.0;
  double sacc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};  // this warp's S tiles (r1 < 32)
  int64_t i0 = u_beg / a.nb1, ib = u_beg - i0 * a.nb1;
  int s = 0;
  uint32_t ph = 0;
  // swizzled A-fragment offsets of step 1 (rows m0 + g and m0 + g + 8 share the swizzle phase g)
  const double* Arow = sm + (m0 + g) * 16;
  int64_t q = 0;  // the CTA's box sequence
  for (int64_t u = u_beg; u < u_end; u++) {
    const int64_t i1b = ib * ROWS;
    const int nr = (int)min((int64_t)ROWS, a.n1 - i1b);
    // this unit's U1 fragments for step 2 (a0 = U1[row][r1], rows of this warp's tile), loaded
    // before the stage waits so their latency overlaps them
    double ua[4][2][2];
#pragma unroll
    for (int ks = 0; ks < 4; ks++) {
      const int row = m0 + 4 * ks + t4;
      const bool ok = rows_on && row < nr;
#pragma unroll
      for (int m1 = 0; m1 < 2; m1++) {
        const int r1 = 16 * m1 + g;
        ua[ks][m1][0] = ok && r1 < R1 ? __ldg(&a.U1[(i1b + row) * R1 + r1]) : 0.0;
        ua[ks][m1][1] = ok && r1 + 8 < R1 ? __ldg(&a.U1[(i1b + row) * R1 + r1 + 8]) : 0.0;
      }
    }
    // step 1: M tile (rows m0.., 8 columns r2) = B_unit U2 on DMMA, box by box; a0 = B[m0 + g][k],
    // a1 = B[m0 + g + 8][k] from the swizzled box (rows g and g + 8 share the swizzle phase g)
    double c[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < NBOX; k++, q++) {
      mbar_wait(&full[s], ph);
      if (rows_on && !a.stream_only) {
        const double* A = Arow + (size_t)s * SD;
#pragma unroll
        for (int kk = 0; kk < 4; kk++) {
          const int cb = kk * 4 + t4;  // column within the box
          const int off = ((((cb >> 1) ^ g)) << 1) + (cb & 1);
          dmma_16x8x4(c, A[off], A[off + 128], u2f[k * 4 + kk]);
        }
      }
      __syncwarp();
      if (lane == 0 && release_last(&rel[s])) {
        rel[s] = 0;
        if (q + NS < q_end) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue_box(q + NS, s);
        }
      }
      if (++s == NS) { s = 0; ph ^= 1; }
    }
    // step 2: S += U1_tile^T M_tile; b0 = M[4 ks + t4][g] fetched from the C fragments by shuffles
    // (row r of the tile sits in lane (r % 8) * 4 + col / 2, register 2 (r >= 8) + col % 2)
#pragma unroll
    for (int ks = 0; ks < 4; ks++) {
      const int src = ((4 * ks + t4) & 7) * 4 + (g >> 1);
      const double lo = __shfl_sync(0xffffffffu, c[ks >= 2 ? 2 : 0], src);
      const double hi = __shfl_sync(0xffffffffu, c[ks >= 2 ? 3 : 1], src);
      const double b0 = (g & 1) ? hi : lo;
      dmma_16x8x4(sacc[0], ua[ks][0][0], ua[ks][0][1], b0);
      if (MT1 > 1) dmma_16x8x4(sacc[1], ua[ks][1][0], ua[ks][1][1], b0);
    }
    // end of the i0 slab (or of this CTA's range): P += U0[i0, :] outer sum_w S_w
    const bool slab_end = (ib + 1 == a.nb1) || (u + 1 == u_end);
    if (slab_end) {
#pragma unroll
      for (int m1 = 0; m1 < 2; m1++)
        if (m1 < MT1) {
          double* so = Sp + ((warp * MT1 + m1) * 16 + g) * 8 + 2 * t4;
          *reinterpret_cast<double2*>(so) = make_double2(sacc[m1][0], sacc[m1][1]);
          *reinterpret_cast<double2*>(so + 64) = make_double2(sacc[m1][2], sacc[m1][3]);
          sacc[m1][0] = sacc[m1][1] = sacc[m1][2] = sacc[m1][3] = 0.0;
        }
      compute_bar();
      for (int e = tid; e < MT1 * 128; e += K3_CW * 32) {  // S = sum of the warps' tiles, in order
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < K3_CW; w++) v += Sp[w * MT1 * 128 + e];
        Ss[e] = v;
      }
      compute_bar();
      const double* u0 = a.U0 + i0 * R0;
#pragma unroll
      for (int k = 0; k < K3_PMAX; k++) {
        const int e = tid + k * K3_CW * 32;
        if (e < NP) {
          const int r0 = e / R12, cc = e - r0 * R12, r1 = cc / R2;
          P[k] = fma(__ldg(&u0[r0]), Ss[r1 * 8 + cc - r1 * R2], P[k]);
        }
      }
    }
    if (++ib == a.nb1) { ib = 0; i0++; }
  }
#pragma unroll
  for (int k = 0; k < K3_PMAX; k++) {
    const int e = tid + k * K3_CW * 32;
    if (e < NP) a.part[(size_t)blockIdx.x * NP + e] = P[k];
  }
}

// T[e] = sum over the CTA slots in order: one warp per output, lanes load 32 slots at a time
// (all in flight), then a fixed-order shuffle tree
__global__ void kron3_reduce_kernel(const double* __restrict__ part, int grid, int np, double* __restrict__ T) {
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (e >= np) return;
  double s = 0.0;
  for (int b = lane; b < grid; b += 32) s += part[(size_t)b * np + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) T[e] = s;
}

// ---- register-streaming variant (n2 <= 64): every warp streams its own 16-row tiles of b with 16-byte
// loads straight into DMMA A fragments (two tiles in flight per warp: the next tile's loads are issued
// before the current one is multiplied), no shared-memory ring and no CTA barrier until the end.
// Lane (g, t4) loads row g and g + 8 of the tile, 16-byte chunks t4, t4 + 4, ... (each load
// instruction covers 64 contiguous bytes of 8 rows); its k-step ks then multiplies column
// 8 (ks / 2) + 2 t4 + ks % 2 -- the same permutation of the k index for every row and for the U2
// fragments, so the DMMA contraction is unchanged.
template <int NCH, int MT1>
__global__ void __launch_bounds__(K3_T, 1) kron3_stream_kernel(K3Args a) {
  constexpr int KS = 2 * NCH;  // k-steps (n2 = 8 NCH columns)
  constexpr int CPL = 8;       // core columns (r1, r2) per lane: R1 R2 <= 256
  extern __shared__ __align__(16) double k3s[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int R0 = a.R0, R1 = a.R1, R2 = a.R2, R12 = R1 * R2, NP = R0 * R12;
  const int64_t n1 = a.n1, n2 = a.n2;
  const int nt1 = (int)((n1 + 15) / 16);  // tiles per i0 slab
  const int64_t tiles = a.n0 * nt1;
  const int64_t t_beg = tiles * blockIdx.x / gridDim.x, t_end = tiles * (blockIdx.x + 1) / gridDim.x;
  const int PWS = ((NP + 1) & ~1) + MT1 * 128;  // per warp: its core partial, then its S tile(s)
  double* Pw = k3s + (size_t)warp * PWS;
  double* Sw = Pw + ((NP + 1) & ~1);
  for (int e = lane; e < NP; e += 32) Pw[e] = 0.0;
  int sidx[CPL];  // core column c = lane + 32 j -> its S element (r1 = c / R2, r2 = c % R2)
#pragma unroll
  for (int j = 0; j < CPL; j++) {
    const int c = lane + 32 * j, r1 = c / R2;
    sidx[j] = c < R12 ? r1 * 8 + c - r1 * R2 : 0;
  }

  double u2f[KS];  // b0 = U2[column of (ks, t4)][g]
#pragma unroll
  for (int ks = 0; ks < KS; ks++) {
    const int col = 8 * (ks >> 1) + 2 * t4 + (ks & 1);
    u2f[ks] = (col < n2 && g < R2) ? __ldg(&a.U2[(size_t)col * R2 + g]) : 0.0;
  }
  double sacc[MT1][4];
#pragma unroll
  for (int m = 0; m < MT1; m++) sacc[m][0] = sacc[m][1] = sacc[m][2] = sacc[m][3] = 0.0;

  // this warp's tiles t_beg + warp + 8 k, tracked as (slab i0, tile of the slab) without divisions
  struct Pos {
    int64_t i0;
    int ts;  // tile within the slab
  };
  auto advance = [&](Pos p) {
    p.ts += K3_CW;
    while (p.ts >= nt1) {
      p.ts -= nt1;
      p.i0++;
    }
    return p;
  };
  auto load_tile = [&](Pos p, double2 (&v)[2][NCH]) {
    const int64_t i1b = (int64_t)p.ts * 16;
    const int nr = (int)min((int64_t)16, n1 - i1b);
    const double* base = a.B + (p.i0 * n1 + i1b) * n2;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int r = g + 8 * h;
#pragma unroll
      for (int j = 0; j < NCH; j++)
        v[h][j] = r < nr ? __ldg(reinterpret_cast<const double2*>(base + r * n2) + 4 * j + t4)
                         : make_double2(0.0, 0.0);
    }
  };
  double sqa = 0.0;  // this lane's share of ||b||^2 (a.sqpart)
  int64_t cur_i0 = -1;
  auto flush = [&]() {  // Pw += U0[cur_i0, :] outer S_w (this warp's S over the slab's tiles it ran)
#pragma unroll
    for (int m = 0; m < MT1; m++) {
      double* so = Sw + (m * 16 + g) * 8 + 2 * t4;
      *reinterpret_cast<double2*>(so) = make_double2(sacc[m][0], sacc[m][1]);
      *reinterpret_cast<double2*>(so + 64) = make_double2(sacc[m][2], sacc[m][3]);
      sacc[m][0] = sacc[m][1] = sacc[m][2] = sacc[m][3] = 0.0;
    }
    __syncwarp();
    double sv[CPL];
#pragma unroll
    for (int j = 0; j < CPL; j++) sv[j] = Sw[sidx[j]];
    const double* u0 = a.U0 + cur_i0 * R0;
    for (int r0 = 0; r0 < R0; r0++) {
      const double w = __ldg(&u0[r0]);
#pragma unroll
      for (int j = 0; j < CPL; j++)
        if (lane + 32 * j < R12) Pw[r0 * R12 + lane + 32 * j] = fma(w, sv[j], Pw[r0 * R12 + lane + 32 * j]);
    }
    __syncwarp();
  };
  // one tile: step 1 (M = B_tile U2, DMMA, two independent accumulator chains), step 2
  // (S_w += U1_tile^T M through shuffles)
  auto run_tile = [&](Pos p, const double2 (&v)[2][NCH]) {
    const int64_t i1b = (int64_t)p.ts * 16;
    const int nr = (int)min((int64_t)16, n1 - i1b);
    if (p.i0 != cur_i0) {
      if (cur_i0 >= 0) flush();
      cur_i0 = p.i0;
    }
    double ua[4][MT1][2];
#pragma unroll
    for (int ks = 0; ks < 4; ks++) {
      const int row = 4 * ks + t4;
      const bool ok = row < nr;
#pragma unroll
      for (int m = 0; m < MT1; m++) {
        const int r1 = 16 * m + g;
        ua[ks][m][0] = ok && r1 < R1 ? __ldg(&a.U1[(i1b + row) * R1 + r1]) : 0.0;
        ua[ks][m][1] = ok && r1 + 8 < R1 ? __ldg(&a.U1[(i1b + row) * R1 + r1 + 8]) : 0.0;
      }
    }
    if (a.sqpart) {  // ||b||^2 on the side: every element of b is in exactly one lane's tile loads
#pragma unroll
      for (int j = 0; j < NCH; j++)
        sqa = fma(v[1][j].y, v[1][j].y, fma(v[1][j].x, v[1][j].x, fma(v[0][j].y, v[0][j].y, fma(v[0][j].x, v[0][j].x, sqa))));
    }
    double c[4] = {0.0, 0.0, 0.0, 0.0}, d[4] = {0.0, 0.0, 0.0, 0.0};
    if (!a.stream_only) {
#pragma unroll
      for (int j = 0; j < NCH; j++) {
        dmma_16x8x4(c, v[0][j].x, v[1][j].x, u2f[2 * j]);
        dmma_16x8x4(d, v[0][j].y, v[1][j].y, u2f[2 * j + 1]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < NCH; j++) c[0] += v[0][j].x + v[1][j].y;  // consume the loads
    }
#pragma unroll
    for (int e = 0; e < 4; e++) c[e] += d[e];
#pragma unroll
    for (int ks = 0; ks < 4; ks++) {
      const int src = ((4 * ks + t4) & 7) * 4 + (g >> 1);
      const double lo = __shfl_sync(0xffffffffu, c[ks >= 2 ? 2 : 0], src);
      const double hi = __shfl_sync(0xffffffffu, c[ks >= 2 ? 3 : 1], src);
      const double b0 = (g & 1) ? hi : lo;
#pragma unroll
      for (int m = 0; m < MT1; m++) dmma_16x8x4(sacc[m], ua[ks][m][0], ua[ks][m][1], b0);
    }
  };
  double2 va[2][NCH], vb[2][NCH];
  int64_t t = t_beg + warp;
  Pos pa{t_beg / nt1, (int)(t_beg % nt1)};
  pa = advance(Pos{pa.i0, pa.ts + warp - K3_CW});
  if (t < t_end) load_tile(pa, va);
  for (; t < t_end; t += 2 * K3_CW) {
    const Pos pb = advance(pa);
    if (t + K3_CW < t_end) load_tile(pb, vb);
    run_tile(pa, va);
    if (t + K3_CW >= t_end) break;
    pa = advance(pb);
    if (t + 2 * K3_CW < t_end) load_tile(pa, va);
    run_tile(pb, vb);
  }
  if (cur_i0 >= 0) flush();
  __shared__ double sqw[K3_CW];
  if (a.sqpart) {
    sqa = warp_sum(sqa);
    if (lane == 0) sqw[warp] = sqa;
  }
  __syncthreads();
  for (int e = tid; e < NP; e += K3_T) {  // the warps' partials in order
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < K3_CW; w++) v += k3s[(size_t)w * PWS + e];
    a.part[(size_t)blockIdx.x * NP + e] = v;
  }
  if (a.sqpart && tid == 0) {
    double v = 0.0;
    for (int w = 0; w < K3_CW; w++) v += sqw[w];
    a.sqpart[blockIdx.x] = v;
  }
}

}  // namespace

static int g_k3_stream_only = 0;

// Profiling aid: later K13 launches only stream b through the ring (no arithmetic).
extern "C" int ks_debug_kron3_stream_only(int32_t on) {
  g_k3_stream_only = on;
  return KS_OK;
}

// Geometry the streaming kernel handles (else the caller contracts on the materialised right group)
extern "C" int ks_kron3_supported(int64_t n0, int64_t n1, int64_t n2, int32_t R0, int32_t R1, int32_t R2) {
  return n0 >= 1 && n1 >= 1 && n0 * n1 < (int64_t(1) << 31) && n2 >= 8 && n2 <= 128 && n2 % 8 == 0 && R0 >= 1 && R1 >= 1 && R2 >= 1 &&
         R1 <= 32 && R2 <= 8 && R1 * R2 <= 256 && R0 * R1 * R2 <= K3_PMAX * K3_CW * 32;
}

namespace ks {
int sumsq_diff(cudaStream_t st, const double* a, const double* b, int64_t n, double* out);
}

static int kron3_contract_impl(const double* U0, const double* U1, const double* U2, const double* B, int64_t n0,
                               int64_t n1, int64_t n2, int32_t R0, int32_t R1, int32_t R2, double* T, double* bsq,
                               cudaStream_t st);

// T (R0 x R1 R2, row-major) = (U0 kron U1 kron U2)^T b; U_k: n_k x R_k row-major, b: n0 n1 n2.
extern "C" int ks_kron3_contract(const double* U0, const double* U1, const double* U2, const double* B,
                                 int64_t n0, int64_t n1, int64_t n2, int32_t R0, int32_t R1, int32_t R2,
                                 double* T, void* stream) {
  return kron3_contract_impl(U0, U1, U2, B, n0, n1, n2, R0, R1, R2, T, nullptr, (cudaStream_t)stream);
}

// The same and bsq[0] = ||b||^2 (from the same pass when n2 <= 64)
extern "C" int ks_kron3_contract_sumsq(const double* U0, const double* U1, const double* U2, const double* B,
                                       int64_t n0, int64_t n1, int64_t n2, int32_t R0, int32_t R1, int32_t R2,
                                       double* T, double* bsq, void* stream) {
  KS_REQUIRE(bsq, KS_EINVAL, "kron3_contract_sumsq needs an output for ||b||^2");
  return kron3_contract_impl(U0, U1, U2, B, n0, n1, n2, R0, R1, R2, T, bsq, (cudaStream_t)stream);
}

static int kron3_contract_impl(const double* U0, const double* U1, const double* U2, const double* B, int64_t n0,
                               int64_t n1, int64_t n2, int32_t R0, int32_t R1, int32_t R2, double* T, double* bsq,
                               cudaStream_t st) {
  KS_REQUIRE(ks_kron3_supported(n0, n1, n2, R0, R1, R2), KS_ESIZE, "kron3 contraction: unsupported geometry");
  KS_REQUIRE(((uintptr_t)B & 15) == 0, KS_EINVAL, "kron3 contraction: 16-byte aligned b");
  K3Args a{};
  a.U0 = U0; a.U1 = U1; a.U2 = U2; a.B = B;
  a.stream_only = g_k3_stream_only;
  a.n0 = n0; a.n1 = n1; a.n2 = n2; a.R0 = R0; a.R1 = R1; a.R2 = R2;
  const int np = R0 * R1 * R2;
  const int mt1 = (R1 + 15) / 16;
  if (n2 <= 64 && (size_t)K3_CW * (((np + 1) & ~1) + mt1 * 128) * 8 <= (size_t)K3_SMEM) {
    // register-streaming kernel: 16-row tiles over every warp of the grid
    const int64_t tiles = n0 * ((n1 + 15) / 16);
    const int grid = (int)std::min<int64_t>(ks::num_sms(), (tiles + K3_CW - 1) / K3_CW);
    ks::Scratch<double> part((size_t)grid * np, st), sqp(bsq ? grid : 0, st);
    KS_REQUIRE(part.p && (!bsq || sqp.p), KS_ECUDA, "scratch allocation failed");
    a.part = part.p;
    a.sqpart = sqp.p;
    const size_t smem = (size_t)K3_CW * (((np + 1) & ~1) + mt1 * 128) * 8;
    int rc = KS_EINVAL;
#define KS_K3S(NCH, MT)                                                                                        if ((int)(n2 / 8) == NCH && mt1 == MT) {                                                                       KS_TRY_CUDA(cudaFuncSetAttribute(kron3_stream_kernel<NCH, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,                                      (int)smem));                                                                kron3_stream_kernel<NCH, MT><<<grid, K3_T, smem, st>>>(a);                                                   rc = KS_OK;                                                                                                }
    KS_K3S(1, 1) KS_K3S(2, 1) KS_K3S(3, 1) KS_K3S(4, 1) KS_K3S(5, 1) KS_K3S(6, 1) KS_K3S(7, 1) KS_K3S(8, 1)
    KS_K3S(1, 2) KS_K3S(2, 2) KS_K3S(3, 2) KS_K3S(4, 2) KS_K3S(5, 2) KS_K3S(6, 2) KS_K3S(7, 2) KS_K3S(8, 2)
#undef KS_K3S
    if (rc) return rc;
    KS_CHECK_LAUNCH();
    kron3_reduce_kernel<<<(np + 7) / 8, 256, 0, st>>>(part.p, grid, np, T);
    KS_CHECK_LAUNCH();
    if (bsq) {
      kron3_reduce_kernel<<<1, 256, 0, st>>>(sqp.p, grid, 1, bsq);
      KS_CHECK_LAUNCH();
    }
    return KS_OK;
  }
  if (bsq) {  // the TMA-ring kernel has no side sum: a separate pass
    const int rc0 = ks::sumsq_diff(st, B, nullptr, n0 * n1 * n2, bsq);
    if (rc0) return rc0;
  }
  // TMA-ring kernel (64 < n2 <= 128)
  a.rows = (int)std::min<int64_t>(K3_ROWS, (n1 + 15) / 16 * 16);  // m16 row tiles, one per compute warp
  a.nb1 = (int)((n1 + a.rows - 1) / a.rows);
  const int nbox = (int)((n2 + 15) / 16);
  a.stage_doubles = (a.rows * 16 + 127) & ~127;  // one 16-column box per stage, 1 KB aligned
  const int fixed = K3_CW * mt1 * 128 + mt1 * 128 + 64;  // doubles (+ mbarriers)
  a.stages = std::min(16, (K3_SMEM / 8 - 128 - fixed) / a.stage_doubles);
  KS_REQUIRE(a.stages >= 2, KS_ESIZE, "kron3 contraction: stages do not fit shared memory");
  const size_t smem = ((size_t)a.stages * a.stage_doubles + fixed) * 8 + 1024;
  CUtensorMap tmB;
  KS_REQUIRE(ks::make_tmap_f64(&tmB, B, (uint64_t)(n0 * n1), (uint64_t)n2, (uint64_t)n2, (uint32_t)a.rows),
             KS_EINVAL, "kron3 contraction: tensor map");
  const int64_t units = n0 * a.nb1;
  const int grid = (int)std::min<int64_t>(ks::num_sms(), units);
  ks::Scratch<double> part((size_t)grid * np, st);
  KS_REQUIRE(part.p, KS_ECUDA, "scratch allocation failed");
  a.part = part.p;
  int rc = KS_EINVAL;
  switch (nbox) {
#define KS_K3(NB)                                                                                          \
  case NB: {                                                                                               \
    KS_TRY_CUDA(cudaFuncSetAttribute(kron3_contract_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     (int)smem));                                                          \
    kron3_contract_kernel<NB><<<grid, K3_T, smem, st>>>(tmB, a);                                           \
    rc = KS_OK;                                                                                            \
    break;                                                                                                 \
  }
    KS_K3(1) KS_K3(2) KS_K3(3) KS_K3(4) KS_K3(5) KS_K3(6) KS_K3(7) KS_K3(8)
#undef KS_K3
  }
  if (rc) return rc;
  KS_CHECK_LAUNCH();
  kron3_reduce_kernel<<<(np + 7) / 8, 256, 0, st>>>(part.p, grid, np, T);
  KS_CHECK_LAUNCH();
  return KS_OK;
}
