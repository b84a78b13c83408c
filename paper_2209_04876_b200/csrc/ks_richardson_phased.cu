// Persistent Richardson loop in the preconditioner's eigenbasis (the default path of the fused
// two-factor solve, reference solvers.py:201-248 applied to the sketched normal operator of
// kron.py:258-354 with the preconditioner of solvers.py:166-198): one CTA per SM, all passes (the
// right-hand-side pass, then every iteration) in one cooperative launch.
//
// Each CTA owns a fixed, contiguous range of chunks of the sketch (device work plan), i.e. a
// contiguous range of packed left rows and of samples.  Per pass, in blocks of up to ROWCAP rows,
// in three phases separated by CTA barriers:
//
//   Y phase (DMMA warps)   Y = L X' over the block's rows: m16n8 tiles (row tile, n8 strip),
//                          several row tiles in flight per warp (independent m16n8k4 chains;
//                          X' fragments resident in registers)
//   sample phase (all 12 warps: 48 quarter-warps, each owning a contiguous group of rows with
//                          about 1/48 of the block's samples)
//                          z_u = sum_t v_t (v_t (y_u . r_t)) r_t, the packed right rows r_t read
//                          from L2 with 16-byte loads, each row's sample range from a shared
//                          table, z_u written over y_u
//   G phase (DMMA warps)   G += L^T Z over the block's rows (accumulators in registers)
//
// The packed left rows of the block (L) stay in shared memory: when a CTA's rows fit one block
// (BASELINE c3) they are loaded once per solve.  Separating the phases keeps the FP64 pipe busy
// with long independent DMMA streams instead of interleaving them with the latency-bound sample
// work (a phase-separated variant that ran the sample work beside the DMMA work was measured
// slower: both share the FP64 pipe).  After the apply, the CTA partials of G are reduced in a
// fixed order (reduce-scatter over CTAs, one bulk copy per reducer), the step' =
// dinv o (G' + lam x' - rhs') and its norm are formed, and every CTA updates its register copy
// of x'.  Two grid barriers per iteration (one release-add arrival counter), no host round trips.
#include "ks_persistent.cuh"

#include <cfloat>

using namespace ks_rich;

namespace {

constexpr int MW = 8;                 // DMMA warps
constexpr int NW = 12;                // all warps (the sample phase uses every one)
constexpr int NT = NW * 32;           // 384 threads: <= 168 registers each
constexpr int NQ = NW * 4;            // quarter-warps of the sample phase

constexpr int SMEM_MAX = 232448;

template <int DL, int DR>
struct PhSmem {
  static constexpr int DLP = DL + PAD, DRP = DR + PAD, NE = DL * DR;
  static constexpr int QR = 8;                                 // entries per quarter-warp list (<= 16 x 16 rows / 48 + 2)
  // int16 row lists, cost histogram / cursors (32 ints), the block's resident-row offsets
  // (16 x 16 ints) and three scalars
  static constexpr int QLIST = (NQ * QR * 2 + 32 * 4 + 16 * CH_ROWS * 4 + 4 * 4 + 7) / 8;
  static constexpr int FIXED = 256 + 1024 + 16 * CH_ROWS + QLIST;  // W scratch, history, row table, row lists
  static constexpr int PER_NB = CH_ROWS * DLP + CH_ROWS * DRP;  // L rows + Y/Z rows per chunk
  static constexpr int NB_FIT = (SMEM_MAX / 8 - 64 - FIXED - CH_ROWS * DLP) / PER_NB;
  static constexpr int NB = NB_FIT > 16 ? 16 : NB_FIT;        // chunks per block
  static constexpr int L_ROWS = NB * CH_ROWS + CH_ROWS;       // + one chunk of rows past the block
  static constexpr int L_OFF = 0;
  static constexpr int YZ_OFF = L_OFF + L_ROWS * DLP;         // NB x CH_ROWS x DRP (also the reduce staging)
  static constexpr int W_OFF = YZ_OFF + NB * CH_ROWS * DRP;
  static constexpr int H_OFF = W_OFF + 256;
  static constexpr int C_OFF = H_OFF + 1024;
  static constexpr int Q_OFF = C_OFF + NB * CH_ROWS;    // one int2 per row of a block
  static constexpr int DOUBLES = Q_OFF + QLIST;
  static constexpr size_t BYTES = (size_t)DOUBLES * 8 + 3 * 8;  // + mbarriers (L load, reduce operands, resident R)
  static_assert(NB >= 4, "at least four chunks per block");
  static_assert(NB * CH_ROWS <= NQ * (QR - 2), "quarter row lists hold a block's rows");
  static_assert(NB * CH_ROWS <= 256 && 2 * NB * CH_ROWS + 1 <= NB * CH_ROWS * DRP, "row ids fit 8 bits; setup scratch fits Y/Z");
  static_assert(BYTES <= SMEM_MAX, "shared memory per CTA");
  static_assert(L_ROWS * DLP + NB * CH_ROWS * DRP >= DL * DRP + DR * DRP + DL * DRP,
                "back-transform staging lives in the L and Y/Z buffers");
  static_assert(NB * CH_ROWS * DRP >= DL * DRP, "the step is staged in the Y/Z buffer");
};

__device__ long long g_ws_prof[6 * 1025];  // profiling instantiation only (ks_debug_richardson_phases)
__device__ long long g_ws_split[8];        // profiling: CTA 0 apply split, summed over iterations
__device__ unsigned long long g_ws_cta[2 * 256];  // profiling: per-CTA apply start / end (globaltimer) at iteration 5

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Grid barrier: one arrival counter (red.release.gpu), polled by one thread per CTA with acquire
// loads; counts are monotonic (target = epoch x grid), so nothing is reset between barriers.
// (Measured at c3 against cooperative_groups' grid sync -- the same -- and against a two-level
// counter tree with acq_rel group atomics -- ~1.7k cycles slower per barrier.)
constexpr int BAR_WORDS = 32;

__device__ __forceinline__ void red_add_release_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned* ctr, int G, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_add_release_gpu(ctr, 1u);
    while (ld_acquire_gpu(ctr) < (unsigned)G * epoch) {
    }
  }
  __syncthreads();
}

// N row tiles of Y = L X' (m16n8 tiles of one n8 strip, tiles t0, t0 + WPS, ...): N independent
// m16n8k4 chains over the k-steps, X' fragments in registers, results to the Y/Z rows
template <int N, int XK, int DLP, int DRP, int WPS>
__device__ __forceinline__ void y_pass(const double* Ls, double* YZ, int t0, const double (&xf)[XK], int g, int t4,
                                       int n0) {
  double acc[N][4];
#pragma unroll
  for (int i = 0; i < N; i++) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
#pragma unroll
  for (int k = 0; k < XK; k++) {
#pragma unroll
    for (int i = 0; i < N; i++) {
      const double* L = Ls + (t0 + i * WPS) * CH_ROWS * DLP;
      dmma_16x8x4(acc[i], L[g * DLP + 4 * k + t4], L[(g + 8) * DLP + 4 * k + t4], xf[k]);
    }
  }
#pragma unroll
  for (int i = 0; i < N; i++) {
    double* Y = YZ + (t0 + i * WPS) * CH_ROWS * DRP;
    *reinterpret_cast<double2*>(&Y[g * DRP + n0]) = make_double2(acc[i][0], acc[i][1]);
    *reinterpret_cast<double2*>(&Y[(g + 8) * DRP + n0]) = make_double2(acc[i][2], acc[i][3]);
  }
}

template <int DL, int DR, bool PROF>
__global__ void __launch_bounds__(NT, 1) richardson_phased_kernel(PArgs a) {
  using S = PhSmem<DL, DR>;
  constexpr int DLP = S::DLP, DRP = S::DRP, NE = S::NE, ROWCAP = S::NB * CH_ROWS;
  constexpr int GT_N = DR / 8, G_TILES = (DL / 16) * GT_N;
  constexpr int G_PER_W = (G_TILES + MW - 1) / MW;
  constexpr int Y_STRIPS = DR / 8;     // n8 strips of a 16-row Y tile
  static_assert(MW % Y_STRIPS == 0, "strips divide the DMMA warps");
  constexpr int WPS = MW / Y_STRIPS;   // DMMA warps per strip (they split the row tiles)
  constexpr int YB = 2;                // Y row tiles in flight per warp
  constexpr int XK = DL / 4;           // k-steps of Y = L X' (X' fragments per strip)
  constexpr int QE2 = DR / 16;         // double2 per lane of a quarter-warp row
  constexpr int SB = 2;                // samples per step of the sample phase
  constexpr int PAIR_C = 3;            // rows of >= PAIR_C steps are split over two quarter-warps
  extern __shared__ __align__(128) double sm[];
  uint64_t* lbar = reinterpret_cast<uint64_t*>(sm + S::DOUBLES);
  uint64_t* auxbar = lbar + 1;
  uint64_t* rbar = lbar + 2;
  int* rtab = reinterpret_cast<int*>(sm + S::C_OFF);  // per row of the block: sample range [tb, te)
  // sample-phase work lists: per quarter-warp, its entries (row | PAIRED | PIECE_B); per row, the
  // slot of its right rows in the resident region (or -1)
  unsigned short* qrows = reinterpret_cast<unsigned short*>(sm + S::Q_OFF);
  int* qhist = reinterpret_cast<int*>(qrows + NQ * S::QR);  // 16 cost buckets, then 16 cursors
  int* roff = qhist + 32;
  int* qscal = roff + 16 * CH_ROWS;  // [0]: paired rows, [1]: resident samples of the block
  double* Ls = sm + S::L_OFF;
  double* Ws = sm + S::W_OFF;
  double* Hs = sm + S::H_OFF;
  __shared__ int s_flag;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int G = gridDim.x, b = blockIdx.x;
  const bool is_mma = warp < MW;
  const bool prof = PROF && b == 0 && tid == 0;

  // this CTA's share of the sketch: the left rows and samples of its chunk range (contiguous in
  // the packed slabs; a row split between two CTAs' chunks contributes its samples to each)
  if (a.apply_only && a.stop && *a.stop) return;  // the sharded loop has stopped: a uniform no-op
  const int64_t c_beg = a.range[b], c_end = a.range[b + 1];
  int64_t u0 = 0, t_lo = 0, t_hi = 0;
  int nrows = 0;
  if (c_end > c_beg) {
    const Chunk cf = a.chunks[c_beg], cl = a.chunks[c_end - 1];
    u0 = cf.u_b;
    nrows = (int)(cl.u_e - cf.u_b);
    t_lo = cf.t_b;
    t_hi = cl.t_e;
  }
  const int nblk = (nrows + ROWCAP - 1) / ROWCAP;
  const bool resident = nblk <= 1;  // the L rows stay loaded for the whole solve
  const int epc = ((NE + G - 1) / G + 1) & ~1;  // reduce slice per CTA
  // Shared-memory layout.  With several row blocks: L (L_ROWS) | Y/Z (ROWCAP rows) at fixed
  // offsets.  When the CTA's rows fit one block, Y/Z follows the rows the tiles read and the space
  // the block leaves free holds a resident copy of part of the CTA's right rows r_t (loaded once
  // per launch): their share of the per-iteration L2 stream of the sample phase is gone.
  double* YZ = sm + S::YZ_OFF;
  double* Rres = nullptr;
  int rcap = 0;  // right rows that fit the resident region
  if (resident && nrows > 0 && !a.apply_only) {
    const int lrows = ((nrows + CH_ROWS - 1) / CH_ROWS) * CH_ROWS;
    YZ = Ls + (lrows + CH_ROWS) * DLP;  // the tiles read L rows < lrows; one chunk more, as L_ROWS
    const int yz = max(lrows * DRP, max(G * epc, DL * DRP));  // also the reduce operands and the step
    Rres = YZ + ((yz + 15) & ~15);  // 128-byte aligned
    rcap = max(0, (int)((sm + S::W_OFF) - Rres) / DRP);
  }
  double* AUXs = YZ;  // reduce operands (the Y/Z rows are dead by then)
  if (tid == 0) {
    mbar_init(lbar, 1);
    mbar_init(auxbar, 1);
    mbar_init(rbar, 1);
    fence_barrier_init();
  }
  // rows past the block are read by the Y / G tiles (multiplied into Y rows the sample phase
  // zeroes, or by zero rows of Z): keep them finite
  for (int e = tid; e < S::L_ROWS * DLP; e += NT) Ls[e] = 0.0;
  __syncthreads();
  unsigned epoch = 0;
  uint32_t auxphase = 0, lphase = 0;
  int q_rows = 0, q_steps = 0, q_wsteps = 0;  // this quarter-warp's sample-phase rows / steps, its warp's steps
  long long sp[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // profiling: apply split of CTA 0
  long long pt = 0;
  auto split = [&](int k) {
    if (prof) {
      const long long now = clock64();
      sp[k] += now - pt;
      pt = now;
    }
  };

  // DMMA-warp state: X' fragments of strip (warp % Y_STRIPS): x'[4k + t4][8 strip + g]
  const int ystrip = warp % Y_STRIPS, ywarp = warp / Y_STRIPS;
  double xf[XK];
#pragma unroll
  for (int k = 0; k < XK; k++)
    xf[k] = a.apply_only == 2 ? __ldg(&a.x_in[(4 * k + t4) * DR + 8 * ystrip + g]) : 0.0;
  // reduce-thread state (one element of this CTA's slice per 8-thread group, lane ql == 0):
  // rhs', dinv, x' and the last step' of that element
  double my_rhs = 0.0, my_dv = 0.0, my_x = 0.0, my_st = 0.0;
  double tol = 0.0;
  int status = 0, iters = 0, hlen = 0;

  const int it_first = a.apply_only == 2 ? 0 : -1, it_last = a.apply_only ? it_first + 1 : a.max_iters;
  for (int it = it_first; it < it_last; it++) {
    const bool rp = it < 0;  // right-hand-side pass: s_t = v_t (v_t b_t), no Y
    if (prof && !rp) {
      g_ws_prof[it * 6 + 0] = clock64();
      pt = clock64();
    }
    if (PROF && it == 5 && tid == 0 && b < 256) g_ws_cta[2 * b] = gtimer();
    // ---------------- apply: G = sum_c L_c^T Z_c ----------------
    // element e of CTA b's partial G goes to the slice of its reducer c = e / epc at
    // part[(c G + b) epc + e - c epc]: a reducer's G x epc operands are one contiguous block.  With
    // several row blocks the partial accumulates there between blocks (the G accumulators live
    // only in the G phase, so the sample phase has the registers for deep load batches).
    auto part_at = [&](int tile, int h) {
      const int m0 = (tile / GT_N) * 16, n0 = (tile % GT_N) * 8;
      const int e = (m0 + g + 8 * h) * DR + n0 + 2 * t4;
      const int c = e / epc;
      return reinterpret_cast<double2*>(a.part + ((size_t)c * G + b) * epc + (e - c * epc));
    };
    if (nblk == 0 && is_mma) {  // no rows: a zero partial
#pragma unroll
      for (int i = 0; i < G_PER_W; i++)
        if (warp * G_PER_W + i < G_TILES)
          for (int h = 0; h < 2; h++) *part_at(warp * G_PER_W + i, h) = make_double2(0.0, 0.0);
    }
    for (int blk = 0; blk < nblk; blk++) {
      const int r0 = blk * ROWCAP, nbr = min(ROWCAP, nrows - r0);  // the block's rows: u0 + [r0, r0 + nbr)
      const int ntile = (nbr + CH_ROWS - 1) / CH_ROWS;
      if (!resident || it == it_first) {  // first pass of the launch, or rows that do not stay resident
        // the block's left rows (contiguous in the packed slab), one bulk copy, and each row's
        // sample range within this CTA's samples
        if (tid == 0) {
          const uint32_t bytes = (uint32_t)(nbr * DLP * 8);
          mbar_arrive_expect_tx(lbar, bytes);
          bulk_copy(Ls, a.Lpack + (u0 + r0) * DLP, bytes, lbar);
        }
        for (int r = tid; r < nbr; r += NT) {
          const int64_t u = u0 + r0 + r;
          rtab[2 * r] = (int)(ks_max64(__ldg(&a.seg[u]), t_lo) - t_lo);
          rtab[2 * r + 1] = (int)(ks_min64(__ldg(&a.seg[u + 1]), t_hi) - t_lo);
        }
        if (tid < 32) qhist[tid] = 0;
        __syncthreads();
        // Sample-phase work lists.  The block's rows are ranked by cost (steps of SB samples,
        // decreasing).  The heaviest rows (>= PAIR_C steps, at most NQ / 2 of them) are each split
        // in two halves run side by side by a pair of quarter-warps of one warp, their partial z
        // summed with one shuffle; the other rows are dealt to the quarter-warps in snake order
        // (the largest ones to the quarters without a pair).  Every quarter then has about the
        // same number of steps.  Rows are independent and a row's samples are always summed in the
        // same order, so the assignment (ties broken by atomics) does not change any result.
        // In resident mode the right rows of the heaviest rows -- the critical path -- are copied
        // to shared memory, in rank order while they fit.
        int* sc_rank = reinterpret_cast<int*>(YZ);  // setup scratch: row of each rank, count prefix
        int* sc_pre = sc_rank + ROWCAP;
        for (int r = tid; r < nbr; r += NT) atomicAdd(&qhist[min(15, (rtab[2 * r + 1] - rtab[2 * r] + SB - 1) / SB)], 1);
        __syncthreads();
        if (tid == 0) {  // exclusive prefix over decreasing cost: qhist[c] = rows costing more than c
          int acc = 0;
          for (int c = 15; c >= 0; c--) {
            const int h = qhist[c];
            qhist[c] = acc;
            acc += h;
          }
          qscal[0] = min(qhist[PAIR_C - 1], NQ / 2);
        }
        __syncthreads();
        for (int r = tid; r < nbr; r += NT) {
          const int c = min(15, (rtab[2 * r + 1] - rtab[2 * r] + SB - 1) / SB);
          sc_rank[qhist[c] + atomicAdd(&qhist[16 + c], 1)] = r;
        }
        __syncthreads();
        const int npair = qscal[0];
        if (warp == 0) {  // sample counts of the ranks, exclusive prefix (nbr <= 256: 8 per lane)
          int loc[8], sum = 0;
#pragma unroll
          for (int j = 0; j < 8; j++) {
            const int k = lane * 8 + j;
            loc[j] = k < nbr ? rtab[2 * sc_rank[k] + 1] - rtab[2 * sc_rank[k]] : 0;
            sum += loc[j];
          }
          int inc = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
          }
          int run = inc - sum;
#pragma unroll
          for (int j = 0; j < 8; j++) {
            if (lane * 8 + j <= nbr) sc_pre[lane * 8 + j] = run;
            run += loc[j];
          }
          if (lane == 31 && nbr == 256) sc_pre[256] = run;
        }
        __syncthreads();
        const int cap = (resident && it == it_first) ? rcap : 0;
        for (int k = tid; k < nbr; k += NT) {
          const int r = sc_rank[k];
          const bool res = sc_pre[k + 1] <= cap;
          roff[r] = res ? sc_pre[k] : -1;
          if (res && (k + 1 == nbr || sc_pre[k + 2] > cap)) qscal[1] = sc_pre[k + 1];
          if (k < npair) {
            qrows[(2 * k) * S::QR] = (unsigned short)(r | 0x100);
            qrows[(2 * k + 1) * S::QR] = (unsigned short)(r | 0x300);
          } else {
            const int kk = k - npair, round = kk / NQ, pos = kk - round * NQ;
            const int q = (round & 1) ? pos : NQ - 1 - pos;
            qrows[q * S::QR + round + (q < 2 * npair ? 1 : 0)] = (unsigned short)r;
          }
        }
        if (tid == 0 && (cap == 0 || sc_pre[1] > cap)) qscal[1] = 0;
        __syncthreads();
        const int nres = qscal[1];
        if (nres > 0) {  // resident mode, first pass: the heaviest rows' right rows
          if (tid == 0) mbar_arrive_expect_tx(rbar, (uint32_t)(nres * DRP * 8));
          __syncthreads();
          for (int r = tid; r < nbr; r += NT)
            if (roff[r] >= 0)
              bulk_copy(Rres + roff[r] * DRP, a.Rpack + (t_lo + rtab[2 * r]) * DRP,
                        (uint32_t)((rtab[2 * r + 1] - rtab[2 * r]) * DRP * 8), rbar);
        }
        {  // this quarter's entries and steps; the warp's step count (its quarters run in lockstep)
          const int qid = warp * 4 + (lane >> 3);
          q_rows = qid < 2 * npair ? 1 : 0;
          q_steps = 0;
          for (int round = 0; round * NQ < nbr - npair; round++) {
            const int kk = round * NQ + ((round & 1) ? qid : NQ - 1 - qid);
            if (kk < nbr - npair) q_rows++;
          }
          mbar_wait(lbar, lphase);
          lphase ^= 1;
          for (int k = 0; k < q_rows; k++) {
            const int e = qrows[qid * S::QR + k], r = e & 0xff;
            const int cnt = rtab[2 * r + 1] - rtab[2 * r];
            q_steps += max(1, ((e & 0x100) ? (cnt + 1) / 2 + SB - 1 : cnt + SB - 1) / SB);
          }
          q_wsteps = max(q_steps, __shfl_xor_sync(0xffffffffu, q_steps, 8));
          q_wsteps = max(q_wsteps, __shfl_xor_sync(0xffffffffu, q_wsteps, 16));
          if (nres > 0) mbar_wait(rbar, 0);
          __syncthreads();  // the Y/Z scratch is free again
        }
      }
      split(0);
      // ---- Y phase: Y = L X' over the block's rows: m16n8 tile (row tile, strip); the row tiles
      // of a strip are split over its warps, YB of them in flight per warp
      if (!rp && is_mma) {
        // passes of YB row tiles, then one pass over the remaining ones: every DMMA issued is a
        // real one (no predicated-off tiles)
        int t0 = ywarp;
        for (; t0 + (YB - 1) * WPS < ntile; t0 += WPS * YB)
          y_pass<YB, XK, DLP, DRP, WPS>(Ls, YZ, t0, xf, g, t4, 8 * ystrip + 2 * t4);
        const int rem = t0 < ntile ? (ntile - t0 + WPS - 1) / WPS : 0;
        if constexpr (YB > 1) if (rem == 1) y_pass<1, XK, DLP, DRP, WPS>(Ls, YZ, t0, xf, g, t4, 8 * ystrip + 2 * t4);
        if constexpr (YB > 2) if (rem == 2) y_pass<2, XK, DLP, DRP, WPS>(Ls, YZ, t0, xf, g, t4, 8 * ystrip + 2 * t4);
        if constexpr (YB > 3) if (rem == 3) y_pass<3, XK, DLP, DRP, WPS>(Ls, YZ, t0, xf, g, t4, 8 * ystrip + 2 * t4);
        if constexpr (YB > 4) if (rem == 4) y_pass<4, XK, DLP, DRP, WPS>(Ls, YZ, t0, xf, g, t4, 8 * ystrip + 2 * t4);
        if constexpr (YB > 5) if (rem == 5) y_pass<5, XK, DLP, DRP, WPS>(Ls, YZ, t0, xf, g, t4, 8 * ystrip + 2 * t4);
        if constexpr (YB > 6) if (rem == 6) y_pass<6, XK, DLP, DRP, WPS>(Ls, YZ, t0, xf, g, t4, 8 * ystrip + 2 * t4);
        if constexpr (YB > 7) if (rem == 7) y_pass<7, XK, DLP, DRP, WPS>(Ls, YZ, t0, xf, g, t4, 8 * ystrip + 2 * t4);
      }
      __syncthreads();
      split(1);
      // ---- sample phase: each quarter-warp runs through its list of rows (dealt by cost when the
      // block was loaded); z_u is written over y_u, rows past the block (up to the row-tile
      // boundary) are zeroed
      {
        const int ql = lane & 7, qid = warp * 4 + (lane >> 3);
        for (int rr = nbr + qid; rr < ntile * CH_ROWS; rr += NQ) {
          double* YZr = YZ + rr * DRP;
#pragma unroll
          for (int m = 0; m < QE2; m++) *reinterpret_cast<double2*>(&YZr[2 * ql + 16 * m]) = make_double2(0.0, 0.0);
        }
        const double* Rbase = a.Rpack + t_lo * DRP;
        const unsigned short* myrows = qrows + qid * S::QR;
        const int nsteps = q_steps, wsteps = q_wsteps;
        const unsigned pmask = 0xffffu << (lane & 16);  // the 16 lanes of this quarter's pair
        int k = 0, cr = 0, t = 0, te = 0, srem = 0, ro = -1, rtb = 0, ent = 0;
        double2 y[QE2], z[QE2];
#pragma unroll
        for (int m = 0; m < QE2; m++) z[m] = y[m] = make_double2(0.0, 0.0);
        auto start_row = [&]() {  // entry k: a row, or one half of a paired row
          ent = myrows[k];
          cr = ent & 0xff;
          rtb = rtab[2 * cr];
          const int tend = rtab[2 * cr + 1], half = (tend - rtb + 1) / 2;
          t = (ent & 0x200) ? rtb + half : rtb;
          te = (ent & 0x100) ? ((ent & 0x200) ? tend : rtb + half) : tend;
          srem = max(1, (((ent & 0x100) ? half : tend - rtb) + SB - 1) / SB);
          ro = roff[cr];
          const double* YZr = YZ + cr * DRP;
#pragma unroll
          for (int m = 0; m < QE2; m++) {
            y[m] = rp ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(&YZr[2 * ql + 16 * m]);
            z[m] = make_double2(0.0, 0.0);
          }
        };
        if (k < q_rows) start_row();
        for (int step = 0; step < wsteps; step++) {
          const int n = step < nsteps ? max(0, min(SB, te - t)) : 0;
          // SB samples per step: their loads in flight together (the right rows come from L2),
          // dot products and shuffle reductions interleaved; z accumulates in sample order.
          // Every load is of a valid row (samples past the step's count re-read the last one and
          // get weight 0), so the step has no branches and no zero fills.
          double2 rv[SB][QE2], pv[SB];
#pragma unroll
          for (int i = 0; i < SB; i++) {
            const int ti = max(0, min(t + i, te - 1));
            const double* Rt = ro >= 0 ? Rres + (ro + ti - rtb) * DRP : Rbase + ti * DRP;
#pragma unroll
            for (int m = 0; m < QE2; m++) rv[i][m] = *reinterpret_cast<const double2*>(&Rt[2 * ql + 16 * m]);
            pv[i] = *reinterpret_cast<const double2*>(&Rt[DR]);  // v_t, v_t b_t (row padding)
            if (i >= n) pv[i].x = 0.0;
          }
          double sv[SB];
          if (rp) {
#pragma unroll
            for (int i = 0; i < SB; i++) sv[i] = pv[i].x * pv[i].y;
          } else {
            double d[SB];
#pragma unroll
            for (int i = 0; i < SB; i++) {
              d[i] = 0.0;
#pragma unroll
              for (int m = 0; m < QE2; m++) d[i] = fma(y[m].y, rv[i][m].y, fma(y[m].x, rv[i][m].x, d[i]));
            }
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {  // within the quarter (full-warp shuffles, lanes stay in their 8-group)
              double e[SB];
#pragma unroll
              for (int i = 0; i < SB; i++) e[i] = __shfl_xor_sync(0xffffffffu, d[i], o);
#pragma unroll
              for (int i = 0; i < SB; i++) d[i] += e[i];
            }
#pragma unroll
            for (int i = 0; i < SB; i++) sv[i] = pv[i].x * (pv[i].x * d[i]);
          }
#pragma unroll
          for (int i = 0; i < SB; i++) {  // sv = 0 past the step's count: z unchanged
#pragma unroll
            for (int m = 0; m < QE2; m++) {
              z[m].x = fma(sv[i], rv[i][m].x, z[m].x);
              z[m].y = fma(sv[i], rv[i][m].y, z[m].y);
            }
          }
          t += SB;
          if (step < nsteps && --srem == 0) {  // the entry is done: z_u over y_u (each lane its own elements)
            if (ent & 0x100) {  // both halves of a paired row end on this step: z_u = z_first + z_second
#pragma unroll
              for (int m = 0; m < QE2; m++) {
                z[m].x += __shfl_xor_sync(pmask, z[m].x, 8);
                z[m].y += __shfl_xor_sync(pmask, z[m].y, 8);
              }
            }
            if (!(ent & 0x200)) {
              double* YZr = YZ + cr * DRP;
#pragma unroll
              for (int m = 0; m < QE2; m++) *reinterpret_cast<double2*>(&YZr[2 * ql + 16 * m]) = z[m];
            }
            if (++k < q_rows) start_row();
          }
        }
      }
      __syncthreads();
      split(2);
      // ---- G phase: G += L^T Z over the block's rows (K = rows, zero Z rows past the block)
      if (is_mma) {
        double gacc[G_PER_W][4];
#pragma unroll
        for (int i = 0; i < G_PER_W; i++) {
          if (blk > 0 && warp * G_PER_W + i < G_TILES) {
            const double2 lo = *part_at(warp * G_PER_W + i, 0), hi = *part_at(warp * G_PER_W + i, 1);
            gacc[i][0] = lo.x; gacc[i][1] = lo.y; gacc[i][2] = hi.x; gacc[i][3] = hi.y;
          } else {
            gacc[i][0] = gacc[i][1] = gacc[i][2] = gacc[i][3] = 0.0;
          }
        }
        const int nk = (nbr + 3) / 4;
        // a warp's tiles share their rows of L^T when they lie in one m16 band (e.g. d_L = d_R = 64:
        // 32 tiles, 4 per warp, 8 per band): then one pair of A fragments per k-step
        constexpr bool BAND = G_TILES % MW == 0 && GT_N % G_PER_W == 0;
        if constexpr (BAND) {
          const int m0 = (warp * G_PER_W / GT_N) * 16, n0 = (warp * G_PER_W % GT_N) * 8;
#pragma unroll 2
          for (int kk = 0; kk < nk; kk++) {
            const double* Lr = Ls + (4 * kk + t4) * DLP;
            const double* Zr = YZ + (4 * kk + t4) * DRP + n0 + g;
            const double a0 = Lr[m0 + g], a1 = Lr[m0 + g + 8];
#pragma unroll
            for (int i = 0; i < G_PER_W; i++) dmma_16x8x4(gacc[i], a0, a1, Zr[8 * i]);
          }
        } else {
          for (int kk = 0; kk < nk; kk++) {
            const double* Lr = Ls + (4 * kk + t4) * DLP;
            const double* Zr = YZ + (4 * kk + t4) * DRP;
#pragma unroll
            for (int i = 0; i < G_PER_W; i++) {
              const int tile = warp * G_PER_W + i;
              if (tile < G_TILES) {
                const int m0 = (tile / GT_N) * 16, n0 = (tile % GT_N) * 8;
                dmma_16x8x4(gacc[i], Lr[m0 + g], Lr[m0 + g + 8], Zr[n0 + g]);
              }
            }
          }
        }
        split(7);  // profiling: the G DMMA loop (split 3 is then the partial stores)
#pragma unroll
        for (int i = 0; i < G_PER_W; i++)
          if (warp * G_PER_W + i < G_TILES)
            for (int h = 0; h < 2; h++)
              *part_at(warp * G_PER_W + i, h) = make_double2(gacc[i][2 * h], gacc[i][2 * h + 1]);
      }
      split(3);
      __syncthreads();  // the block's L and Y/Z rows are free
    }
    // ---------------- partials -> reducers (written by the G phase) ----------------
    if (is_mma) asm volatile("fence.proxy.async.global;" ::: "memory");  // read back by the bulk-copy proxy
    if (prof && !rp) g_ws_prof[it * 6 + 1] = clock64();
    if (PROF && it == 5 && tid == 0 && b < 256) g_ws_cta[2 * b + 1] = gtimer();
    grid_barrier(a.flags, G, ++epoch);
    if (prof && !rp) g_ws_prof[it * 6 + 2] = clock64();
    if (prof) pt = clock64();
    // ---------------- reduce: step' = dinv o (sum_cta G + lam x' - rhs') ----------------
    {
      const int e0 = b * epc, e1 = min(NE, e0 + epc);
      const int ne_cta = e1 > e0 ? e1 - e0 : 0;
      if (ne_cta > 0) {
        if (tid == 0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          const uint32_t bytes = (uint32_t)(G * epc * 8);
          mbar_arrive_expect_tx(auxbar, bytes);
          bulk_copy(AUXs, a.part + (size_t)b * G * epc, bytes, auxbar);
        }
        mbar_wait(auxbar, auxphase);
        auxphase ^= 1;
      }
      split(4);
      const int eo = tid >> 3, ql = lane & 7;
      const unsigned qmask = 0xffu << (lane & 24);
      if (eo < ne_cta) {  // 8 threads per element: fixed-order compensated sum over the CTA partials
        double s = 0.0, cmp = 0.0;
        for (int p = ql; p < G; p += 8) {
          const double vv = AUXs[p * epc + eo];
          const double tt = s + vv;
          cmp += (fabs(s) >= fabs(vv)) ? ((s - tt) + vv) : ((vv - tt) + s);
          s = tt;
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          const double os = __shfl_xor_sync(qmask, s, o);
          const double oc = __shfl_xor_sync(qmask, cmp, o);
          const bool up = lane & o;
          const double lo = up ? os : s, hi = up ? s : os;
          const double tt = lo + hi;
          const double bb = tt - lo;
          const double err = (lo - (tt - bb)) + (hi - bb);
          cmp = (up ? oc : cmp) + (up ? cmp : oc) + err;
          s = tt;
        }
        if (ql == 0 && a.apply_only) {
          a.g_out[e0 + eo] = s + cmp;  // this GPU's reduced partial (the sharded loop all-reduces it)
        } else if (ql == 0) {
          const int e = e0 + eo, i = e / DR, k = e - i * DR;
          double r;
          if (rp) {
            r = s + cmp;
            a.rhs[e] = r;
            if (a.dinv) {
              my_dv = __ldg(&a.dinv[e]);
            } else {  // solvers.py:186-191 on kron(wL, wR) + lam
              const double ev = __dadd_rn(__dmul_rn(__ldg(&a.wL[i]), __ldg(&a.wR[k])), a.lam);
              my_dv = ev > 0.0 ? __ddiv_rn(1.0, ev) : 0.0;
            }
            my_rhs = r;
          } else {
            r = __dsub_rn(__dadd_rn(s + cmp, __dmul_rn(a.lam, my_x)), my_rhs);
          }
          my_st = r * my_dv;
          a.step[i * DRP + k] = my_st;  // padded rows: fetched with one bulk copy
        }
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (a.apply_only) return;
    if (prof && !rp) g_ws_prof[it * 6 + 3] = clock64();
    grid_barrier(a.flags, G, ++epoch);
    if (prof) pt = clock64();
    if (prof && !rp) g_ws_prof[it * 6 + 4] = clock64();
    // ---------------- norm, stopping rules (solvers.py:226-247), update ----------------
    // every CTA fetches step' (one bulk copy) and forms ||step'|| from it in the same fixed order
    // (identical in every CTA); tid 0 applies the stopping and divergence rules
    if (tid == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const uint32_t bytes = (uint32_t)(DL * DRP * 8);
      mbar_arrive_expect_tx(auxbar, bytes);
      bulk_copy(AUXs, a.step, bytes, auxbar);
    }
    mbar_wait(auxbar, auxphase);  // also before a stop: the buffers are reused after the loop
    auxphase ^= 1;
    split(6);
    double sq = 0.0;
    {  // the same order as a strided loop, loads issued together
      constexpr int NPT = (NE + NT - 1) / NT;
      double sv[NPT];
#pragma unroll
      for (int i = 0; i < NPT; i++) {
        const int e = tid + i * NT;
        sv[i] = e < NE ? AUXs[(e / DR) * DRP + e % DR] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < NPT; i++)
        if (tid + i * NT < NE) sq = fma(sv[i], sv[i], sq);
    }
    const double nrm = sqrt(block_sum(sq, Ws + 192));
    if (rp) {  // tol = residual_tol * ||P rhs|| (solvers.py:212-214)
      tol = a.residual_tol * fmax(nrm, DBL_MIN);
      continue;  // block_sum ended with a barrier: the step buffer is free
    }
    if (tid == 0) {
      Hs[it] = nrm;
      int div = 0;  // solvers.py:240-247: five increases in a row and a tenfold growth
      if (it + 1 > 5) {
        bool inc = true;
        for (int i = it - 5; i < it; i++) inc &= Hs[i + 1] > Hs[i];
        div = inc && (Hs[it] > 10.0 * Hs[it - 5]);
      }
      s_flag = div;
    }
    __syncthreads();
    split(5);
    hlen = it + 1;
    if (nrm <= tol) {
      status = 1;
      break;
    }
    if (s_flag) {
      status = 2;
      break;
    }
    if (is_mma) {
#pragma unroll
      for (int k = 0; k < XK; k++)
        xf[k] = __dsub_rn(xf[k], __dmul_rn(a.damping, AUXs[(4 * k + t4) * DRP + 8 * ystrip + g]));
    }
    my_x = __dsub_rn(my_x, __dmul_rn(a.damping, my_st));
    iters = it + 1;
    if (prof) g_ws_prof[it * 6 + 5] = clock64();
    __syncthreads();
  }
  __syncthreads();
  // back to the natural basis, one row per CTA: x = VL x' VR^T (CTAs 0..DL-1) and, when asked,
  // rhs = VL rhs' VR^T (CTAs DL..2 DL-1); the L and Y/Z buffers (contiguous) are free now
  double* Xs = Ls;
  double* VRts = Xs + DL * DRP;
  double* Ms = VRts + DR * DRP;
  const bool want_rhs = a.rhs_nat_out != nullptr;
  if (b < (want_rhs ? 2 * DL : DL)) {
    if (is_mma && ywarp == 0) {
#pragma unroll
      for (int k = 0; k < XK; k++) Xs[(4 * k + t4) * DRP + 8 * ystrip + g] = xf[k];
    }
    __syncthreads();
    for (int row = b; row < (want_rhs ? 2 * DL : DL); row += G) {
      const bool is_rhs = row >= DL;
      const int r = is_rhs ? row - DL : row;
      stage(VRts, a.VRt, DR, DR, DRP);
      if (is_rhs) stage(Ms, a.rhs, DL, DR, DRP);
      for (int k = tid; k < DL; k += NT) Ws[k] = __ldg(&a.VL[r * DL + k]);
      cp_async_wait_all();
      __syncthreads();
      vecmat(Ws, is_rhs ? Ms : Xs, DL, DR, DRP, Ws + 64);  // (VL M)[r, :]
      __syncthreads();
      vecmat(Ws + 64, VRts, DR, DR, DRP, Ws + 128);        // ((VL M) VR^T)[r, :]
      __syncthreads();
      double* dst = is_rhs ? a.rhs_nat_out : a.x_out;
      for (int c = tid; c < DR; c += NT) dst[r * DR + c] = Ws[128 + c];
      __syncthreads();
    }
  }
  if (prof)
    for (int k = 0; k < 8; k++) g_ws_split[k] = sp[k];
  if (b == 0) {
    for (int i = tid; i < hlen; i += NT) a.hist[i] = Hs[i];
    if (tid == 0) {
      a.state[0] = status;
      a.state[1] = iters;
      a.state[2] = hlen;
    }
  }
}

template <int DL, int DR, bool PROF>
int launch_one(cudaStream_t st, PArgs& a, int grid) {
  using S = PhSmem<DL, DR>;
  auto kern = richardson_phased_kernel<DL, DR, PROF>;
  KS_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES));
  int per_sm = 0;
  KS_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, S::BYTES));
  KS_REQUIRE(per_sm >= 1 && grid <= per_sm * ks::num_sms(), KS_ESIZE,
             "persistent Richardson kernel does not fit co-resident");
  KS_TRY_CUDA(cudaMemsetAsync(a.flags, 0, sizeof(unsigned) * BAR_WORDS, st));
  void* args[] = {&a};
  KS_TRY_CUDA(cudaLaunchCooperativeKernel((void*)kern, grid, NT, args, S::BYTES, st));
  return KS_OK;
}

template <int DL, int DR>
int launch_pair(cudaStream_t st, PArgs& a, int grid, bool prof) {
  return prof ? launch_one<DL, DR, true>(st, a, grid) : launch_one<DL, DR, false>(st, a, grid);
}

}  // namespace

static int block_chunks(int dL, int dR) {  // PhSmem<dL, dR>::NB
#define KS_NB(L, R) \
  if (dL == L && dR == R) return PhSmem<L, R>::NB;
  KS_NB(16, 16) KS_NB(16, 32) KS_NB(16, 64) KS_NB(32, 16) KS_NB(32, 32) KS_NB(32, 64) KS_NB(64, 16) KS_NB(64, 32)
  KS_NB(64, 64)
#undef KS_NB
  return 0;
}

namespace ks {

bool richardson_phased_supported(int dL, int dR, int grid) {
  auto ok = [](int d) { return d == 16 || d == 32 || d == 64; };
  if (!ok(dL) || !ok(dR) || grid > 192) return false;
  const int ne = dL * dR, epc = ((ne + grid - 1) / grid + 1) & ~1;
  // one reduce element per 8-thread group; the reduce operands fit the staging buffer (the Y/Z rows)
  const int64_t stage = (int64_t)block_chunks(dL, dR) * CH_ROWS * (dR + PAD);
  return epc <= NT / 8 && (int64_t)grid * epc <= stage;
}

int richardson_phased_launch(cudaStream_t st, PArgs& a, int dL, int dR, int grid, bool prof) {
  KS_REQUIRE(richardson_phased_supported(dL, dR, grid), KS_ESIZE, "phase-separated loop: unsupported geometry");
  KS_REQUIRE(a.eig_mode && a.rhs_in_kernel && a.flags, KS_EINVAL, "phase-separated loop runs in the eigenbasis");
  if (dL == 16 && dR == 16) return launch_pair<16, 16>(st, a, grid, prof);
  if (dL == 16 && dR == 32) return launch_pair<16, 32>(st, a, grid, prof);
  if (dL == 16 && dR == 64) return launch_pair<16, 64>(st, a, grid, prof);
  if (dL == 32 && dR == 16) return launch_pair<32, 16>(st, a, grid, prof);
  if (dL == 32 && dR == 32) return launch_pair<32, 32>(st, a, grid, prof);
  if (dL == 32 && dR == 64) return launch_pair<32, 64>(st, a, grid, prof);
  if (dL == 64 && dR == 16) return launch_pair<64, 16>(st, a, grid, prof);
  if (dL == 64 && dR == 32) return launch_pair<64, 32>(st, a, grid, prof);
  if (dL == 64 && dR == 64) return launch_pair<64, 64>(st, a, grid, prof);
  return KS_EINVAL;
}

}  // namespace ks

// Average cycles of CTA 0 per phase over the last profiled phase-separated run (after
// ks_debug_richardson_profile(1)): apply, flag barrier 1, reduce, flag barrier 2, norm + update,
// and the loop overhead to the next iteration's start.
extern "C" int ks_debug_richardson_phases(int32_t iters, double* out6) {
  if (iters < 2 || iters > 1024) return KS_EINVAL;
  long long h[6 * 1025];
  KS_TRY_CUDA(cudaMemcpyFromSymbol(h, g_ws_prof, sizeof(long long) * 6 * iters));
  for (int k = 0; k < 6; k++) out6[k] = 0.0;
  for (int it = 0; it + 1 < iters; it++) {
    const long long* p = &h[it * 6];
    for (int k = 0; k < 5; k++) out6[k] += (double)(p[k + 1] - p[k]);
    out6[5] += (double)(h[(it + 1) * 6] - p[5]);
  }
  for (int k = 0; k < 6; k++) out6[k] /= (iters - 1);
  return KS_OK;
}

// Profiling aid: CTA 0's apply phase of the last profiled run, SM cycles per iteration: L load
// wait, Y phase, sample phase, G phase (thread 0).
extern "C" int ks_debug_richardson_apply_split(int32_t iters, double* out8) {
  if (iters < 1) return KS_EINVAL;
  long long h[8];
  KS_TRY_CUDA(cudaMemcpyFromSymbol(h, g_ws_split, sizeof(h)));
  for (int k = 0; k < 8; k++) out8[k] = (double)h[k] / iters;
  return KS_OK;
}

// Profiling aid: per-CTA apply start / end (%globaltimer ns) of iteration 5 of the last profiled run,
// out[2 b], out[2 b + 1] (the spread of the ends is the skew the first grid barrier absorbs).
extern "C" int ks_debug_richardson_cta_apply(int32_t nctas, uint64_t* out) {
  if (nctas < 1 || nctas > 256) return KS_EINVAL;
  KS_TRY_CUDA(cudaMemcpyFromSymbol(out, g_ws_cta, sizeof(unsigned long long) * 2 * nctas));
  return KS_OK;
}
