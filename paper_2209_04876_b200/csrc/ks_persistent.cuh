// Shared definitions of the persistent Richardson loop kernels (ks_richardson_persistent.cu: the
// single-role kernel, natural basis or eigenbasis; ks_richardson_phased.cu: the phase-separated
// eigenbasis kernel) and of their device work plan: chunk geometry, kernel arguments, bulk-copy /
// staging helpers.
#pragma once
#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace ks_rich {

constexpr int CH_ROWS = 16;  // distinct left rows per chunk 
constexpr int PLAN_ROWS = 8;  // left rows per group of the device work plan (a chunk holds <= CH_ROWS)
constexpr int CH_S = 64;     // samples per chunk (>= DL: the free slab holds a DL x DRP matrix)
constexpr int PAD = 4;       // row padding (doubles) of packed / staged rows
constexpr int BARRIER_WORDS = 32;  // grid-barrier counter (own 128-byte line) of the phase-separated loop

struct Chunk {
  int64_t u_b, u_e;  // left rows [u_b, u_e)
  int64_t t_b, t_e;  // samples  [t_b, t_e)
};

struct PArgs {
  const double* Lpack;    // u_left x (DL+PAD)
  const double* Rpack;    // nnz x (DR+PAD); pad slot 0 carries v_t
  const int64_t* seg;     // u_left + 1
  const Chunk* chunks;
  const int64_t* range;   // grid + 1: chunk range of every CTA
  const double* VL;       // DL x DL
  const double* VR;       // DR x DR
  const double* VRt;      // DR x DR
  const double* dinv;     // DL x DR, or null: dinv(i, j) = pseudo-reciprocal(wL[i] wR[j] + lam)
  const double* wL;       // DL (eigenvalues of the left factor's Gram) when dinv is null
  const double* wR;       // DR
  double* rhs;            // DL x DR (input, or output when rhs_in_kernel)
  int rhs_in_kernel;      // pass -1 builds rhs = sum_t v_t (v_t b_t) L_u R_t^T (Rpack pad slot 1 = v_t b_t)
  int eig_mode;           // the packed rows are L VL / R VR: the loop runs in the preconditioner's
                          // eigenbasis, where the preconditioner is the diagonal dinv (no P3/P4)
  double* rhs_nat_out;    // eig_mode: VL rhs' VR^T (natural-order right-hand side), may be null
  double lam, damping, residual_tol;
  int max_iters;
  double* part;           // grid x DL x DR
  double* R;              // DL x DR
  double* T;              // DL x DR
  double* step;           // DL x DR
  double* rowsq;          // DL
  double* x_out;          // DL x DR
  double* hist;           // max_iters
  int* state;             // [status, iters, hist_len]
  unsigned* flags;        // grid-barrier counters (ks_rich::BARRIER_WORDS, zeroed before the launch)
  long long* prof;        // profiling build only: CTA 0's phase clocks, 6 per iteration
  // apply-only launches of the phase-separated kernel (the row-sharded loop, distributed.py):
  // 1 = right-hand-side pass, 2 = one normal-operator apply at x_in; the reduced d_L x d_R result
  // goes to g_out and the launch ends there (no step, no update); nothing runs when *stop != 0
  int apply_only;
  const double* x_in;     // d_L x d_R (eigenbasis x'), apply_only == 2
  double* g_out;          // d_L x d_R
  const int* stop;        // device flag (may be null)
};


__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// 16-byte global->shared copies that bypass registers and L1 (all issued back to back, so their
// L2 latencies overlap; ptxas would otherwise interleave loads with dependent arithmetic).
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// rows x cols (cols even) row-major global matrix -> padded smem (row stride ld, 16B aligned rows)
__device__ __forceinline__ void stage(double* dst, const double* __restrict__ src, int rows, int cols, int ld) {
  const int pairs = rows * (cols / 2);
  for (int e = threadIdx.x; e < pairs; e += blockDim.x) {
    const int i = e / (cols / 2), j = 2 * (e - i * (cols / 2));
    cp_async16(dst + i * ld + j, src + (size_t)i * cols + j);
  }
}

// out[j] = sum_k w[k] M[k][j] for j < cols (cols <= blockDim / 4); 4 threads per output,
// interleaved k-split.
__device__ __forceinline__ void vecmat(const double* w, const double* M, int K, int cols, int ld, double* out) {
  const int j = threadIdx.x >> 2, part = threadIdx.x & 3;
  double s = 0.0;
  if (j < cols)
    for (int k = part; k < K; k += 4) s = fma(w[k], M[k * ld + j], s);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (j < cols && part == 0) out[j] = s;
}

}  // namespace ks_rich

namespace ks {
// The phase-separated eigenbasis loop (ks_richardson_phased.cu).  Returns KS_OK or a KS_* error.
int richardson_phased_launch(cudaStream_t st, ks_rich::PArgs& a, int dL, int dR, int grid, bool prof);
// Geometry / device check for richardson_phased_launch (else the single-role kernel runs).
bool richardson_phased_supported(int dL, int dR, int grid);
}  // namespace ks
