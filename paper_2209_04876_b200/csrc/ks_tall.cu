// Split-K C(M x N) = alpha A^T B for tall operands (K >> M, N; M, N <= 128) on FP64 tensor cores.
// Used for the Gram matrices A~^T A~ (reference solvers.py:146, :439) and the JL projection
// G A~ (leverage.py:127).  Each CTA stages 32-row slabs of A and B in padded shared memory,
// runs DMMA m16n8k4 over its K-range and writes a private partial; a warp-per-output fixed-order
// reduction sums the partials (deterministic).
#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace {

constexpr int TK = 32;       // k rows per slab
constexpr int TT = 256;      // threads
constexpr int TW = TT / 32;  // warps

template <int MP, int NP>  // padded M, N (multiples of 16 / 8)
__global__ void __launch_bounds__(TT) tall_tn_kernel(int M, int N, int64_t K, int64_t chunk,
                                                     const double* __restrict__ A, int64_t a_ks, int64_t a_ms,
                                                     const double* __restrict__ B, int64_t b_ks, int64_t b_ns,
                                                     double* __restrict__ part) {
  constexpr int LDA = MP + 4, LDB = NP + 4;
  constexpr int TILES = (MP / 16) * (NP / 8);
  constexpr int PER_W = (TILES + TW - 1) / TW;
  extern __shared__ double tsm[];
  double* As = tsm;
  double* Bs = tsm + TK * LDA;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  const int64_t kbeg = (int64_t)blockIdx.x * chunk;
  const int64_t kend = ks_min64(K, kbeg + chunk);
  double acc[PER_W][4];
#pragma unroll
  for (int i = 0; i < PER_W; i++) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
  const bool a_kfast = (a_ks == 1);
  const bool b_kfast = (b_ks == 1);
  for (int64_t k0 = kbeg; k0 < kend; k0 += TK) {
    for (int e = tid; e < TK * MP; e += TT) {
      int kk, mm;
      if (a_kfast) { mm = e / TK; kk = e - mm * TK; } else { kk = e / MP; mm = e - kk * MP; }
      const int64_t gk = k0 + kk;
      const bool ok = gk < kend && mm < M;
      ks_cp_async8(&As[kk * LDA + mm], ok ? A + gk * a_ks + (int64_t)mm * a_ms : A, ok);
    }
    for (int e = tid; e < TK * NP; e += TT) {
      int kk, nn;
      if (b_kfast) { nn = e / TK; kk = e - nn * TK; } else { kk = e / NP; nn = e - kk * NP; }
      const int64_t gk = k0 + kk;
      const bool ok = gk < kend && nn < N;
      ks_cp_async8(&Bs[kk * LDB + nn], ok ? B + gk * b_ks + (int64_t)nn * b_ns : B, ok);
    }
    ks_cp_async_wait_all();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PER_W; i++) {
      const int tile = warp + i * TW;
      if (tile < TILES) {
        const int m0 = (tile / (NP / 8)) * 16, n0 = (tile % (NP / 8)) * 8;
#pragma unroll
        for (int kk = 0; kk < TK; kk += 4) {
          const double a0 = As[(kk + t4) * LDA + m0 + g];
          const double a1 = As[(kk + t4) * LDA + m0 + g + 8];
          const double b0 = Bs[(kk + t4) * LDB + n0 + g];
          dmma_16x8x4(acc[i], a0, a1, b0);
        }
      }
    }
    __syncthreads();
  }
  double* out = part + (int64_t)blockIdx.x * M * N;
#pragma unroll
  for (int i = 0; i < PER_W; i++) {
    const int tile = warp + i * TW;
    if (tile < TILES) {
      const int m0 = (tile / (NP / 8)) * 16, n0 = (tile % (NP / 8)) * 8;
      const int r0 = m0 + g, c0 = n0 + 2 * t4;
      if (r0 < M && c0 < N) out[r0 * N + c0] = acc[i][0];
      if (r0 < M && c0 + 1 < N) out[r0 * N + c0 + 1] = acc[i][1];
      if (r0 + 8 < M && c0 < N) out[(r0 + 8) * N + c0] = acc[i][2];
      if (r0 + 8 < M && c0 + 1 < N) out[(r0 + 8) * N + c0 + 1] = acc[i][3];
    }
  }
}

__global__ void reduce_parts_warp_kernel(const double* __restrict__ part, int64_t nparts, int64_t count,
                                         double alpha, double* __restrict__ out) {
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= count) return;
  double s = 0.0;
  for (int64_t k = lane; k < nparts; k += 32) s += part[k * count + e];
  s = warp_sum(s);
  if (lane == 0) out[e] = alpha * s;
}

// Second version for the aligned shapes of the solve (Grams of d = 16..128 factors, the JL
// product G A~ with r <= 80): 16-byte cp.async staging (k-fast A stored [m][k], m-fast A stored
// [k][m], n-fast B stored [k][n]), two-slab double buffering (the next slab's loads in flight
// while the current one's DMMAs run), TK2 = 16 k-rows per slab so that all SMs get a K-range.
constexpr int TK2 = 16;
__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}

// SYM (Gram A^T A: B == A, MP == NP, A m-fast): A staged once, only the m16 x n8 tiles that reach
// the upper triangle (n0 + 8 > m0) computed, the upper entries written with their mirrors.
template <int MP, int NP, bool AK, bool SYM = false>
__global__ void __launch_bounds__(TT) tall_tn2_kernel(int M, int N, int64_t K, int64_t chunk,
                                                      const double* __restrict__ A, int64_t a_ld,
                                                      const double* __restrict__ B, int64_t b_ld,
                                                      double* __restrict__ part) {
  constexpr int LDK = TK2 + 4;               // A stored [m][k] (AK)
  constexpr int LDA = MP + 4, LDB = NP + 4;  // A stored [k][m]; B stored [k][n]
  constexpr int ASZ = AK ? MP * LDK : TK2 * LDA, BSZ = TK2 * LDB;
  static_assert(!SYM || (MP == NP && !AK), "SYM: square, A m-fast");
  constexpr int MB = MP / 16, NB = NP / 8;
  // SYM: upper tiles = sum over m-blocks mb of (NB - 2 mb)
  constexpr int TILES = SYM ? MB * NB - MB * (MB - 1) : MB * NB;
  constexpr int PER_W = (TILES + TW - 1) / TW;
  auto tile_mn = [](int tile, int& m0, int& n0) {
    if (!SYM) {
      m0 = (tile / NB) * 16;
      n0 = (tile % NB) * 8;
      return;
    }
    int mb = 0;
#pragma unroll
    for (int q = 0; q < MB; q++) {
      const int cnt = NB - 2 * q;
      if (mb == q && tile >= cnt) { tile -= cnt; mb = q + 1; }
    }
    m0 = mb * 16;
    n0 = (2 * mb + tile) * 8;
  };
  extern __shared__ __align__(16) double tsm2[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  const int64_t kbeg = (int64_t)blockIdx.x * chunk;
  const int64_t kend = ks_min64(K, kbeg + chunk);
  const int nslab = (int)((kend - kbeg + TK2 - 1) / TK2);
  auto stage = [&](int sl, int buf) {
    double* As = tsm2 + buf * (ASZ + BSZ);
    double* Bs = As + ASZ;
    const int64_t k0 = kbeg + (int64_t)sl * TK2;
    (void)Bs;
    if (AK) {  // A(m, k) = A[m a_ld + k]: pairs along k
      for (int e = tid; e < MP * (TK2 / 2); e += TT) {
        const int mm = e / (TK2 / 2), kk = 2 * (e % (TK2 / 2));
        const int64_t gk = k0 + kk;
        const bool ok = gk < kend && mm < M;  // K-ranges end on even k (host: K even)
        cp16(&As[mm * LDK + kk], ok ? A + (int64_t)mm * a_ld + gk : A, ok);
      }
    } else {  // A(m, k) = A[k a_ld + m]: pairs along m
      for (int e = tid; e < TK2 * (MP / 2); e += TT) {
        const int kk = e / (MP / 2), mm = 2 * (e % (MP / 2));
        const int64_t gk = k0 + kk;
        const bool ok = gk < kend && mm < M;  // M even (host)
        cp16(&As[kk * LDA + mm], ok ? A + gk * a_ld + mm : A, ok);
      }
    }
    if (!SYM) for (int e = tid; e < TK2 * (NP / 2); e += TT) {  // B(k, n) = B[k b_ld + n]: pairs along n
      const int kk = e / (NP / 2), nn = 2 * (e % (NP / 2));
      const int64_t gk = k0 + kk;
      const bool ok = gk < kend && nn < N;  // N even (host)
      cp16(&Bs[kk * LDB + nn], ok ? B + gk * b_ld + nn : B, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[PER_W][4];
#pragma unroll
  for (int i = 0; i < PER_W; i++) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
  if (nslab > 0) stage(0, 0);
  for (int sl = 0; sl < nslab; sl++) {
    if (sl + 1 < nslab) {
      stage(sl + 1, (sl + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* As = tsm2 + (sl & 1) * (ASZ + BSZ);
    const double* Bs = SYM ? As : As + ASZ;  // SYM: LDA == LDB
#pragma unroll
    for (int i = 0; i < PER_W; i++) {
      const int tile = warp + i * TW;
      if (tile < TILES) {
        int m0, n0;
        tile_mn(tile, m0, n0);
#pragma unroll
        for (int kk = 0; kk < TK2; kk += 4) {
          const double a0 = AK ? As[(m0 + g) * LDK + kk + t4] : As[(kk + t4) * LDA + m0 + g];
          const double a1 = AK ? As[(m0 + g + 8) * LDK + kk + t4] : As[(kk + t4) * LDA + m0 + g + 8];
          const double b0 = Bs[(kk + t4) * LDB + n0 + g];
          dmma_16x8x4(acc[i], a0, a1, b0);
        }
      }
    }
    __syncthreads();  // the buffer is restaged two slabs later
  }
  double* out = part + (int64_t)blockIdx.x * M * N;
#pragma unroll
  for (int i = 0; i < PER_W; i++) {
    const int tile = warp + i * TW;
    if (tile < TILES) {
      int m0, n0;
      tile_mn(tile, m0, n0);
      const int r0 = m0 + g, c0 = n0 + 2 * t4;
      if (SYM) {  // each upper entry (r <= c) and its mirror, from the one accumulator that owns it
#pragma unroll
        for (int v = 0; v < 4; v++) {
          const int r = r0 + (v >> 1) * 8, c = c0 + (v & 1);
          if (r <= c && c < N) {
            out[r * N + c] = acc[i][v];
            out[c * N + r] = acc[i][v];
          }
        }
        continue;
      }
      if (r0 < M && c0 < N) out[r0 * N + c0] = acc[i][0];
      if (r0 < M && c0 + 1 < N) out[r0 * N + c0 + 1] = acc[i][1];
      if (r0 + 8 < M && c0 < N) out[(r0 + 8) * N + c0] = acc[i][2];
      if (r0 + 8 < M && c0 + 1 < N) out[(r0 + 8) * N + c0 + 1] = acc[i][3];
    }
  }
}

template <int MP, int NP, bool AK, bool SYM = false>
void launch_tall2(cudaStream_t st, int nparts, int M, int N, int64_t K, int64_t chunk, const double* A, int64_t a_ld,
                  const double* B, int64_t b_ld, double* part) {
  constexpr int ASZ = AK ? MP * (TK2 + 4) : TK2 * (MP + 4), BSZ = TK2 * (NP + 4);
  const size_t smem = sizeof(double) * 2 * (ASZ + BSZ);
  cudaFuncSetAttribute(tall_tn2_kernel<MP, NP, AK, SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tall_tn2_kernel<MP, NP, AK, SYM><<<nparts, TT, smem, st>>>(M, N, K, chunk, A, a_ld, B, b_ld, part);
}

template <int MP, int NP>
void launch_tall(cudaStream_t st, int nparts, int M, int N, int64_t K, int64_t chunk, const double* A, int64_t a_ks,
                 int64_t a_ms, const double* B, int64_t b_ks, int64_t b_ns, double* part) {
  const size_t smem = sizeof(double) * TK * ((MP + 4) + (NP + 4));
  cudaFuncSetAttribute(tall_tn_kernel<MP, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tall_tn_kernel<MP, NP><<<nparts, TT, smem, st>>>(M, N, K, chunk, A, a_ks, a_ms, B, b_ks, b_ns, part);
}

}  // namespace

namespace ks {

int gemm_tn_tall_dmma(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                      int64_t a_ks, int64_t a_ms, const double* B, int64_t b_ks, int64_t b_ns, double* C) {
  // the 16-byte / double-buffered kernel for aligned shapes: B n-fast, A k-fast or m-fast, even
  // M / N / K and leading dimensions, 16-byte aligned operands
  const bool akf = a_ks == 1, amf = a_ms == 1;
  const int64_t a_ld = akf ? a_ms : a_ks;
  const bool aligned = (((uintptr_t)A | (uintptr_t)B) & 15) == 0;
  if (!ks::env(ks::ENV_TALL_OLD) && aligned && b_ns == 1 && (b_ks & 1) == 0 && (akf || amf) && (a_ld & 1) == 0 &&
      (M & 1) == 0 && (N & 1) == 0 && (K & 1) == 0 && M <= 128 && N <= 128 && K >= 2 * TK2) {
    const int mp2 = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 80 ? 80 : 128;
    const int np2 = N <= 16 ? 16 : N <= 32 ? 32 : N <= 64 ? 64 : 128;
    const int64_t cap2 = num_sms();
    int64_t chunk2 = (K + cap2 - 1) / cap2;
    chunk2 = (chunk2 + TK2 - 1) / TK2 * TK2;
    const int64_t nparts2 = (K + chunk2 - 1) / chunk2;
    Scratch<double> part2(nparts2 * M * N, st);
    KS_REQUIRE(part2.p, KS_ECUDA, "scratch allocation failed");
    const int np2_i = (int)nparts2;
    bool done = false;
    // Gram A^T A (same operand, A m-fast, M = N in {16, 32, 64, 128}): the symmetric kernel
    if (!akf && A == B && a_ld == b_ks && M == N && M == mp2 && mp2 != 80 && !ks::env(ks::ENV_TALL_OLD)) {
      if (M == 16) launch_tall2<16, 16, false, true>(st, np2_i, (int)M, (int)N, K, chunk2, A, a_ld, B, b_ks, part2.p);
      if (M == 32) launch_tall2<32, 32, false, true>(st, np2_i, (int)M, (int)N, K, chunk2, A, a_ld, B, b_ks, part2.p);
      if (M == 64) launch_tall2<64, 64, false, true>(st, np2_i, (int)M, (int)N, K, chunk2, A, a_ld, B, b_ks, part2.p);
      if (M == 128) launch_tall2<128, 128, false, true>(st, np2_i, (int)M, (int)N, K, chunk2, A, a_ld, B, b_ks, part2.p);
      done = true;
    }
#define KS_TALL2(MM, NN)                                                                                         \
  if (!done && mp2 == MM && np2 == NN) {                                                                         \
    if (akf) launch_tall2<MM, NN, true>(st, np2_i, (int)M, (int)N, K, chunk2, A, a_ld, B, b_ks, part2.p);        \
    else launch_tall2<MM, NN, false>(st, np2_i, (int)M, (int)N, K, chunk2, A, a_ld, B, b_ks, part2.p);           \
    done = true;                                                                                                 \
  }
    KS_TALL2(16, 16) KS_TALL2(16, 32) KS_TALL2(16, 64) KS_TALL2(16, 128)
    KS_TALL2(32, 16) KS_TALL2(32, 32) KS_TALL2(32, 64) KS_TALL2(32, 128)
    KS_TALL2(64, 16) KS_TALL2(64, 32) KS_TALL2(64, 64) KS_TALL2(64, 128)
    KS_TALL2(80, 16) KS_TALL2(80, 32) KS_TALL2(80, 64) KS_TALL2(80, 128)
    KS_TALL2(128, 16) KS_TALL2(128, 32) KS_TALL2(128, 64) KS_TALL2(128, 128)
#undef KS_TALL2
    KS_CHECK_LAUNCH();
    const int64_t count2 = M * N;
    reduce_parts_warp_kernel<<<ceil_div_u(count2 * 32, 256), 256, 0, st>>>(part2.p, nparts2, count2, alpha, C);
    KS_CHECK_LAUNCH();
    return KS_OK;
  }
  const int mp = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : 128;
  const int np = N <= 16 ? 16 : N <= 32 ? 32 : N <= 64 ? 64 : 128;
  int64_t nparts = (K + 63) / 64;
  const int64_t cap = num_sms();
  if (nparts > cap) nparts = cap;
  int64_t chunk = (K + nparts - 1) / nparts;
  chunk = (chunk + TK - 1) / TK * TK;
  nparts = (K + chunk - 1) / chunk;
  Scratch<double> part(nparts * M * N, st);
  KS_REQUIRE(part.p, KS_ECUDA, "scratch allocation failed");
  const int np_i = (int)nparts;
#define KS_TALL(MM, NN)                                                                                  \
  if (mp == MM && np == NN)                                                                              \
    launch_tall<MM, NN>(st, np_i, (int)M, (int)N, K, chunk, A, a_ks, a_ms, B, b_ks, b_ns, part.p);
  KS_TALL(16, 16) KS_TALL(16, 32) KS_TALL(16, 64) KS_TALL(16, 128)
  KS_TALL(32, 16) KS_TALL(32, 32) KS_TALL(32, 64) KS_TALL(32, 128)
  KS_TALL(64, 16) KS_TALL(64, 32) KS_TALL(64, 64) KS_TALL(64, 128)
  KS_TALL(128, 16) KS_TALL(128, 32) KS_TALL(128, 64) KS_TALL(128, 128)
#undef KS_TALL
  KS_CHECK_LAUNCH();
  const int64_t count = M * N;
  reduce_parts_warp_kernel<<<ceil_div_u(count * 32, 256), 256, 0, st>>>(part.p, nparts, count, alpha, C);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

}  // namespace ks

// =============================================================================================
// Q (r x d) = scale * GA G^-1 for a symmetric positive definite Gram G (d x d), one CTA:
// right-looking Cholesky G = L L^T in shared memory, then forward / backward substitution of
// the r right-hand sides GA^T, all rows of a substitution step in parallel.  This is the
// (1 + eps/4) (g a_tilde) gram_tilde^-1 factor of the JL estimator (leverage.py:114-127).
// info[0] = k+1 if pivot k is not positive (caller falls back to LU).
// =============================================================================================
namespace {

constexpr int JP_CPW = 2;  // right-hand-side columns per warp and pass
constexpr int JP_COLS = 16 * JP_CPW;  // columns per CTA with 512 threads (factor + solve launches)

__device__ unsigned long long g_jlp_ts[4];  // globaltimer stamps of CTA 0 (debug)
__device__ __forceinline__ unsigned long long jlp_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define JLP_STAMP(k) \
  if (blockIdx.x == 0 && threadIdx.x == 0) g_jlp_ts[k] = jlp_now();

// mode 0: factor + solve; 1: factor only (L and 1/diag(L) to Lg, d*(d+1) + d doubles); 2: solve
// only with the factor from Lg (lets the factorization run before GA is ready).
__global__ void __launch_bounds__(512) jl_projection_kernel(const double* __restrict__ G, int d,
                                                            const double* __restrict__ GA, int r, double scale,
                                                            double* __restrict__ Q, int32_t* __restrict__ info,
                                                            double* __restrict__ Lg, int mode) {
  extern __shared__ double sm[];
  const int ld = d + 1;
  double* L = sm;                   // d x ld (lower triangle used)
  double* Y = sm + (size_t)d * ld;  // d x r  (right-hand sides, overwritten by the solution)
  __shared__ int s_bad;
  __shared__ double s_rdiag[64];
  JLP_STAMP(0)
  const int tid = threadIdx.x, nt = blockDim.x, tx = tid & 31, ty = tid >> 5, nty = nt >> 5;
  if (mode != 2) {
    for (int e = tid; e < d * d; e += nt) ks_cp_async8(&L[(e / d) * ld + (e % d)], G + e);
  } else {
    for (int e = tid; e < d * ld; e += nt) ks_cp_async8(&L[e], Lg + e);
    if (d <= 64)
      for (int e = tid; e < d; e += nt) ks_cp_async8(&s_rdiag[e], Lg + (size_t)d * ld + e);
  }
  if (mode == 2 && d <= 64) {  // this CTA's right-hand-side columns only
    const int cpc = nty * JP_CPW, c_lo = blockIdx.x * cpc, nc = min(r, c_lo + cpc) - c_lo;
    for (int e = tid; e < d * nc; e += nt) {
      const int c = c_lo + e / d, k = e % d;
      ks_cp_async8(&Y[k * r + c], GA + (size_t)c * d + k);
    }
  } else if (mode != 1) {
    for (int e = tid; e < d * r; e += nt) {
      const int k = e / r, c = e - k * r;
      ks_cp_async8(&Y[e], GA + (size_t)c * d + k);
    }
  }
  if (tid == 0) s_bad = 0;
  ks_cp_async_wait_all();
  __syncthreads();
  JLP_STAMP(1)
  if (mode == 2) {
    // factor already in shared memory
  } else if (d <= 64 && nt == 512) {
    // Register-resident right-looking LDL^T, one barrier per column: thread t owns column
    // j = t % 64, rows i = t / 64 + 8m (m < 8).  At step k the owners of column k publish it
    // (and the pivot owner 1 / d_k) in a double-buffered shared column; everyone then applies
    // the rank-1 update a_ij -= a_ik (a_jk / d_k) to its own entries.  Square roots are kept off
    // the serial chain: L = L_unit diag(sqrt(d)) is formed at the end, in parallel.
    __shared__ double colb[2][64];
    __shared__ double pivb[2];
    __shared__ double dg[64];
    const int j = tid & 63, i0 = tid >> 6;
    // (s_rdiag: reciprocals of the Cholesky diagonal for the substitutions below)
    double a[8];
#pragma unroll
    for (int m = 0; m < 8; m++) {
      const int i = i0 + 8 * m;
      a[m] = (i < d && j < d && j <= i) ? L[i * ld + j] : 0.0;
    }
    for (int k = 0; k < d; k++) {
      const int b = k & 1;
      if (j == k) {
#pragma unroll
        for (int m = 0; m < 8; m++) {
          const int i = i0 + 8 * m;
          if (i >= k && i < d) colb[b][i] = a[m];
          if (i == k) {
            const double p = a[m];
            if (!(p > 0.0) && !s_bad) s_bad = k + 1;
            pivb[b] = p > 0.0 ? 1.0 / p : 1.0;
            dg[k] = p;
          }
        }
      }
      __syncthreads();
      const double rd = pivb[b];
      if (j == k) {
#pragma unroll
        for (int m = 0; m < 8; m++) {
          const int i = i0 + 8 * m;
          if (i > k && i < d) a[m] *= rd;
        }
      } else if (j > k && j < d) {
        const double ljk = colb[b][j] * rd;
#pragma unroll
        for (int m = 0; m < 8; m++) {
          const int i = i0 + 8 * m;
          if (i >= j && i < d) a[m] = fma(-colb[b][i], ljk, a[m]);
        }
      }
    }
    __syncthreads();
    if (j < d) {
      const double dj = dg[j];
      const double sj = dj > 0.0 ? sqrt(dj) : 1.0;
      if (i0 == 0) s_rdiag[j] = 1.0 / sj;
#pragma unroll
      for (int m = 0; m < 8; m++) {
        const int i = i0 + 8 * m;
        if (i < d && j <= i) L[i * ld + j] = (i == j) ? sj : a[m] * sj;
      }
    }
    __syncthreads();
    JLP_STAMP(2)
  } else {
    // right-looking Cholesky, two barriers per column: every thread derives the pivot itself
    for (int k = 0; k < d; k++) {
      const double p = L[k * ld + k];
      const double lkk = p > 0.0 ? sqrt(p) : 1.0;
      for (int i = k + 1 + tid; i < d; i += nt) L[i * ld + k] /= lkk;
      __syncthreads();
      if (tid == 0) {
        if (!(p > 0.0) && !s_bad) s_bad = k + 1;
        L[k * ld + k] = lkk;
      }
      for (int i = k + 1 + ty; i < d; i += nty) {
        const double lik = L[i * ld + k];
        for (int jj = k + 1 + tx; jj <= i; jj += 32) L[i * ld + jj] = fma(-lik, L[jj * ld + k], L[i * ld + jj]);
      }
      __syncthreads();
    }
  }
  if (mode == 1) {
    if (d > 64 || nt != 512)
      for (int k = tid; k < d && k < 64; k += nt) s_rdiag[k] = 1.0 / L[k * ld + k];
    __syncthreads();
    for (int e = tid; e < d * ld; e += nt) Lg[e] = L[e];
    for (int e = tid; e < d && e < 64; e += nt) Lg[(size_t)d * ld + e] = s_rdiag[e];
    if (tid == 0 && blockIdx.x == 0) info[0] = s_bad;
    return;
  }
  // L Z = Y, then L^T X = Z.  Right-hand-side columns are independent: for d <= 64 a warp solves
  // JP_CPW columns at once with the column in registers (lane l owns rows l and l + 32); the
  // per-element operation order is the textbook one (divide by the pivot, then fma updates).
  if (d <= 64 && (nt == 512 || mode == 2)) {
    const int lane = tx, warp = ty;
    const int cpc = nty * JP_CPW;  // columns per CTA
    const int c_lo = blockIdx.x * cpc, c_hi = min(r, c_lo + cpc);
    for (int c0 = c_lo + warp; c0 < c_hi; c0 += nty * JP_CPW) {
      double y0[JP_CPW], y1[JP_CPW];
#pragma unroll
      for (int j = 0; j < JP_CPW; j++) {
        const int c = c0 + j * nty;
        y0[j] = (c < c_hi && lane < d) ? Y[lane * r + c] : 0.0;
        y1[j] = (c < c_hi && lane + 32 < d) ? Y[(lane + 32) * r + c] : 0.0;
      }
      for (int k = 0; k < d; k++) {
        const double rk = s_rdiag[k];
        const bool u0 = lane > k && lane < d, u1 = lane + 32 > k && lane + 32 < d;
        const double l0 = u0 ? L[lane * ld + k] : 0.0, l1 = u1 ? L[(lane + 32) * ld + k] : 0.0;
#pragma unroll
        for (int j = 0; j < JP_CPW; j++) {
          const double yk = __shfl_sync(0xffffffffu, k < 32 ? y0[j] : y1[j], k & 31) * rk;
          if (lane == (k & 31)) { if (k < 32) y0[j] = yk; else y1[j] = yk; }
          if (u0) y0[j] = fma(-l0, yk, y0[j]);
          if (u1) y1[j] = fma(-l1, yk, y1[j]);
        }
      }
      for (int k = d - 1; k >= 0; k--) {
        const double rk = s_rdiag[k];
        const bool u0 = lane < k, u1 = lane + 32 < k;
        const double l0 = u0 ? L[k * ld + lane] : 0.0, l1 = u1 ? L[k * ld + lane + 32] : 0.0;
#pragma unroll
        for (int j = 0; j < JP_CPW; j++) {
          const double yk = __shfl_sync(0xffffffffu, k < 32 ? y0[j] : y1[j], k & 31) * rk;
          if (lane == (k & 31)) { if (k < 32) y0[j] = yk; else y1[j] = yk; }
          if (u0) y0[j] = fma(-l0, yk, y0[j]);
          if (u1) y1[j] = fma(-l1, yk, y1[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < JP_CPW; j++) {
        const int c = c0 + j * nty;
        if (c < c_hi && lane < d) Q[(size_t)c * d + lane] = scale * y0[j];
        if (c < c_hi && lane + 32 < d) Q[(size_t)c * d + lane + 32] = scale * y1[j];
      }
    }
  } else if (blockIdx.x == 0) {
    for (int c = tid; c < r; c += nt) {
      for (int k = 0; k < d; k++) {
        const double yk = Y[k * r + c] / L[k * ld + k];
        Y[k * r + c] = yk;
        for (int i = k + 1; i < d; i++) Y[i * r + c] = fma(-L[i * ld + k], yk, Y[i * r + c]);
      }
      for (int k = d - 1; k >= 0; k--) {
        const double yk = Y[k * r + c] / L[k * ld + k];
        Y[k * r + c] = yk;
        for (int i = 0; i < k; i++) Y[i * r + c] = fma(-L[k * ld + i], yk, Y[i * r + c]);
      }
    }
    __syncthreads();
    for (int e = tid; e < r * d; e += nt) {
      const int c = e / d, k = e - c * d;
      Q[e] = scale * Y[k * r + c];
    }
  }
  if (tid == 0 && blockIdx.x == 0 && mode == 0) info[0] = s_bad;
  JLP_STAMP(3)
}

}  // namespace

extern "C" int ks_debug_jl_projection_stamps(uint64_t* out) {
  KS_TRY_CUDA(cudaMemcpyFromSymbol(out, g_jlp_ts, sizeof(unsigned long long) * 4));
  return KS_OK;
}

extern "C" int ks_jl_projection(const double* G, int32_t d, const double* GA, int32_t r, double scale, double* Q,
                                int32_t* info, void* stream) {
  const size_t smem = sizeof(double) * ((size_t)d * (d + 1) + (size_t)d * r);
  KS_REQUIRE(d >= 1 && r >= 1 && smem <= 220 * 1024, KS_ESIZE, "jl_projection: d=%d r=%d too large", d, r);
  KS_TRY_CUDA(cudaFuncSetAttribute(jl_projection_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  const unsigned grid = d <= 64 ? ceil_div_u(r, JP_COLS) : 1;
  jl_projection_kernel<<<grid, 512, smem, (cudaStream_t)stream>>>(G, d, GA, r, scale, Q, info, nullptr, 0);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_jl_cholesky(const double* G, int32_t d, double* Lws, int32_t* info, void* stream) {
  const size_t smem = sizeof(double) * ((size_t)d * (d + 1));
  KS_REQUIRE(d >= 1 && smem <= 220 * 1024, KS_ESIZE, "jl_cholesky: d=%d too large", d);
  KS_TRY_CUDA(cudaFuncSetAttribute(jl_projection_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  jl_projection_kernel<<<1, 512, smem, (cudaStream_t)stream>>>(G, d, nullptr, 0, 1.0, nullptr, info, Lws, 1);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_jl_solve(const double* Lws, int32_t d, const double* GA, int32_t r, double scale, double* Q,
                           void* stream) {
  const size_t smem = sizeof(double) * ((size_t)d * (d + 1) + (size_t)d * r);
  KS_REQUIRE(d >= 1 && r >= 1 && smem <= 220 * 1024, KS_ESIZE, "jl_solve: d=%d r=%d too large", d, r);
  KS_TRY_CUDA(cudaFuncSetAttribute(jl_projection_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  // solve only: 4 warps per CTA, JP_CPW columns per warp, ~r / 8 CTAs (the triangular solves are
  // sequential in d per column: spread the columns over SMs)
  const int nthr = d <= 64 ? 128 : 512;
  const unsigned grid = d <= 64 ? ceil_div_u(r, (nthr / 32) * JP_CPW) : 1;
  jl_projection_kernel<<<grid, nthr, smem, (cudaStream_t)stream>>>(nullptr, d, GA, r, scale, Q, nullptr, (double*)Lws,
                                                                    2);
  KS_CHECK_LAUNCH();
  return KS_OK;
}
