// ProductSampler tables on device (reference leverage.py:159-175), one CTA per factor:
//   total = scores.sum()   -- NumPy's pairwise summation order, bit-exact (subtrees summed by
//                             1024 threads, top of the recursion combined level by level)
//   probs = scores / total
//   cdf   = np.cumsum(probs) -- sequential fl-chain s_k = fl(s_{k-1} + p_k), bit-exact: a block
//                             speculates 1024 steps at once with exact integer arithmetic on the
//                             current binade's grid, then every lane verifies its step with the
//                             real IEEE addition; the first failing lane's verified value restarts
//                             the scan (failures happen only at binade crossings and ties).
#include "ks_common.cuh"
#include "ks_pairwise.cuh"

namespace {

constexpr int ST_T = 1024;
constexpr int ST_D = 10;  // 2^ST_D = ST_T subtrees
constexpr int MAXF = 8;

struct TabArgs {
  const double* scores[MAXF];
  int64_t n[MAXF];
  double* probs[MAXF];
  double* cdf[MAXF];
  int32_t* flags;
  int renorm;
  int cdf_only;  // probs (and flags) already formed by the multi-CTA path: only the cumsum runs
};

__device__ __forceinline__ double ulp_of(double x) {
  int e;
  frexp(x, &e);  // x = m 2^e, m in [0.5, 1)
  return ldexp(1.0, e - 53);
}

// Exact cumsum from position pos (prev = the exact value before it) by verified block speculation.
// Three block barriers per window: the per-window shared arrays are double-buffered (window
// parity), every warp forms the prefix of the warp totals itself, and the verified restart value is
// published beside the first failure's index, so nothing is re-synchronised at the end of a window.
struct CumsumSmem {
  int64_t c_wsum[2][ST_T / 32];
  double c_spec[2][ST_T], c_real[2][ST_T];
  int c_first[2];
};

__device__ void cumsum_windows(const double* __restrict__ probs, double* __restrict__ cdf, int64_t n, int64_t pos,
                               double prev, CumsumSmem& S) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int it = 0; pos < n; it++) {
    const int buf = it & 1;
    const int64_t i = pos + tid;
    const bool valid = i < n;
    const double x = valid ? probs[i] : 0.0;
    double ref = prev;
    if (ref == 0.0) ref = probs[pos];
    // u = ulp(ref) and 1/u as exact powers of two from the exponent bits (a division by u is a
    // multiplication by 1/u); tiny references keep the library path
    const long long eb = (__double_as_longlong(ref) >> 52) & 0x7ff;
    const bool fastu = ref > 0.0 && eb > 53 && eb < 2045;
    const double u = fastu ? __longlong_as_double((eb - 52) << 52) : (ref > 0.0 ? ulp_of(ref) : 0x1.0p-1074);
    const double iu = fastu ? __longlong_as_double((2098 - eb) << 52) : 0.0;
    long long qi = 0;
    if (valid) {
      const double qd = fastu ? x * iu : x / u;
      qi = (qd < 0x1.0p52) ? __double2ll_rn(qd) : (1ll << 52);
    }
    // inclusive block scan of qi: warp scan, warp totals published, each warp adds the prefix
    long long v = qi;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    if (lane == 31) S.c_wsum[buf][wid] = v;
    if (tid == 0) S.c_first[buf] = ST_T;
    __syncthreads();
    long long wt = lane < wid ? S.c_wsum[buf][lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wt += __shfl_xor_sync(0xffffffffu, wt, o);
    const long long Q = v + wt;
    const double base = fastu ? prev * iu : prev / u;
    const double spec = (double)((long long)base + Q) * u;
    S.c_spec[buf][tid] = spec;
    __syncthreads();
    const double sprev = (tid == 0) ? prev : S.c_spec[buf][tid - 1];
    const double real = __dadd_rn(sprev, x);
    if (valid && real != spec) {
      S.c_real[buf][tid] = real;
      atomicMin(&S.c_first[buf], tid);
    }
    __syncthreads();
    const int fst = S.c_first[buf];
    if (valid && tid < fst) cdf[i] = spec;
    if (valid && tid == fst) cdf[i] = real;
    int64_t adv = (fst < ST_T) ? (int64_t)fst + 1 : (int64_t)ST_T;
    if (pos + adv > n) adv = n - pos;
    prev = ((int)adv - 1 == fst) ? S.c_real[buf][fst] : S.c_spec[buf][adv - 1];
    pos += adv;
  }
}

__global__ void __launch_bounds__(ST_T) sampler_tables_kernel(TabArgs A) {
  __shared__ double slot[ST_T];
  __shared__ int8_t stopd[ST_T];
  __shared__ int s_bad;
  const int f = blockIdx.x, tid = threadIdx.x;
  const double* __restrict__ scores = A.scores[f];
  const int64_t n = A.n[f];
  double* __restrict__ probs = A.probs[f];
  double* __restrict__ cdf = A.cdf[f];
  if (!A.cdf_only) {  // (else probs and flags were formed by the multi-CTA path)
  if (tid == 0) s_bad = 0;
  // the nonnegative / finite check rides in the pairwise pass: every element is read there exactly
  // once by its subtree's owner (a separate strided pass would be one dependent L2 round trip per
  // 1024 elements on this single SM)
  bool bad = false;
  // ---- pairwise total: subtree of this thread at depth ST_D (or the leaf it falls into)
  {
    int64_t s = 0, len = n;
    int depth = 0;
    bool owner = true;
    for (; depth < ST_D; depth++) {
      if (len <= PW_BLOCK) {
        owner = (tid & ((1 << (ST_D - depth)) - 1)) == 0;
        break;
      }
      int64_t n2;
      pw_split(len, &n2);
      if ((tid >> (ST_D - 1 - depth)) & 1) {
        s += n2;
        len -= n2;
      } else {
        len = n2;
      }
    }
    stopd[tid] = owner ? (int8_t)depth : (int8_t)-1;
    if (owner) {
      auto get = [&](int64_t i) {
        const double v = scores[i];
        bad |= !(v >= 0.0) || !isfinite(v);
        return v;
      };
      slot[tid] = pw_sum_seq(get, s, len);
    }
  }
  if (__syncthreads_or(bad) && tid == 0) s_bad = 1;
  __syncthreads();
  // combine the top ST_D levels: node (l, i) is internal iff its left-most slot descended past l
  for (int l = ST_D - 1; l >= 0; l--) {
    if (tid < (1 << l)) {
      const int s0 = tid << (ST_D - l);
      if (stopd[s0] > l) slot[s0] = slot[s0] + slot[s0 + (1 << (ST_D - l - 1))];
    }
    __syncthreads();
  }
  const double total = slot[0];
  if (tid == 0) {
    int fl = s_bad ? 1 : 0;
    if (!(total > 0.0)) fl |= 2;
    A.flags[f] = fl;
  }
  {  // probs = scores / total, 8 loads in flight per thread (one SM streams the whole vector)
    constexpr int U = 8;
    for (int64_t i0 = tid; i0 < n; i0 += (int64_t)ST_T * U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t i = i0 + (int64_t)u * ST_T;
        v[u] = i < n ? scores[i] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t i = i0 + (int64_t)u * ST_T;
        if (i < n) probs[i] = v[u] / total;
      }
    }
  }
  }  // !cdf_only
  __syncthreads();
  if (cdf == nullptr) return;
  __shared__ CumsumSmem csm;
  cumsum_windows(probs, cdf, n, 0, 0.0, csm);
  __syncthreads();
  if (A.renorm) {
    const double last = cdf[n - 1];
    __syncthreads();
    for (int64_t i = tid; i < n; i += ST_T) cdf[i] = cdf[i] / last;
  }
}

// ---- multi-CTA total and probabilities (n >= TAB_MULTI_N): the same NumPy pairwise tree, its top
// TAB_KB levels over CTAs (leaf gl = CTA x 1024 + thread at depth TAB_KB + ST_D), so the sum is
// bit-identical to the one-CTA kernel's; then the elementwise division over every CTA and the
// exact cumsum by the one-CTA kernel (cdf_only).
constexpr int TAB_KB = 6, TAB_NB = 1 << TAB_KB, TAB_DT = TAB_KB + ST_D;
constexpr int64_t TAB_MULTI_N = 32768;

__global__ void __launch_bounds__(ST_T) tables_partial_kernel(TabArgs A, double* __restrict__ cpart,
                                                              int8_t* __restrict__ cstop, int* __restrict__ cbad) {
  __shared__ double slot[ST_T];
  __shared__ int8_t stopd[ST_T];
  const int f = blockIdx.y, c = blockIdx.x, tid = threadIdx.x;
  const double* __restrict__ scores = A.scores[f];
  const int64_t n = A.n[f];
  const int64_t gl = (int64_t)c * ST_T + tid;
  bool bad = false;
  {
    int64_t s = 0, len = n;
    int depth = 0;
    bool owner = true;
    for (; depth < TAB_DT; depth++) {
      if (len <= PW_BLOCK) {
        owner = (gl & ((1ll << (TAB_DT - depth)) - 1)) == 0;
        break;
      }
      int64_t n2;
      pw_split(len, &n2);
      if ((gl >> (TAB_DT - 1 - depth)) & 1) {
        s += n2;
        len -= n2;
      } else {
        len = n2;
      }
    }
    stopd[tid] = owner ? (int8_t)depth : (int8_t)-1;
    if (owner) {
      auto get = [&](int64_t i) {
        const double v = scores[i];
        bad |= !(v >= 0.0) || !isfinite(v);
        return v;
      };
      slot[tid] = pw_sum_seq(get, s, len);
    }
  }
  if (__syncthreads_or(bad) && tid == 0) atomicOr(&cbad[f], 1);
  // the CTA's part of the tree: global levels TAB_DT - 1 .. TAB_KB
  for (int l = ST_D - 1; l >= 0; l--) {
    if (tid < (1 << l)) {
      const int s0 = tid << (ST_D - l);
      if (stopd[s0] > l + TAB_KB) slot[s0] = slot[s0] + slot[s0 + (1 << (ST_D - l - 1))];
    }
    __syncthreads();
  }
  if (tid == 0) {
    cpart[f * TAB_NB + c] = stopd[0] >= 0 ? slot[0] : 0.0;
    cstop[f * TAB_NB + c] = stopd[0];
  }
}

__global__ void tables_total_kernel(TabArgs A, const double* __restrict__ cpart, const int8_t* __restrict__ cstop,
                                    const int* __restrict__ cbad, double* __restrict__ totals) {
  __shared__ double sl[TAB_NB];
  __shared__ int8_t sd[TAB_NB];
  const int f = blockIdx.x, tid = threadIdx.x;
  sl[tid] = cpart[f * TAB_NB + tid];
  sd[tid] = cstop[f * TAB_NB + tid];
  __syncthreads();
  for (int l = TAB_KB - 1; l >= 0; l--) {  // the top levels, same rule as inside a CTA
    if (tid < (1 << l)) {
      const int s0 = tid << (TAB_KB - l);
      if (sd[s0] > l) sl[s0] = sl[s0] + sl[s0 + (1 << (TAB_KB - l - 1))];
    }
    __syncthreads();
  }
  if (tid == 0) {
    const double total = sl[0];
    totals[f] = total;
    int fl = cbad[f] ? 1 : 0;
    if (!(total > 0.0)) fl |= 2;
    A.flags[f] = fl;
  }
}

__global__ void tables_probs_kernel(TabArgs A, const double* __restrict__ totals) {
  const int f = blockIdx.y;
  const int64_t n = A.n[f];
  const double total = totals[f];
  const double* __restrict__ scores = A.scores[f];
  double* __restrict__ probs = A.probs[f];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    probs[i] = scores[i] / total;
}

}  // namespace

extern "C" int ks_sampler_tables_batched(int32_t nf, const double* const* scores, const int64_t* n,
                                         int32_t renormalise, double* const* probs, double* const* cdf,
                                         int32_t* flags, void* stream) {
  KS_REQUIRE(nf >= 1 && nf <= MAXF, KS_EINVAL, "1..%d score vectors supported", MAXF);
  TabArgs a{};
  for (int f = 0; f < nf; f++) {
    KS_REQUIRE(n[f] >= 1, KS_EINVAL, "score vector %d must be nonempty", f);
    a.scores[f] = scores[f];
    a.n[f] = n[f];
    a.probs[f] = probs[f];
    a.cdf[f] = cdf ? cdf[f] : nullptr;
  }
  a.flags = flags;
  a.renorm = renormalise;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nmax = 0;
  for (int f = 0; f < nf; f++) nmax = n[f] > nmax ? n[f] : nmax;
  if (nmax >= TAB_MULTI_N && !ks::env(ks::ENV_TABLES_ONE_CTA)) {  // KS_TABLES_ONE_CTA: A/B
    // large vectors: the total and the probabilities over TAB_NB CTAs per vector, then the cumsum
    ks::Scratch<double> cpart((size_t)nf * TAB_NB, st), totals(nf, st);
    ks::Scratch<int8_t> cstop((size_t)nf * TAB_NB, st);
    ks::Scratch<int> cbad(nf, st);
    KS_REQUIRE(cpart.p && totals.p && cstop.p && cbad.p, KS_ECUDA, "scratch allocation failed");
    KS_TRY_CUDA(cudaMemsetAsync(cbad.p, 0, sizeof(int) * nf, st));
    tables_partial_kernel<<<dim3(TAB_NB, nf), ST_T, 0, st>>>(a, cpart.p, cstop.p, cbad.p);
    KS_CHECK_LAUNCH();
    tables_total_kernel<<<nf, TAB_NB, 0, st>>>(a, cpart.p, cstop.p, cbad.p, totals.p);
    KS_CHECK_LAUNCH();
    tables_probs_kernel<<<dim3(64, nf), 512, 0, st>>>(a, totals.p);
    KS_CHECK_LAUNCH();
    if (cdf) {
      a.cdf_only = 1;
      sampler_tables_kernel<<<nf, ST_T, 0, st>>>(a);
      KS_CHECK_LAUNCH();
    }
    return KS_OK;
  }
  sampler_tables_kernel<<<nf, ST_T, 0, st>>>(a);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_sampler_tables(const double* scores, int64_t n, int32_t renormalise, double* probs,
                                 double* cdf, int32_t* flags, void* stream) {
  double* cdfs[1] = {cdf};
  double* prb[1] = {probs};
  return ks_sampler_tables_batched(1, &scores, &n, renormalise, prb, cdf ? cdfs : nullptr, flags, stream);
}
