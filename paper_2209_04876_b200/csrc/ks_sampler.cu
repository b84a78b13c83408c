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
};

__device__ __forceinline__ int64_t block_incl_scan_i64(int64_t v, int64_t* wsum) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) wsum[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int64_t t = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    if (lane < nw) wsum[lane] = t;
  }
  __syncthreads();
  if (wid > 0) v += wsum[wid - 1];
  __syncthreads();
  return v;
}

__device__ __forceinline__ double ulp_of(double x) {
  int e;
  frexp(x, &e);  // x = m 2^e, m in [0.5, 1)
  return ldexp(1.0, e - 53);
}

__global__ void __launch_bounds__(ST_T) sampler_tables_kernel(TabArgs A) {
  __shared__ double slot[ST_T];
  __shared__ int8_t stopd[ST_T];
  __shared__ int64_t wsum[32];
  __shared__ double s_spec[ST_T];
  __shared__ int s_bad, s_first;
  const int f = blockIdx.x, tid = threadIdx.x;
  const double* __restrict__ scores = A.scores[f];
  const int64_t n = A.n[f];
  double* __restrict__ probs = A.probs[f];
  double* __restrict__ cdf = A.cdf[f];
  if (tid == 0) s_bad = 0;
  __syncthreads();
  {
    bool bad = false;
    for (int64_t i = tid; i < n; i += ST_T) {
      const double v = scores[i];
      bad |= !(v >= 0.0) || !isfinite(v);
    }
    if (__syncthreads_or(bad) && tid == 0) s_bad = 1;
  }
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
      auto get = [&](int64_t i) { return scores[i]; };
      slot[tid] = pw_sum_seq(get, s, len);
    }
  }
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
  for (int64_t i = tid; i < n; i += ST_T) probs[i] = scores[i] / total;
  __syncthreads();
  if (cdf == nullptr) return;
  // ---- exact cumsum by verified block speculation
  double prev = 0.0;
  int64_t pos = 0;
  while (pos < n) {
    const int64_t i = pos + tid;
    const bool valid = i < n;
    const double x = valid ? probs[i] : 0.0;
    double ref = prev;
    if (ref == 0.0) ref = probs[pos];
    const double u = (ref > 0.0) ? ulp_of(ref) : 0x1.0p-1074;
    long long qi = 0;
    if (valid) {
      const double qd = x / u;
      qi = (qd < 0x1.0p52) ? __double2ll_rn(qd) : (1ll << 52);
    }
    const int64_t Q = block_incl_scan_i64(qi, wsum);
    const double base = prev / u;
    const double spec = (double)((long long)base + Q) * u;
    s_spec[tid] = spec;
    if (tid == 0) s_first = ST_T;
    __syncthreads();
    const double sprev = (tid == 0) ? prev : s_spec[tid - 1];
    const double real = __dadd_rn(sprev, x);
    if (valid && real != spec) atomicMin(&s_first, tid);
    __syncthreads();
    const int fst = s_first;
    if (valid && tid < fst) cdf[i] = spec;
    if (valid && tid == fst) {
      cdf[i] = real;
      s_spec[tid] = real;
    }
    int64_t adv = (fst < ST_T) ? (int64_t)fst + 1 : (int64_t)ST_T;
    if (pos + adv > n) adv = n - pos;
    __syncthreads();
    prev = s_spec[adv - 1];
    pos += adv;
    __syncthreads();
  }
  if (A.renorm) {
    const double last = cdf[n - 1];
    __syncthreads();
    for (int64_t i = tid; i < n; i += ST_T) cdf[i] = cdf[i] / last;
  }
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
  sampler_tables_kernel<<<nf, ST_T, 0, (cudaStream_t)stream>>>(a);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_sampler_tables(const double* scores, int64_t n, int32_t renormalise, double* probs,
                                 double* cdf, int32_t* flags, void* stream) {
  double* cdfs[1] = {cdf};
  double* prb[1] = {probs};
  return ks_sampler_tables_batched(1, &scores, &n, renormalise, prb, cdf ? cdfs : nullptr, flags, stream);
}
