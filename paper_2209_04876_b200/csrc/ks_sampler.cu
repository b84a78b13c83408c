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
constexpr int TAB_TD = 8, TAB_T = 1 << TAB_TD;  // threads per CTA of the partial sums (registers for
                                               // the leaves' loads in flight)
constexpr int TAB_KB = 8, TAB_NB = 1 << TAB_KB, TAB_DT = TAB_KB + TAB_TD;
constexpr int64_t TAB_MULTI_N = 32768;  // below it the one-CTA kernel is as fast (its 1 launch vs 12)

__global__ void __launch_bounds__(TAB_T) tables_partial_kernel(TabArgs A, double* __restrict__ cpart,
                                                               int8_t* __restrict__ cstop, int* __restrict__ cbad) {
  __shared__ double slot[TAB_T];
  __shared__ int8_t stopd[TAB_T];
  const int f = blockIdx.y, c = blockIdx.x, tid = threadIdx.x;
  const double* __restrict__ scores = A.scores[f];
  const int64_t n = A.n[f];
  const int64_t gl = (int64_t)c * TAB_T + tid;
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
  for (int l = TAB_TD - 1; l >= 0; l--) {
    if (tid < (1 << l)) {
      const int s0 = tid << (TAB_TD - l);
      if (stopd[s0] > l + TAB_KB) slot[s0] = slot[s0] + slot[s0 + (1 << (TAB_TD - l - 1))];
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

// ---- multi-CTA exact cumsum (n >= TAB_MULTI_N, n <= ST_T * ST_T): cdf = np.cumsum(probs) is the
// chain s_k = fl(s_{k-1} + p_k).  While the running sum stays in one binade [2^e, 2^(e+1)) every step
// adds p_k rounded to that binade's grid u (a step with p_k / u exactly half-way rounds to even on the
// running sum's last bit: such a step starts a segment of its own), so inside a segment
// s_k = s_start + u (q_j + ... + q_k), q_j = rint(p_j / u): exact integer prefix sums, one element per
// thread over all CTAs.  Binades are guessed from an approximate (any-order) prefix; each segment's
// first value is formed exactly from the previous segment's end in a short sequential pass over the
// segments; then EVERY step is verified against the real IEEE addition, and from the first mismatch
// (a tie's round-half-even, a misjudged binade) the one-CTA window path takes over -- the result is
// the exact sequential cumsum in every case.
constexpr int CS_SEGMAX = 4096;  // segments per vector at most (else the window path from the start)
__device__ long long g_cs_dbg[16];  // profiling aid: first failed step and segment count per vector

struct CsArgs {
  double* ctot;       // nf x NB: CTA sums of p (approximate prefix)
  double* coff;       // nf x (NB + 1): exclusive CTA offsets
  long long* cq;      // nf x NB: CTA segmented tails
  int* cb;            // nf x NB: CTA has a boundary
  int* ccnt;          // nf x NB: boundaries in the CTA
  long long* carry;   // nf x NB: q sum since the last boundary before the CTA
  int* cseg0;         // nf x NB: segment id of the CTA's first boundary
  int* nseg;          // nf
  long long* qg;      // nf x n: segmented prefix Q of every element
  int* sid;           // nf x n: segment id of every element
  int64_t* sk0;       // nf x SEGMAX: segment starts
  int* se;            // nf x SEGMAX: binades
  long long* sq0;     // nf x SEGMAX: q at the start
  long long* sqend;   // nf x SEGMAX: Q at the last element
  double* sbase;      // nf x SEGMAX: exact first values
  unsigned long long* fail;  // nf: first failed step
  int nb;             // CTAs per vector
  int64_t nmax;
};

__device__ __forceinline__ int cs_binade(double a) {  // biased exponent of a > 0 (normal), -1 otherwise
  const int eb = (int)((__double_as_longlong(a) >> 52) & 0x7ff);
  return (a > 0.0 && eb >= 54 && eb < 2045) ? eb : -1;
}
__device__ __forceinline__ long long cs_q(double p, int eb) {  // rint(p / u), exact power-of-two scaling
  return eb < 0 ? 0 : __double2ll_rn(p * __longlong_as_double((long long)(2098 - eb) << 52));
}
__device__ __forceinline__ double cs_u(int eb) { return eb < 0 ? 0.0 : __longlong_as_double((long long)(eb - 52) << 52); }

// block inclusive scan of a double (any order), returns the block total in *tot
__device__ __forceinline__ double cs_scan_d(double v, double* sm, double* tot) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) sm[wid] = v;
  __syncthreads();
  double w = 0.0, all = 0.0;
  for (int i = 0; i < ST_T / 32; i++) {
    if (i < wid) w += sm[i];
    all += sm[i];
  }
  *tot = all;
  __syncthreads();
  return v + w;
}

// the element view every pass shares: p, approximate prefix, binade, boundary, q
struct CsElem {
  double p;
  int e;
  bool bnd;
  long long q;
};
__device__ __forceinline__ CsElem cs_elem(const double* __restrict__ probs, int64_t n, int64_t k, double coff_c,
                                          double coff_next, bool has_next, double* sm) {
  const int tid = threadIdx.x;
  CsElem r;
  r.p = k < n ? probs[k] : 0.0;
  double tot;
  const double incl = cs_scan_d(r.p, sm, &tot);
  // the CTA's last element takes the next CTA's offset as its prefix, so both CTAs judge the binade
  // of that element from the same value
  const double a = (tid == ST_T - 1 && has_next) ? coff_next : coff_c + incl;
  r.e = cs_binade(a);
  __shared__ int se_prev[ST_T];
  se_prev[tid] = r.e;
  __syncthreads();
  const int ep = tid > 0 ? se_prev[tid - 1] : (k > 0 ? cs_binade(coff_c) : -2);
  __syncthreads();
  // a step whose p / u is exactly half-way between grid points rounds to even on the RUNNING sum's
  // last bit: it starts a segment of its own (its value is formed exactly in the sequential pass)
  bool tie = false;
  if (r.e >= 0 && k < n) {
    const double fq = r.p * __longlong_as_double((long long)(2098 - r.e) << 52);
    tie = fq - floor(fq) == 0.5;
  }
  r.bnd = k < n && (k == 0 || r.e != ep || tie);
  r.q = k < n ? cs_q(r.p, r.e) : 0;
  return r;
}

// block segmented inclusive scan of (flag, value): (f1, v1) + (f2, v2) = (f1 | f2, f2 ? v2 : v1 + v2)
__device__ __forceinline__ void cs_segscan(int& fl, long long& v, int* smf, long long* smv) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int f2 = __shfl_up_sync(0xffffffffu, fl, o);
    const long long v2 = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) {
      v = fl ? v : v2 + v;
      fl |= f2;
    }
  }
  if (lane == 31) {
    smf[wid] = fl;
    smv[wid] = v;
  }
  __syncthreads();
  int pf = 0;
  long long pv = 0;
  for (int i = 0; i < wid; i++) {
    pv = smf[i] ? smv[i] : pv + smv[i];
    pf |= smf[i];
  }
  v = fl ? v : pv + v;
  fl |= pf;
  __syncthreads();
}

__global__ void __launch_bounds__(ST_T) cs_sum_kernel(TabArgs A, CsArgs C) {
  __shared__ double sm[ST_T / 32];
  const int f = blockIdx.y, c = blockIdx.x;
  const int64_t n = A.n[f], k = (int64_t)c * ST_T + threadIdx.x;
  const double p = k < n ? A.probs[f][k] : 0.0;
  double tot;
  cs_scan_d(p, sm, &tot);
  if (threadIdx.x == 0) C.ctot[f * C.nb + c] = tot;
}

__global__ void __launch_bounds__(ST_T) cs_offsets_kernel(TabArgs A, CsArgs C) {
  __shared__ double sm[ST_T / 32];
  const int f = blockIdx.x, c = threadIdx.x;
  const double v = c < C.nb ? C.ctot[f * C.nb + c] : 0.0;
  double tot;
  const double incl = cs_scan_d(v, sm, &tot);
  if (c < C.nb) C.coff[f * (C.nb + 1) + c] = incl - v;
  if (c == C.nb - 1) C.coff[f * (C.nb + 1) + C.nb] = incl;
}

__global__ void __launch_bounds__(ST_T) cs_local_kernel(TabArgs A, CsArgs C) {
  __shared__ double sm[ST_T / 32];
  __shared__ int smf[ST_T / 32];
  __shared__ long long smv[ST_T / 32];
  const int f = blockIdx.y, c = blockIdx.x, tid = threadIdx.x;
  const int64_t n = A.n[f], k = (int64_t)c * ST_T + tid;
  const double* co = C.coff + f * (C.nb + 1);
  const CsElem el = cs_elem(A.probs[f], n, k, co[c], co[c + 1], c + 1 < C.nb, sm);
  int fl = el.bnd;
  long long v = el.q;
  cs_segscan(fl, v, smf, smv);
  const int cnt = __syncthreads_count(el.bnd);
  if (tid == ST_T - 1) {
    C.cb[f * C.nb + c] = fl;
    C.cq[f * C.nb + c] = v;
    C.ccnt[f * C.nb + c] = cnt;
  }
}

__global__ void __launch_bounds__(ST_T) cs_carry_kernel(TabArgs A, CsArgs C) {
  __shared__ int smf[ST_T / 32];
  __shared__ long long smv[ST_T / 32];
  __shared__ double smd[ST_T / 32];
  const int f = blockIdx.x, c = threadIdx.x;
  const bool in = c < C.nb;
  int fl = in ? C.cb[f * C.nb + c] : 0;
  long long v = in ? C.cq[f * C.nb + c] : 0;
  cs_segscan(fl, v, smf, smv);
  // exclusive: the inclusive value of the CTA before
  __shared__ long long sv[ST_T];
  sv[c] = v;
  __syncthreads();
  const long long excl = c > 0 ? sv[c - 1] : 0;
  // boundary counts: exclusive scan (as doubles: exact below 2^53)
  double tot;
  const double cnt = in ? (double)C.ccnt[f * C.nb + c] : 0.0;
  const double incl = cs_scan_d(cnt, smd, &tot);
  if (in) {
    C.carry[f * C.nb + c] = excl;
    C.cseg0[f * C.nb + c] = (int)(incl - cnt);
  }
  if (c == 0) C.nseg[f] = (int)tot;
}

__global__ void __launch_bounds__(ST_T) cs_segments_kernel(TabArgs A, CsArgs C) {
  __shared__ double sm[ST_T / 32];
  __shared__ int smf[ST_T / 32];
  __shared__ long long smv[ST_T / 32];
  __shared__ long long sQ[ST_T];
  const int f = blockIdx.y, c = blockIdx.x, tid = threadIdx.x;
  const int64_t n = A.n[f], k = (int64_t)c * ST_T + tid;
  if (C.nseg[f] > CS_SEGMAX) return;
  const double* co = C.coff + f * (C.nb + 1);
  const CsElem el = cs_elem(A.probs[f], n, k, co[c], co[c + 1], c + 1 < C.nb, sm);
  int fl = el.bnd;
  long long v = el.q;
  cs_segscan(fl, v, smf, smv);
  const long long Qg = fl ? v : C.carry[f * C.nb + c] + v;  // the segmented prefix over all CTAs
  // segment id: the CTA's first id + boundaries up to this element - 1
  int bi = el.bnd;
  {
    double tot;
    const double incl = cs_scan_d((double)bi, sm, &tot);
    bi = (int)incl;
  }
  const int j = C.cseg0[f * C.nb + c] + bi - 1;  // (j = first id - 1 before the CTA's first boundary)
  sQ[tid] = Qg;
  __syncthreads();
  if (k < n) {
    C.qg[f * C.nmax + k] = Qg;
    C.sid[f * C.nmax + k] = j;
    if (el.bnd) {
      const int64_t b0 = (int64_t)f * CS_SEGMAX;
      C.sk0[b0 + j] = k;
      C.se[b0 + j] = el.e;
      C.sq0[b0 + j] = el.q;
      if (j > 0) C.sqend[b0 + j - 1] = tid > 0 ? sQ[tid - 1] : C.carry[f * C.nb + c];
    }
    if (k == n - 1) C.sqend[(int64_t)f * CS_SEGMAX + j] = Qg;
  }
}

constexpr int CS_BT = 256;
__global__ void __launch_bounds__(CS_BT) cs_bases_kernel(TabArgs A, CsArgs C) {
  // the segment records staged in shared memory by every thread (chunks of CS_BT), then the
  // sequential pass over them by one thread
  __shared__ double sp0[CS_BT], sdq[CS_BT];
  __shared__ double s_end;
  const int f = blockIdx.x, tid = threadIdx.x;
  const int ns = C.nseg[f];
  if (ns > CS_SEGMAX) {
    if (tid == 0) C.fail[f] = 0;  // too many segments: the window path from the start
    return;
  }
  const int64_t b0 = (int64_t)f * CS_SEGMAX;
  if (tid == 0) s_end = 0.0;
  for (int j0 = 0; j0 < ns; j0 += CS_BT) {
    const int j = j0 + tid;
    __syncthreads();
    if (j < ns) {
      sp0[tid] = A.probs[f][C.sk0[b0 + j]];
      sdq[tid] = (double)(C.sqend[b0 + j] - C.sq0[b0 + j]) * cs_u(C.se[b0 + j]);
    }
    __syncthreads();
    if (tid == 0) {
      double end = s_end;
      const int m = min(CS_BT, ns - j0);
      for (int i = 0; i < m; i++) {
        const double base = __dadd_rn(end, sp0[i]);
        C.sbase[b0 + j0 + i] = base;
        end = base + sdq[i];
      }
      s_end = end;
    }
  }
  if (tid == 0) C.fail[f] = (unsigned long long)A.n[f];
}

__device__ __forceinline__ double cs_value(const CsArgs& C, int f, int64_t k) {
  const int64_t b0 = (int64_t)f * CS_SEGMAX;
  const int j = C.sid[f * C.nmax + k];
  return C.sbase[b0 + j] + (double)(C.qg[f * C.nmax + k] - C.sq0[b0 + j]) * cs_u(C.se[b0 + j]);
}

__global__ void __launch_bounds__(ST_T) cs_values_kernel(TabArgs A, CsArgs C) {
  const int f = blockIdx.y;
  const int64_t n = A.n[f], k = (int64_t)blockIdx.x * ST_T + threadIdx.x;
  if (k >= n || C.nseg[f] > CS_SEGMAX) return;
  const double s = cs_value(C, f, k);
  const double prev = k > 0 ? cs_value(C, f, k - 1) : 0.0;
  A.cdf[f][k] = s;
  if (__dadd_rn(prev, A.probs[f][k]) != s) atomicMin(&C.fail[f], (unsigned long long)k);
}

// the verified prefix is final; from the first failed step on, the one-CTA window path
__global__ void __launch_bounds__(ST_T) cs_finish_kernel(TabArgs A, CsArgs C) {
  __shared__ CumsumSmem csm;
  const int f = blockIdx.x;
  const int64_t n = A.n[f];
  const int64_t k1 = (int64_t)C.fail[f];
  if (threadIdx.x == 0 && f < 8) {
    g_cs_dbg[2 * f] = k1;
    g_cs_dbg[2 * f + 1] = C.nseg[f];
  }
  if (k1 < n) cumsum_windows(A.probs[f], A.cdf[f], n, k1, k1 > 0 ? A.cdf[f][k1 - 1] : 0.0, csm);
}

// cdf /= cdf[n - 1] over every CTA (np.cumsum(p) / its last entry, as in the one-CTA kernel)
__global__ void cs_renorm_kernel(TabArgs A) {
  const int f = blockIdx.y;
  const int64_t n = A.n[f];
  double* cdf = A.cdf[f];
  const double last = cdf[n - 1];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (i != n - 1) cdf[i] = cdf[i] / last;
  // the last entry (read by every CTA) is divided by a second launch's single thread
}

__global__ void cs_renorm_last_kernel(TabArgs A) {
  const int f = blockIdx.x;
  double* cdf = A.cdf[f];
  const int64_t n = A.n[f];
  cdf[n - 1] = cdf[n - 1] / cdf[n - 1];
}

}  // namespace

// Profiling aid: the multi-CTA cumsum's first failed step and segment count of vector f (last call)
extern "C" int ks_debug_cumsum_stats(int32_t f, int64_t* out2) {
  if (f < 0 || f >= 8) return KS_EINVAL;
  long long h[16];
  KS_TRY_CUDA(cudaMemcpyFromSymbol(h, g_cs_dbg, sizeof(h)));
  out2[0] = h[2 * f];
  out2[1] = h[2 * f + 1];
  return KS_OK;
}

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
    tables_partial_kernel<<<dim3(TAB_NB, nf), TAB_T, 0, st>>>(a, cpart.p, cstop.p, cbad.p);
    KS_CHECK_LAUNCH();
    tables_total_kernel<<<nf, TAB_NB, 0, st>>>(a, cpart.p, cstop.p, cbad.p, totals.p);
    KS_CHECK_LAUNCH();
    tables_probs_kernel<<<dim3(64, nf), 512, 0, st>>>(a, totals.p);
    KS_CHECK_LAUNCH();
    if (cdf && nmax <= (int64_t)ST_T * ST_T && !ks::env(ks::ENV_TABLES_ONE_CTA)) {
      // the multi-CTA exact cumsum (segments of one binade, every step verified)
      const int nb = (int)((nmax + ST_T - 1) / ST_T);
      ks::Scratch<double> ctot((size_t)nf * nb, st), coff((size_t)nf * (nb + 1), st), sbase((size_t)nf * CS_SEGMAX, st);
      ks::Scratch<long long> cq((size_t)nf * nb, st), carry((size_t)nf * nb, st), qg((size_t)nf * nmax, st),
          sq0((size_t)nf * CS_SEGMAX, st), sqend((size_t)nf * CS_SEGMAX, st);
      ks::Scratch<int> cb((size_t)nf * nb, st), ccnt((size_t)nf * nb, st), cseg0((size_t)nf * nb, st), nseg(nf, st),
          sid((size_t)nf * nmax, st), se((size_t)nf * CS_SEGMAX, st);
      ks::Scratch<int64_t> sk0((size_t)nf * CS_SEGMAX, st);
      ks::Scratch<unsigned long long> fail(nf, st);
      KS_REQUIRE(ctot.p && coff.p && sbase.p && cq.p && carry.p && qg.p && sq0.p && sqend.p && cb.p && ccnt.p &&
                     cseg0.p && nseg.p && sid.p && se.p && sk0.p && fail.p,
                 KS_ECUDA, "scratch allocation failed");
      CsArgs c{ctot.p, coff.p, cq.p, cb.p, ccnt.p, carry.p, cseg0.p, nseg.p, qg.p, sid.p, sk0.p, se.p, sq0.p,
               sqend.p, sbase.p, fail.p, nb, nmax};
      cs_sum_kernel<<<dim3(nb, nf), ST_T, 0, st>>>(a, c);
      KS_CHECK_LAUNCH();
      cs_offsets_kernel<<<nf, ST_T, 0, st>>>(a, c);
      KS_CHECK_LAUNCH();
      cs_local_kernel<<<dim3(nb, nf), ST_T, 0, st>>>(a, c);
      KS_CHECK_LAUNCH();
      cs_carry_kernel<<<nf, ST_T, 0, st>>>(a, c);
      KS_CHECK_LAUNCH();
      cs_segments_kernel<<<dim3(nb, nf), ST_T, 0, st>>>(a, c);
      KS_CHECK_LAUNCH();
      cs_bases_kernel<<<nf, CS_BT, 0, st>>>(a, c);
      KS_CHECK_LAUNCH();
      cs_values_kernel<<<dim3(nb, nf), ST_T, 0, st>>>(a, c);
      KS_CHECK_LAUNCH();
      cs_finish_kernel<<<nf, ST_T, 0, st>>>(a, c);
      KS_CHECK_LAUNCH();
      if (renormalise) {
        cs_renorm_kernel<<<dim3(64, nf), 512, 0, st>>>(a);
        KS_CHECK_LAUNCH();
        cs_renorm_last_kernel<<<nf, 1, 0, st>>>(a);
        KS_CHECK_LAUNCH();
      }
    } else if (cdf) {
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
