// NumPy-exact random streams on the GPU.
//
// The reference draws every random number from numpy.random.Generator(PCG64) seeded through
// SeedSequence.spawn (solvers.py:415-416, leverage.py:124-126, :196-198, :217).  For bit-exact
// parity the GPU reproduces those streams instead of shipping host-generated arrays:
//   * PCG64 (XSL-RR 128/64, NumPy's default bit generator): the LCG is advanced in O(log n)
//     (Brown's jump-ahead), so every thread starts at its own offset of the stream.
//   * Generator.random(): (raw >> 11) * 2^-53.
//   * Generator.standard_normal(): NumPy's 256-layer ziggurat (Marsaglia-Tsang/Doornik).  Each
//     normal consumes a data-dependent number of raw draws (1 in ~99% of cases), so draw i's
//     start position is resolved in parallel: every position computes "value, consumption if
//     a normal started here"; 128-position chunks record their exit offset for each possible
//     entry offset (walks from different entries merge after a step or two); a one-block scan
//     composes the chunk maps; a final pass emits the chain values.  The ziggurat tables
//     (ki/wi/fi) are read from the installed NumPy's libnpyrandom.a by the host and passed in.
#include "ks_common.cuh"

typedef unsigned __int128 u128;

namespace {

__host__ __device__ constexpr u128 mk128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

// PCG_DEFAULT_MULTIPLIER_128 of the PCG family (O'Neill 2014), used by numpy.random.PCG64.
constexpr u128 PCG_MULT = mk128(0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL);

__device__ __forceinline__ uint64_t pcg_output(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(hi >> 58);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = PCG_MULT, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ double to_unit(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }

constexpr int RAW_PER_THREAD = 16;

// raw[p] = p-th 64-bit output after `skip` draws (output of the state after p+skip+1 steps)
__global__ void pcg_raw_kernel(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il, uint64_t skip,
                               int64_t count, uint64_t* __restrict__ raw) {
  const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * RAW_PER_THREAD;
  if (p0 >= count) return;
  const u128 inc = mk128(ih, il);
  u128 s = pcg_advance(mk128(sh, sl), inc, skip + (uint64_t)p0 + 1);
  const int n = (int)ks_min64(RAW_PER_THREAD, count - p0);
  for (int k = 0; k < n; k++) {
    raw[p0 + k] = pcg_output(s);
    s = s * PCG_MULT + inc;
  }
}

__global__ void pcg_uniform_kernel(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il,
                                   uint64_t skip, int64_t count, double* __restrict__ out) {
  const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * RAW_PER_THREAD;
  if (p0 >= count) return;
  const u128 inc = mk128(ih, il);
  u128 s = pcg_advance(mk128(sh, sl), inc, skip + (uint64_t)p0 + 1);
  const int n = (int)ks_min64(RAW_PER_THREAD, count - p0);
  for (int k = 0; k < n; k++) {
    out[p0 + k] = to_unit(pcg_output(s));
    s = s * PCG_MULT + inc;
  }
}

// ziggurat constants of NumPy's standard normal (r and 1/r of the 256-layer table)
constexpr double ZIG_R = 3.6541528853610087963519472518;
constexpr double ZIG_INV_R = 0.27366123732975827203338247596;

struct ZigTables {
  const uint64_t* ki;
  const double* wi;
  const double* fi;
};

// Value and raw-draw consumption of a normal whose first draw is raw[p]; -1 if the draw would
// read past `limit`.  Mirrors NumPy's random_standard_normal; IEEE ops without contraction.
__device__ int zig_eval(const uint64_t* __restrict__ raw, int64_t p, int64_t limit,
                        const ZigTables& T, double* out) {
  int64_t q = p;
  for (;;) {
    if (q >= limit) return -1;
    uint64_t r = raw[q++];
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = __dmul_rn((double)rabs, T.wi[idx]);
    if (sign) x = -x;
    if (rabs < T.ki[idx]) {
      *out = x;
      return (int)(q - p);
    }
    if (idx == 0) {
      for (;;) {
        if (q + 1 >= limit) return -1;
        const double u1 = to_unit(raw[q++]);
        const double u2 = to_unit(raw[q++]);
        const double xx = __dmul_rn(-ZIG_INV_R, log1p(-u1));
        const double yy = -log1p(-u2);
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          const double v = __dadd_rn(ZIG_R, xx);
          *out = ((rabs >> 8) & 1) ? -v : v;
          return (int)(q - p);
        }
      }
    } else {
      if (q >= limit) return -1;
      const double u = to_unit(raw[q++]);
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(T.fi[idx - 1], T.fi[idx]), u), T.fi[idx]);
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
        *out = x;
        return (int)(q - p);
      }
    }
  }
}

__global__ void zig_eval_kernel(const uint64_t* __restrict__ raw, int64_t M, int64_t limit,
                                const uint64_t* __restrict__ ki, const double* __restrict__ wi,
                                const double* __restrict__ fi, double* __restrict__ val,
                                int16_t* __restrict__ cons) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= M) return;
  ZigTables T{ki, wi, fi};
  double v = 0.0;
  const int c = zig_eval(raw, p, limit, T, &v);
  val[p] = v;
  cons[p] = (int16_t)(c > 32000 ? -1 : c);
}

constexpr int ZL = 128;  // chunk length (positions)
constexpr int ZK = 16;   // entry offsets tracked per chunk
constexpr int ZCB = 32;  // chunks per block of the chunk / emit kernels
constexpr int ZS = 32;   // chunks per super-chunk (ZCB % ZS == 0)
constexpr int ZT = 256;  // threads of the compose / emit kernels
constexpr int ZCT = 4;   // threads per chunk in the chunk kernel (ZK / ZCT offsets each)

// Stage the consumption table of positions [blk_beg, blk_beg + ZCB*ZL) into shared memory with
// 16-byte asynchronous copies (all in flight at once); positions >= M read as 1.
__device__ __forceinline__ void zig_stage_cons(int16_t* sc, const int16_t* __restrict__ cons, int64_t M,
                                               int64_t blk_beg) {
  constexpr int V = 8;  // int16 per 16-byte copy
  for (int i = threadIdx.x; i < ZCB * ZL / V; i += blockDim.x) {
    const int64_t p = blk_beg + (int64_t)i * V;
    if (p + V <= M) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(sc + i * V);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(cons + p) : "memory");
    } else {
      for (int v = 0; v < V; v++) sc[i * V + v] = (p + v < M) ? cons[p + v] : (int16_t)1;
    }
  }
  ks_cp_async_wait_all();
  __syncthreads();
}

// For each chunk and entry offset o < ZK: exit offset into the next chunk and normals emitted.
__global__ void __launch_bounds__(ZCB * ZCT) zig_chunk_kernel(const int16_t* __restrict__ cons, int64_t M,
                                                       int64_t nchunks, uint8_t* __restrict__ exit_off,
                                                       int32_t* __restrict__ cnt, int32_t* __restrict__ err) {
  __shared__ __align__(16) int16_t sc[ZCB * ZL];
  const int64_t blk_beg = (int64_t)blockIdx.x * ZCB * ZL;
  zig_stage_cons(sc, cons, M, blk_beg);
  // ZCT threads per chunk, ZK / ZCT entry offsets each (each walks offset 0 for the merge mask)
  const int lc = threadIdx.x / ZCT, part = threadIdx.x % ZCT;
  const int64_t c = (int64_t)blockIdx.x * ZCB + lc;
  if (lc >= ZCB || c >= nchunks) return;
  const int beg = lc * ZL;
  const int end = (int)ks_min64(M - blk_beg, beg + ZL);
  uint64_t m0 = 0, m1 = 0;
  int q = beg, c0 = 0;
  while (q < end) {
    const int k = sc[q];
    if (k <= 0) { atomicOr(err, 1); return; }
    const int rel = q - beg;
    if (rel < 64) m0 |= 1ull << rel; else m1 |= 1ull << (rel - 64);
    c0++;
    q += k;
  }
  const int e0 = q - end;
  if (e0 >= ZK) { atomicOr(err, 2); return; }
  for (int o = part * (ZK / ZCT); o < (part + 1) * (ZK / ZCT); o++) {
    int qq = beg + o, steps = 0;
    for (;;) {
      if (qq >= end) break;
      const int rel = qq - beg;
      const bool on0 = rel < 64 ? ((m0 >> rel) & 1) : ((m1 >> (rel - 64)) & 1);
      if (on0) break;
      const int k = sc[qq];
      if (k <= 0) { atomicOr(err, 1); return; }
      steps++;
      qq += k;
    }
    if (qq >= end) {
      const int e = qq - end;
      if (e >= ZK) { atomicOr(err, 2); return; }
      exit_off[c * ZK + o] = (uint8_t)e;
      cnt[c * ZK + o] = steps;
    } else {
      // merged with the offset-0 walk at qq: remaining count = walk-0 positions >= qq
      const int rel = qq - beg;
      const int before = rel >= 64 ? __popcll(m0) + __popcll(m1 & ((1ull << (rel - 64)) - 1))
                                   : __popcll(m0 & ((1ull << rel) - 1));
      exit_off[c * ZK + o] = (uint8_t)e0;
      cnt[c * ZK + o] = steps + (c0 - before);
    }
  }
}

// Compose the maps of ZS consecutive chunks into one super-chunk map.  One block covers
// ZT / ZK super-chunks; their chunk maps are staged in shared memory first.
__global__ void __launch_bounds__(ZT) zig_compose_kernel(const uint8_t* __restrict__ exit_off,
                                                         const int32_t* __restrict__ cnt, int64_t nchunks,
                                                         int64_t nsuper, uint8_t* __restrict__ sexit,
                                                         int32_t* __restrict__ scnt) {
  constexpr int SB = ZT / ZK;  // super-chunks per block
  __shared__ __align__(16) uint8_t se[SB * ZS * ZK];
  __shared__ int32_t sn[SB * ZS * ZK];
  const int64_t cb = (int64_t)blockIdx.x * SB * ZS;  // first chunk of the block
  const int64_t nc = ks_min64(nchunks - cb, SB * ZS);
  for (int i = threadIdx.x; i < nc * ZK; i += ZT) ks_cp_async4(&sn[i], cnt + cb * ZK + i);
  for (int i = threadIdx.x; i < nc * ZK / 4; i += ZT) ks_cp_async4(&se[4 * i], exit_off + cb * ZK + 4 * i);
  ks_cp_async_wait_all();
  __syncthreads();
  const int ls = threadIdx.x / ZK, o = threadIdx.x % ZK;
  const int64_t sidx = (int64_t)blockIdx.x * SB + ls;
  if (sidx >= nsuper) return;
  const int c_end = (int)ks_min64(nc, (ls + 1) * ZS);
  int e = o;
  int32_t k = 0;
  for (int c = ls * ZS; c < c_end; c++) {
    k += sn[c * ZK + e];
    e = se[c * ZK + e];
  }
  sexit[sidx * ZK + o] = (uint8_t)e;
  scnt[sidx * ZK + o] = k;
}
// Small-count variant (nsuper <= ZS2_MAX): the maps are staged in shared memory; the 32 lanes of
// warp 0 compose contiguous blocks of super-chunks for all ZK entry offsets, lane 0 walks the 32
// block maps from entry offset 0, and every lane then walks its block from its entry.  Only the
// one path that matters is followed, instead of composing every map pair.
constexpr int ZS2_MAX = 2048;
constexpr int ZS2_T = 256;
__global__ void __launch_bounds__(ZS2_T) zig_scan_small_kernel(const uint8_t* __restrict__ sexit,
                                                              const int32_t* __restrict__ scnt, int64_t nsuper,
                                                              uint8_t* __restrict__ sentry,
                                                              int64_t* __restrict__ sbase,
                                                              int64_t* __restrict__ total) {
  extern __shared__ __align__(16) unsigned char zs2[];
  int32_t* cn = reinterpret_cast<int32_t*>(zs2);                   // nsuper * ZK
  uint8_t* ex = zs2 + (size_t)ZS2_MAX * ZK * sizeof(int32_t);       // nsuper * ZK
  __shared__ int bexit[32][ZK];
  __shared__ int64_t bcnt[32][ZK];
  __shared__ int bentry[32];
  __shared__ int64_t bbase[32];
  const int nz = (int)nsuper * ZK;
  for (int i = threadIdx.x; i < nz; i += ZS2_T) ks_cp_async4(&cn[i], scnt + i);
  for (int i = threadIdx.x; i < nz / 4; i += ZS2_T) ks_cp_async4(&ex[4 * i], sexit + 4 * i);
  ks_cp_async_wait_all();
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const int per = ((int)nsuper + 31) / 32;
  const int c0 = min((int)nsuper, lane * per), c1 = min((int)nsuper, c0 + per);
#pragma unroll
  for (int o = 0; o < ZK; o++) {
    int e = o;
    int64_t k = 0;
    for (int c = c0; c < c1; c++) {
      k += cn[c * ZK + e];
      e = ex[c * ZK + e];
    }
    bexit[lane][o] = e;
    bcnt[lane][o] = k;
  }
  __syncwarp();
  if (lane == 0) {
    int e = 0;
    int64_t k = 0;
    for (int l = 0; l < 32; l++) {
      bentry[l] = e;
      bbase[l] = k;
      k += bcnt[l][e];
      e = bexit[l][e];
    }
    *total = k;
  }
  __syncwarp();
  int e = bentry[lane];
  int64_t k = bbase[lane];
  for (int c = c0; c < c1; c++) {
    sentry[c] = (uint8_t)e;
    sbase[c] = k;
    k += cn[c * ZK + e];
    e = ex[c * ZK + e];
  }
}

// One block: exclusive prefix of the super-chunk maps applied to entry offset 0
// (sequential per thread over a contiguous range, Hillis-Steele across threads).
constexpr int ZSCAN_T = 512;
__global__ void __launch_bounds__(ZSCAN_T) zig_scan_kernel(const uint8_t* __restrict__ sexit,
                                                          const int32_t* __restrict__ scnt,
                                                          int64_t nsuper, uint8_t* __restrict__ sentry,
                                                          int64_t* __restrict__ sbase,
                                                          int64_t* __restrict__ total) {
  // layout [buffer][offset][thread]: consecutive threads touch consecutive words (no bank conflicts)
  extern __shared__ unsigned char zsm[];
  int64_t (*fc)[ZK][ZSCAN_T] = reinterpret_cast<int64_t (*)[ZK][ZSCAN_T]>(zsm);
  uint8_t (*fe)[ZK][ZSCAN_T] = reinterpret_cast<uint8_t (*)[ZK][ZSCAN_T]>(zsm + 2 * ZSCAN_T * ZK * sizeof(int64_t));
  const int t = threadIdx.x;
  const int64_t per = (nsuper + ZSCAN_T - 1) / ZSCAN_T;
  const int64_t c_beg = ks_min64(nsuper, t * per), c_end = ks_min64(nsuper, c_beg + per);
#pragma unroll
  for (int o = 0; o < ZK; o++) {
    int e = o;
    int64_t k = 0;
    for (int64_t c = c_beg; c < c_end; c++) {
      k += scnt[c * ZK + e];
      e = sexit[c * ZK + e];
    }
    fe[0][o][t] = (uint8_t)e;
    fc[0][o][t] = k;
  }
  __syncthreads();
  int cur = 0;
  for (int off = 1; off < ZSCAN_T; off <<= 1) {
    // gather all ZK compositions into registers first (independent loads overlap), then store
    int ne[ZK];
    int64_t nk[ZK];
#pragma unroll
    for (int o = 0; o < ZK; o++) {
      if (t >= off) {
        const int mid = fe[cur][o][t - off];
        ne[o] = fe[cur][mid][t];
        nk[o] = fc[cur][o][t - off] + fc[cur][mid][t];
      } else {
        ne[o] = fe[cur][o][t];
        nk[o] = fc[cur][o][t];
      }
    }
#pragma unroll
    for (int o = 0; o < ZK; o++) {
      fe[cur ^ 1][o][t] = ne[o];
      fc[cur ^ 1][o][t] = nk[o];
    }
    __syncthreads();
    cur ^= 1;
  }
  int e = (t == 0) ? 0 : fe[cur][0][t - 1];
  int64_t k = (t == 0) ? 0 : fc[cur][0][t - 1];
  for (int64_t c = c_beg; c < c_end; c++) {
    sentry[c] = (uint8_t)e;
    sbase[c] = k;
    k += scnt[c * ZK + e];
    e = sexit[c * ZK + e];
  }
  if (t == ZSCAN_T - 1) *total = fc[cur][0][t];
}


// Emit the chain: per block of ZCB chunks, (1) chunk entry offsets / output bases from the
// super-chunk prefix (ZCB / ZS sequential walks over shared-memory maps), (2) one walk per chunk
// marking its chain positions in a 128-bit mask, (3) every position writes its value to
// base + rank-in-chunk (coalesced reads of val, near-contiguous writes of out).
__global__ void __launch_bounds__(ZT) zig_emit_kernel(const int16_t* __restrict__ cons,
                                                      const double* __restrict__ val, int64_t M, int64_t nchunks,
                                                      const uint8_t* __restrict__ exit_off,
                                                      const int32_t* __restrict__ cnt,
                                                      const uint8_t* __restrict__ sentry,
                                                      const int64_t* __restrict__ sbase, int64_t count,
                                                      double divisor, double* __restrict__ out,
                                                      int64_t* __restrict__ consumed,
                                                      const int64_t* __restrict__ total, int32_t* __restrict__ err) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && *total < count) atomicOr(err, 4);  // position budget exhausted
  __shared__ __align__(16) int16_t sc[ZCB * ZL];
  __shared__ __align__(16) uint8_t se[ZCB * ZK];
  __shared__ int32_t sn[ZCB * ZK];
  __shared__ uint8_t c_entry[ZCB];
  __shared__ int64_t c_base[ZCB];
  __shared__ uint64_t c_mask[ZCB][2];
  const int64_t blk_beg = (int64_t)blockIdx.x * ZCB * ZL;
  const int64_t cb = (int64_t)blockIdx.x * ZCB;
  const int nc = (int)ks_min64(nchunks - cb, ZCB);
  for (int i = threadIdx.x; i < nc * ZK; i += ZT) ks_cp_async4(&sn[i], cnt + cb * ZK + i);
  for (int i = threadIdx.x; i < nc * ZK / 4; i += ZT) ks_cp_async4(&se[4 * i], exit_off + cb * ZK + 4 * i);
  zig_stage_cons(sc, cons, M, blk_beg);  // waits for all copies
  if (threadIdx.x < ZCB / ZS) {
    const int s = threadIdx.x;
    const int64_t sidx = (int64_t)blockIdx.x * (ZCB / ZS) + s;
    if (s * ZS < nc) {
      int e = sentry[sidx];
      int64_t k = sbase[sidx];
      const int c_end = min(nc, (s + 1) * ZS);
      for (int c = s * ZS; c < c_end; c++) {
        c_entry[c] = (uint8_t)e;
        c_base[c] = k;
        k += sn[c * ZK + e];
        e = se[c * ZK + e];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < nc) {
    const int lc = threadIdx.x;
    const int beg = lc * ZL, end = (int)ks_min64(M - blk_beg, beg + ZL);
    uint64_t m0 = 0, m1 = 0;
    for (int q = beg + c_entry[lc]; q < end;) {
      const int rel = q - beg;
      const int step = sc[q];
      if (step <= 0) break;  // reported by zig_chunk_kernel
      q += step;
      if (rel < 64) m0 |= 1ull << rel; else m1 |= 1ull << (rel - 64);
    }
    c_mask[lc][0] = m0;
    c_mask[lc][1] = m1;
  }
  __syncthreads();
  const int npos = (int)ks_min64(M - blk_beg, (int64_t)nc * ZL);
  constexpr int U = 4;  // positions per thread per pass (their loads are issued together)
  for (int i0 = threadIdx.x; i0 < npos; i0 += U * ZT) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = i0 + u * ZT < npos ? val[blk_beg + i0 + u * ZT] : 0.0;
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int i = i0 + u * ZT;
      const int lc = i / ZL, rel = i % ZL;
      if (i >= npos) break;
      const uint64_t m0 = c_mask[lc][0], m1 = c_mask[lc][1];
      const bool on = rel < 64 ? ((m0 >> rel) & 1) : ((m1 >> (rel - 64)) & 1);
      if (!on) continue;
      const int rank = rel >= 64 ? __popcll(m0) + __popcll(m1 & ((1ull << (rel - 64)) - 1))
                                 : __popcll(m0 & ((1ull << rel) - 1));
      const int64_t k = c_base[lc] + rank;
      if (k < count) out[k] = v[u] / divisor;
      if (k == count - 1) *consumed = blk_beg + i + sc[i];
    }
  }
}


// Many PCG64 streams at once: out[m * rows * s + row * s + t] = random() draw (m * s + t) of stream
// `row` (states: 4 words per stream, state hi/lo then increment hi/lo).  The per-row sampler
// draws of fast_factor_matrix_update (tucker.py:361-369, one SeedSequence child per row).
__global__ void pcg_uniform_streams_kernel(const uint64_t* __restrict__ states, int64_t rows, int64_t per,
                                           int64_t s, int seeded, double* __restrict__ out) {
  const int64_t chunks = (per + RAW_PER_THREAD - 1) / RAW_PER_THREAD;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= rows * chunks) return;
  const int64_t row = q / chunks, k0 = (q - row * chunks) * RAW_PER_THREAD;
  u128 inc = mk128(states[4 * row + 2], states[4 * row + 3]);
  u128 st0 = mk128(states[4 * row], states[4 * row + 1]);
  if (seeded) {  // pcg64_set_seed: inc = 2 initseq + 1; state = ((0 M + inc) + initstate) M + inc
    inc = (inc << 1) | 1;
    st0 = (inc + st0) * PCG_MULT + inc;
  }
  u128 st = pcg_advance(st0, inc, (uint64_t)k0 + 1);
  const int n = (int)ks_min64(RAW_PER_THREAD, per - k0);
  for (int j = 0; j < n; j++) {
    const int64_t k = k0 + j, m = k / s, t = k - m * s;
    out[m * rows * s + row * s + t] = to_unit(pcg_output(st));
    st = st * PCG_MULT + inc;
  }
}

}  // namespace

extern "C" int ks_pcg64_random(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il, uint64_t skip,
                               int64_t count, double* out, void* stream) {
  if (count <= 0) return KS_OK;
  const int64_t threads = (count + RAW_PER_THREAD - 1) / RAW_PER_THREAD;
  pcg_uniform_kernel<<<ceil_div_u(threads, 256), 256, 0, (cudaStream_t)stream>>>(sh, sl, ih, il, skip,
                                                                              count, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

extern "C" int ks_pcg64_standard_normal(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il,
                                        int64_t count, double divisor, const uint64_t* ki,
                                        const double* wi, const double* fi, double* out,
                                        int32_t* status, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (count <= 0) return KS_OK;
  const int64_t batch_max = (int64_t)1 << 25;
  uint64_t skip = 0;
  // single batch with a caller status word: no host round trip (errors are OR-ed into *status)
  const bool async = status != nullptr && count <= batch_max;
  int64_t done = 0;
  while (done < count) {
    const int64_t n = ks_min64(batch_max, count - done);
    const int64_t M = n + n / 16 + 4096;            // positions evaluated
    const int64_t limit = M + 256;                  // raw draws generated (tail look-ahead)
    const int64_t nchunks = (M + ZL - 1) / ZL;
    ks::Scratch<uint64_t> raw(limit, st);
    ks::Scratch<double> val(M, st);
    ks::Scratch<int16_t> cons(M, st);
    ks::Scratch<uint8_t> exit_off(nchunks * ZK, st);
    ks::Scratch<int32_t> cnt(nchunks * ZK, st);
    const int64_t nsuper = (nchunks + ZS - 1) / ZS;
    ks::Scratch<uint8_t> sexit(nsuper * ZK, st);
    ks::Scratch<int32_t> scnt(nsuper * ZK, st);
    ks::Scratch<uint8_t> sentry(nsuper, st);
    ks::Scratch<int64_t> sbase(nsuper, st);
    ks::Scratch<int64_t> tail(2, st);  // [0] chain length over M positions, [1] draws consumed
    ks::Scratch<int32_t> err_s(async ? 0 : 1, st);
    int32_t* err = async ? status : err_s.p;
    KS_REQUIRE(raw.p && val.p && cons.p && exit_off.p && cnt.p && tail.p && err && sexit.p && scnt.p &&
               sentry.p && sbase.p,
               KS_ECUDA, "scratch allocation failed");
    if (!async) KS_TRY_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
    const int64_t rthreads = (limit + RAW_PER_THREAD - 1) / RAW_PER_THREAD;
    pcg_raw_kernel<<<ceil_div_u(rthreads, 256), 256, 0, st>>>(sh, sl, ih, il, skip, limit, raw.p);
    KS_CHECK_LAUNCH();
    zig_eval_kernel<<<ceil_div_u(M, 256), 256, 0, st>>>(raw.p, M, limit, ki, wi, fi, val.p, cons.p);
    KS_CHECK_LAUNCH();
    const unsigned nblk = ceil_div_u(nchunks, ZCB);
    zig_chunk_kernel<<<nblk, ZCB * ZCT, 0, st>>>(cons.p, M, nchunks, exit_off.p, cnt.p, err);
    KS_CHECK_LAUNCH();
    zig_compose_kernel<<<ceil_div_u(nsuper, ZT / ZK), ZT, 0, st>>>(exit_off.p, cnt.p, nchunks, nsuper,
                                                                   sexit.p, scnt.p);
    KS_CHECK_LAUNCH();
    if (nsuper <= ZS2_MAX) {
      const size_t smem2 = (size_t)ZS2_MAX * ZK * (sizeof(int32_t) + 1);
      KS_TRY_CUDA(cudaFuncSetAttribute(zig_scan_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem2));
      zig_scan_small_kernel<<<1, ZS2_T, smem2, st>>>(sexit.p, scnt.p, nsuper, sentry.p, sbase.p, tail.p);
    } else {
      const size_t scan_smem = (size_t)2 * ZSCAN_T * ZK * (1 + sizeof(int64_t));
      KS_TRY_CUDA(cudaFuncSetAttribute(zig_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)scan_smem));
      zig_scan_kernel<<<1, ZSCAN_T, scan_smem, st>>>(sexit.p, scnt.p, nsuper, sentry.p, sbase.p, tail.p);
    }
    KS_CHECK_LAUNCH();
    zig_emit_kernel<<<nblk, ZT, 0, st>>>(cons.p, val.p, M, nchunks, exit_off.p, cnt.p, sentry.p, sbase.p, n,
                                         divisor, out + done, tail.p + 1, tail.p, err);
    KS_CHECK_LAUNCH();
    if (async) break;
    int64_t host[2];
    int32_t herr = 0;
    KS_TRY_CUDA(cudaMemcpyAsync(host, tail.p, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KS_TRY_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    KS_TRY_CUDA(cudaStreamSynchronize(st));
    KS_REQUIRE(herr == 0, KS_ENUMERICAL, "ziggurat chain resolution failed (code %d)", herr);
    KS_REQUIRE(host[0] >= n, KS_ENUMERICAL, "ziggurat position budget exhausted");
    skip += (uint64_t)host[1];
    done += n;
  }
  return KS_OK;
}

extern "C" int ks_pcg64_random_streams(const uint64_t* states, int32_t seeded, int64_t rows, int32_t nf, int64_t s,
                                       double* out, void* stream) {
  if (rows <= 0 || s <= 0 || nf <= 0) return KS_OK;
  const int64_t per = (int64_t)nf * s;
  const int64_t threads = rows * ((per + RAW_PER_THREAD - 1) / RAW_PER_THREAD);
  pcg_uniform_streams_kernel<<<ceil_div_u(threads, 256), 256, 0, (cudaStream_t)stream>>>(states, rows, per, s, seeded,
                                                                                          out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}
