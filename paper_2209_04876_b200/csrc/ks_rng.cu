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
//     start position is resolved in parallel: one kernel per super-chunk of 4096 positions
//     draws the raw outputs, computes "value, consumption if a normal started here" at every
//     position, and records for each 128-position chunk and each possible entry offset the exit
//     offset (walks from different entries merge after a step or two), composed into the
//     super-chunk's map; a one-block scan composes the super-chunk maps; a final pass emits the
//     chain values.  The ziggurat tables
//     (ki/wi/fi) are read from the installed NumPy's libnpyrandom.a by the host and passed in.
#include "ks_common.cuh"
#include "ks_pcg_jump.cuh"

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
template <class RAW>
__device__ __forceinline__ int zig_eval(RAW raw, int64_t p, int64_t limit, const ZigTables& T, double* out) {
  int64_t q = p;
  for (;;) {
    if (q >= limit) return -1;
    uint64_t r = raw(q++);
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
        const double u1 = to_unit(raw(q++));
        const double u2 = to_unit(raw(q++));
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
      const double u = to_unit(raw(q++));
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(T.fi[idx - 1], T.fi[idx]), u), T.fi[idx]);
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
        *out = x;
        return (int)(q - p);
      }
    }
  }
}

constexpr int ZL = 128;  // chunk length (positions)
constexpr int ZK = 16;   // entry offsets tracked per chunk
constexpr int ZCB = 32;  // chunks per block of the chunk / emit kernels
constexpr int ZS = 32;   // chunks per super-chunk (ZCB % ZS == 0)
constexpr int ZT = 256;  // threads of the compose / emit kernels

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

// 128-bit position masks of a chunk (m0: positions 0..63, m1: 64..127).
__device__ __forceinline__ void mask_set_range(uint64_t& m0, uint64_t& m1, int a, int b) {  // [a, b)
  auto bits = [](int lo, int hi) -> uint64_t {  // bits [lo, hi) of a word, 0 <= lo <= hi <= 64
    if (hi <= lo) return 0ull;
    const uint64_t up = hi >= 64 ? ~0ull : ((1ull << hi) - 1);
    return up & (~0ull << lo);
  };
  m0 |= bits(min(a, 64), min(b, 64));
  m1 |= bits(max(a, 64) - 64, max(b, 64) - 64);
}

// The chain of a chunk entered at offset o: positions whose consumption is 1 follow each other,
// so the walk only stops at the "special" positions (mask s0/s1: consumption != 1, typically
// ~1.5 per chunk) instead of stepping through all 128.  len: positions of the chunk (< ZL only
// for the last one).  Returns the exit offset into the next chunk (-1: bad consumption), the
// chain positions in m0/m1.
__device__ __forceinline__ int chunk_walk(const int16_t* sc, int len, uint64_t s0, uint64_t s1, int o, uint64_t& m0,
                                          uint64_t& m1) {
  m0 = 0;
  m1 = 0;
  int q = o;
  while (q < len) {
    int sp;
    if (q < 64) {
      const uint64_t t = s0 & (~0ull << q);
      sp = t ? __ffsll((long long)t) - 1 : (s1 ? 63 + __ffsll((long long)s1) : ZL);
    } else {
      const uint64_t t = s1 & (~0ull << (q - 64));
      sp = t ? 63 + __ffsll((long long)t) : ZL;
    }
    if (sp >= len) {  // unit steps to the end of the chunk
      mask_set_range(m0, m1, q, len);
      q = len;
      break;
    }
    mask_set_range(m0, m1, q, sp + 1);
    const int k = sc[sp];
    if (k <= 0) return -1;
    q = sp + k;
  }
  return q - len;
}

// Masks of the positions of chunk c (of a block's staged consumptions) whose consumption is
// not 1; one warp, all lanes.
__device__ __forceinline__ void chunk_special(const int16_t* sc, int c, int len, uint64_t& s0, uint64_t& s1) {
  const int lane = threadIdx.x & 31;
  unsigned b[4];
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int rel = lane + 32 * j;
    b[j] = __ballot_sync(0xffffffffu, rel < len && sc[c * ZL + rel] != 1);
  }
  s0 = (uint64_t)b[0] | ((uint64_t)b[1] << 32);
  s1 = (uint64_t)b[2] | ((uint64_t)b[3] << 32);
}

// Fused front of the chain resolution, one block per super-chunk (ZS chunks of ZL positions):
// the block's raw draws (each thread jumps once to its first position, then strides by ZT with
// the 256-step affine map of the LCG, so shared-memory stores are conflict-free), the value and
// consumption of a normal starting at every position (draws past the staged window are
// recomputed by a jump: astronomically rare), the chunk maps (ZK entry offsets, ZFT threads per
// chunk) and their composition into the super-chunk map.  Replaces the raw / eval / chunk /
// compose launches with one; same outputs.
constexpr int ZRX = 0;            // raw draws staged past the super-chunk (look-ahead; later draws are recomputed)
constexpr int ZRS = ZS * ZL + ZRX;
constexpr int ZSLOW = 256;        // listed slow-path positions per super-chunk (~1.2 % of 4096 expected)
static_assert(ZRS % ZT == 0 && ZT == 256 && ZK <= 32, "front kernel shape");
__global__ void __launch_bounds__(ZT) zig_front_kernel(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il,
                                                       uint64_t skip, int64_t M, int64_t limit,
                                                       const uint64_t* __restrict__ ki, const double* __restrict__ wi,
                                                       const double* __restrict__ fi, double* __restrict__ val,
                                                       int16_t* __restrict__ cons, int64_t nchunks,
                                                       uint8_t* __restrict__ exit_off, int32_t* __restrict__ cnt,
                                                       uint8_t* __restrict__ sexit, int32_t* __restrict__ scnt,
                                                       int32_t* __restrict__ err) {
  __shared__ uint64_t raw_s[ZRS];
  __shared__ __align__(16) int16_t sc[ZS * ZL];
  __shared__ uint8_t se[ZS * ZK];
  __shared__ int32_t sn[ZS * ZK];
  __shared__ uint64_t ki_s[256];
  __shared__ double wi_s[256];
  const int tid = threadIdx.x;
  ki_s[tid] = __ldg(&ki[tid]);
  wi_s[tid] = __ldg(&wi[tid]);
  const int64_t blk_beg = (int64_t)blockIdx.x * ZS * ZL;
  const u128 state0 = mk128(sh, sl), inc = mk128(ih, il);
  // raw draws blk_beg + [0, ZRS): position q is the output of the state after skip + q + 1 steps.
  // One jump to the block's start, then each thread's offset and its ZT-step stride from the
  // precomputed affine maps (ks_pcg_jump.cuh): two 128-bit multiply-adds per draw at most
  __shared__ uint64_t s_blk[2];
  if (tid == 0) {
    const u128 sb = pcg_advance(state0, inc, skip + (uint64_t)blk_beg + 1);
    s_blk[0] = (uint64_t)(sb >> 64);
    s_blk[1] = (uint64_t)sb;
  }
  __syncthreads();
  {
    const u128 sb = mk128(s_blk[0], s_blk[1]);
    u128 st = mk128(ks_pcg::kJump[tid][0], ks_pcg::kJump[tid][1]) * sb +
              mk128(ks_pcg::kJump[tid][2], ks_pcg::kJump[tid][3]) * inc;
    const u128 am = mk128(ks_pcg::kJump[ZT][0], ks_pcg::kJump[ZT][1]);
    const u128 ap = mk128(ks_pcg::kJump[ZT][2], ks_pcg::kJump[ZT][3]) * inc;
#pragma unroll 4
    for (int i = tid; i < ZRS; i += ZT) {
      raw_s[i] = pcg_output(st);
      st = am * st + ap;
    }
  }
  __syncthreads();
  const ZigTables T{ki, wi, fi};
  auto raw = [&](int64_t q) -> uint64_t {
    const int64_t i = q - blk_beg;
    return i < ZRS ? raw_s[i] : pcg_output(pcg_advance(state0, inc, skip + (uint64_t)q + 1));
  };
  // the ziggurat's first test (taken ~99% of the time) for every position from the staged tables;
  // the positions that fail it are listed and evaluated afterwards by whole warps (inline, ~27 %
  // of the warps would carry one lane through the long branch)
  __shared__ int s_nslow;
  __shared__ int s_slow[ZSLOW];
  if (tid == 0) s_nslow = 0;
  __syncthreads();
#pragma unroll 4
  for (int i = tid; i < ZS * ZL; i += ZT) {
    const int64_t p = blk_beg + i;
    int16_t c16 = 1;  // positions >= M read as 1 (as the staged chunk walks do)
    if (p < M) {
      uint64_t r = raw_s[i];
      const int idx = (int)(r & 0xff);
      r >>= 8;
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      double v = __dmul_rn((double)rabs, wi_s[idx]);
      if (r & 1) v = -v;
      if (!(rabs < ki_s[idx]) || p >= limit) {
        const int slot = atomicAdd(&s_nslow, 1);
        if (slot < ZSLOW) {
          s_slow[slot] = i;
          c16 = 0;  // filled in by the slow pass
        } else {  // (list full: evaluate here)
          const int c = zig_eval(raw, p, limit, T, &v);
          c16 = (int16_t)(c > 32000 ? -1 : c);
          val[p] = v;
          cons[p] = c16;
        }
      } else {
        val[p] = v;
        cons[p] = c16;
      }
    }
    sc[i] = c16;
  }
  __syncthreads();
  for (int k = tid; k < min(s_nslow, ZSLOW); k += ZT) {
    const int i = s_slow[k];
    const int64_t p = blk_beg + i;
    double v = 0.0;
    const int c = zig_eval(raw, p, limit, T, &v);
    const int16_t c16 = (int16_t)(c > 32000 ? -1 : c);
    val[p] = v;
    cons[p] = c16;
    sc[i] = c16;
  }
  __syncthreads();
  // chunk maps: one warp per chunk at a time (special-position masks by ballot), lanes 0..ZK-1
  // walk one entry offset each
  {
    const int warp = tid >> 5, lane = tid & 31;
    for (int lc = warp; lc < ZS; lc += ZT / 32) {
      const int64_t c = (int64_t)blockIdx.x * ZS + lc;
      if (c >= nchunks) break;
      const int len = (int)ks_min64(M - blk_beg - (int64_t)lc * ZL, ZL);
      uint64_t s0, s1;
      chunk_special(sc, lc, len, s0, s1);
      if (lane < ZK) {
        uint64_t m0, m1;
        const int e = chunk_walk(sc + lc * ZL, len, s0, s1, lane, m0, m1);
        if (e < 0) atomicOr(err, 1);
        else if (e >= ZK) atomicOr(err, 2);
        const int n = __popcll(m0) + __popcll(m1);
        exit_off[c * ZK + lane] = (uint8_t)(e < 0 ? 0 : e);
        cnt[c * ZK + lane] = n;
        se[lc * ZK + lane] = (uint8_t)(e < 0 || e >= ZK ? 0 : e);
        sn[lc * ZK + lane] = n;
      }
    }
  }
  __syncthreads();
  if (tid < ZK) {  // the super-chunk map: the block's chunk maps composed for every entry offset
    const int nc = (int)ks_min64(nchunks - (int64_t)blockIdx.x * ZS, ZS);
    int e = tid;
    int32_t k = 0;
    for (int c = 0; c < nc; c++) {
      k += sn[c * ZK + e];
      e = se[c * ZK + e];
    }
    sexit[(int64_t)blockIdx.x * ZK + tid] = (uint8_t)e;
    scnt[(int64_t)blockIdx.x * ZK + tid] = k;
  }
}

// Small-count variant (nsuper <= ZS2_MAX): the maps are staged in shared memory; warp o composes
// the 32 contiguous blocks of super-chunks for entry offset o (one block per lane), one thread
// walks the 32 block maps from entry offset 0, and warp 0's lanes then walk their blocks from
// their entries.  Only the one path that matters is followed, instead of composing every map pair.
constexpr int ZS2_MAX = 2048;
constexpr int ZS2_T = 32 * ZK;  // one warp per entry offset
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
  const int lane = threadIdx.x & 31, o = threadIdx.x >> 5;
  const int per = ((int)nsuper + 31) / 32;
  const int c0 = min((int)nsuper, lane * per), c1 = min((int)nsuper, c0 + per);
  {  // lane's block of super-chunks composed for entry offset o (one warp per offset)
    int e = o;
    int64_t k = 0;
    for (int c = c0; c < c1; c++) {
      k += cn[c * ZK + e];
      e = ex[c * ZK + e];
    }
    bexit[lane][o] = e;
    bcnt[lane][o] = k;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
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
  __syncthreads();
  if (o != 0) return;
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
  {  // each chunk's chain positions from its entry offset (mask walk, one warp per chunk)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int lc = warp; lc < nc; lc += ZT / 32) {
      const int len = (int)ks_min64(M - blk_beg - (int64_t)lc * ZL, ZL);
      uint64_t s0, s1;
      chunk_special(sc, lc, len, s0, s1);
      if (lane == 0) {
        uint64_t m0, m1;
        if (chunk_walk(sc + lc * ZL, len, s0, s1, c_entry[lc], m0, m1) < 0) m0 = m1 = 0;  // reported by the front kernel
        c_mask[lc][0] = m0;
        c_mask[lc][1] = m1;
      }
    }
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
    KS_REQUIRE(val.p && cons.p && exit_off.p && cnt.p && tail.p && err && sexit.p && scnt.p &&
               sentry.p && sbase.p,
               KS_ECUDA, "scratch allocation failed");
    if (!async) KS_TRY_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
    const unsigned nblk = ceil_div_u(nchunks, ZCB);
    // one block per super-chunk: raw draws, values / consumptions, chunk and super-chunk maps
    zig_front_kernel<<<(unsigned)nsuper, ZT, 0, st>>>(sh, sl, ih, il, skip, M, limit, ki, wi, fi, val.p, cons.p,
                                                      nchunks, exit_off.p, cnt.p, sexit.p, scnt.p, err);
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
