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
constexpr int ZCB = 128; // chunks per block of the chunk / emit kernels

// For each chunk and entry offset o < ZK: exit offset into the next chunk and normals emitted.
__global__ void zig_chunk_kernel(const int16_t* __restrict__ cons, int64_t M, int64_t nchunks,
                                 uint8_t* __restrict__ exit_off, int32_t* __restrict__ cnt,
                                 int32_t* __restrict__ err) {
  // stage the block's consumption table in shared memory (coalesced), then walk from smem
  __shared__ int16_t sc[ZCB * ZL];
  const int64_t blk_beg = (int64_t)blockIdx.x * ZCB * ZL;
  for (int i = threadIdx.x; i < ZCB * ZL; i += blockDim.x) {
    const int64_t p = blk_beg + i;
    sc[i] = (p < M) ? cons[p] : (int16_t)1;
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const int64_t beg = c * ZL, end = ks_min64(M, beg + ZL);
#define cons(q) sc[(q) - blk_beg]
  uint64_t mask[ZL / 64] = {0, 0};
  int64_t q = beg;
  int c0 = 0;
  while (q < end) {
    const int k = cons(q);
    if (k <= 0) { atomicOr(err, 1); return; }
    mask[(q - beg) >> 6] |= 1ull << ((q - beg) & 63);
    c0++;
    q += k;
  }
  const int e0 = (int)(q - end);
  if (e0 >= ZK) { atomicOr(err, 2); return; }
  exit_off[c * ZK] = (uint8_t)e0;
  cnt[c * ZK] = c0;
  for (int o = 1; o < ZK; o++) {
    int64_t qq = beg + o;
    int steps = 0;
    while (qq < end && !((mask[(qq - beg) >> 6] >> ((qq - beg) & 63)) & 1)) {
      const int k = cons(qq);
      if (k <= 0) { atomicOr(err, 1); return; }
      steps++;
      qq += k;
    }
    if (qq >= end) {
      const int e = (int)(qq - end);
      if (e >= ZK) { atomicOr(err, 2); return; }
      exit_off[c * ZK + o] = (uint8_t)e;
      cnt[c * ZK + o] = steps;
    } else {
      // merged with the offset-0 walk at qq: remaining count = walk-0 positions >= qq
      const int rel = (int)(qq - beg);
      int before = 0;
      if (rel >= 64) before = __popcll(mask[0]) + __popcll(mask[1] & ((1ull << (rel - 64)) - 1));
      else before = __popcll(mask[0] & ((rel == 0) ? 0ull : ((1ull << rel) - 1)));
      exit_off[c * ZK + o] = (uint8_t)e0;
      cnt[c * ZK + o] = steps + (c0 - before);
    }
  }
#undef cons
}

constexpr int ZS = 16;  // chunks per super-chunk

// Compose the maps of ZS consecutive chunks into one super-chunk map.
__global__ void zig_compose_kernel(const uint8_t* __restrict__ exit_off, const int32_t* __restrict__ cnt,
                                   int64_t nchunks, int64_t nsuper, uint8_t* __restrict__ sexit,
                                   int32_t* __restrict__ scnt) {
  const int64_t sidx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sidx >= nsuper) return;
  const int64_t c_beg = sidx * ZS, c_end = ks_min64(nchunks, c_beg + ZS);
  for (int o = 0; o < ZK; o++) {
    int e = o;
    int32_t k = 0;
    for (int64_t c = c_beg; c < c_end; c++) {
      k += cnt[c * ZK + e];
      e = exit_off[c * ZK + e];
    }
    sexit[sidx * ZK + o] = (uint8_t)e;
    scnt[sidx * ZK + o] = k;
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
    for (int o = 0; o < ZK; o++) {
      if (t >= off) {
        const int mid = fe[cur][o][t - off];
        fe[cur ^ 1][o][t] = fe[cur][mid][t];
        fc[cur ^ 1][o][t] = fc[cur][o][t - off] + fc[cur][mid][t];
      } else {
        fe[cur ^ 1][o][t] = fe[cur][o][t];
        fc[cur ^ 1][o][t] = fc[cur][o][t];
      }
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

// Per super-chunk: entry offsets and output bases of its chunks.
__global__ void zig_expand_kernel(const uint8_t* __restrict__ exit_off, const int32_t* __restrict__ cnt,
                                  int64_t nchunks, int64_t nsuper, const uint8_t* __restrict__ sentry,
                                  const int64_t* __restrict__ sbase, uint8_t* __restrict__ entry,
                                  int64_t* __restrict__ base) {
  const int64_t sidx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sidx >= nsuper) return;
  const int64_t c_beg = sidx * ZS, c_end = ks_min64(nchunks, c_beg + ZS);
  int e = sentry[sidx];
  int64_t k = sbase[sidx];
  for (int64_t c = c_beg; c < c_end; c++) {
    entry[c] = (uint8_t)e;
    base[c] = k;
    k += cnt[c * ZK + e];
    e = exit_off[c * ZK + e];
  }
}

__global__ void zig_emit_kernel(const int16_t* __restrict__ cons, const double* __restrict__ val,
                                int64_t M, int64_t nchunks, const uint8_t* __restrict__ entry,
                                const int64_t* __restrict__ base, int64_t count, double divisor,
                                double* __restrict__ out, int64_t* __restrict__ consumed) {
  __shared__ int16_t sc[ZCB * ZL];
  const int64_t blk_beg = (int64_t)blockIdx.x * ZCB * ZL;
  for (int i = threadIdx.x; i < ZCB * ZL; i += blockDim.x) {
    const int64_t p = blk_beg + i;
    sc[i] = (p < M) ? cons[p] : (int16_t)1;
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const int64_t beg = c * ZL, end = ks_min64(M, beg + ZL);
  int64_t q = beg + entry[c];
  int64_t k = base[c];
  while (q < end) {
    const int step = sc[q - blk_beg];
    if (k < count) out[k] = val[q] / divisor;
    if (k == count - 1) *consumed = q + step;
    k++;
    q += step;
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
                                        void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (count <= 0) return KS_OK;
  const int64_t batch_max = (int64_t)1 << 25;
  uint64_t skip = 0;
  const u128 s0 = mk128(sh, sl);
  (void)s0;
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
    ks::Scratch<uint8_t> entry(nchunks, st);
    ks::Scratch<int64_t> base(nchunks + 2, st);  // [nchunks] total, [nchunks+1] consumed
    ks::Scratch<int32_t> err(1, st);
    KS_REQUIRE(raw.p && val.p && cons.p && exit_off.p && cnt.p && entry.p && base.p && err.p &&
               sexit.p && scnt.p && sentry.p && sbase.p,
               KS_ECUDA, "scratch allocation failed");
    KS_TRY_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int32_t), st));
    const int64_t rthreads = (limit + RAW_PER_THREAD - 1) / RAW_PER_THREAD;
    pcg_raw_kernel<<<ceil_div_u(rthreads, 256), 256, 0, st>>>(sh, sl, ih, il, skip, limit, raw.p);
    KS_CHECK_LAUNCH();
    zig_eval_kernel<<<ceil_div_u(M, 256), 256, 0, st>>>(raw.p, M, limit, ki, wi, fi, val.p, cons.p);
    KS_CHECK_LAUNCH();
    zig_chunk_kernel<<<ceil_div_u(nchunks, 128), 128, 0, st>>>(cons.p, M, nchunks, exit_off.p,
                                                               cnt.p, err.p);
    KS_CHECK_LAUNCH();
    zig_compose_kernel<<<ceil_div_u(nsuper, 128), 128, 0, st>>>(exit_off.p, cnt.p, nchunks, nsuper,
                                                                 sexit.p, scnt.p);
    KS_CHECK_LAUNCH();
    const size_t scan_smem = (size_t)2 * ZSCAN_T * ZK * (1 + sizeof(int64_t));
    KS_TRY_CUDA(cudaFuncSetAttribute(zig_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)scan_smem));
    zig_scan_kernel<<<1, ZSCAN_T, scan_smem, st>>>(sexit.p, scnt.p, nsuper, sentry.p, sbase.p,
                                                   base.p + nchunks);
    KS_CHECK_LAUNCH();
    zig_expand_kernel<<<ceil_div_u(nsuper, 128), 128, 0, st>>>(exit_off.p, cnt.p, nchunks, nsuper,
                                                                sentry.p, sbase.p, entry.p, base.p);
    KS_CHECK_LAUNCH();
    zig_emit_kernel<<<ceil_div_u(nchunks, 128), 128, 0, st>>>(cons.p, val.p, M, nchunks, entry.p,
                                                              base.p, n, divisor, out + done,
                                                              base.p + nchunks + 1);
    KS_CHECK_LAUNCH();
    int64_t host[2];
    int32_t herr = 0;
    KS_TRY_CUDA(cudaMemcpyAsync(host, base.p + nchunks, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KS_TRY_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    KS_TRY_CUDA(cudaStreamSynchronize(st));
    KS_REQUIRE(herr == 0, KS_ENUMERICAL, "ziggurat chain resolution failed (code %d)", herr);
    KS_REQUIRE(host[0] >= n, KS_ENUMERICAL, "ziggurat position budget exhausted");
    skip += (uint64_t)host[1];
    done += n;
  }
  return KS_OK;
}
