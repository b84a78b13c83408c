// Stable LSD radix sort of (uint64 key, int64 value) pairs and device-wide scans.
// Used to build the sparse diagonal of a row sketch (kron.py:173-190: np.argsort(kind="stable")
// + np.unique) and the grouped (left, right) ordering of the sketched operator (kron.py:225-300).
#include "ks_common.cuh"

namespace {

constexpr int RS_T = 256;        // threads per tile
constexpr int RS_ROUNDS = 8;     // elements per thread
constexpr int RS_TILE = RS_T * RS_ROUNDS;
constexpr int RS_BITS = 8;
constexpr int RS_DIG = 1 << RS_BITS;

__global__ void __launch_bounds__(RS_T) rs_hist_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                                      int shift, int64_t ntiles,
                                                      int32_t* __restrict__ hist) {
  __shared__ int32_t h[RS_DIG];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
  for (int r = 0; r < RS_ROUNDS; r++) {
    const int64_t i = base + r * RS_T + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & (RS_DIG - 1)], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// Exclusive scan of `n` int32 counts into int64 offsets, single block.
__global__ void __launch_bounds__(1024) scan_small_kernel(const int32_t* __restrict__ in, int64_t n,
                                                          int64_t* __restrict__ out) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t b0 = 0; b0 < n; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    int64_t v = (i < n) ? in[i] : 0;
    const int64_t orig = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    if (lane == 31) wsum[wid] = v;
    __syncthreads();
    if (wid == 0) {
      int64_t t = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += u;
      }
      wsum[lane] = t;
    }
    __syncthreads();
    const int64_t incl = v + (wid > 0 ? wsum[wid - 1] : 0) + carry;
    if (i < n) out[i] = incl - orig;
    __syncthreads();
    if (threadIdx.x == 1023) carry = incl;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(RS_T) rs_scatter_kernel(const uint64_t* __restrict__ kin,
                                                         const int64_t* __restrict__ vin, int64_t n,
                                                         int shift, int64_t ntiles,
                                                         const int64_t* __restrict__ offs,
                                                         uint64_t* __restrict__ kout,
                                                         int64_t* __restrict__ vout) {
  __shared__ int32_t wcnt[RS_T / 32][RS_DIG];
  __shared__ int32_t run[RS_DIG];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  run[tid] = 0;
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
  const int64_t toff = offs[(int64_t)tid * ntiles + blockIdx.x];  // this tile's base for digit `tid`
  __shared__ int64_t s_toff[RS_DIG];
  s_toff[tid] = toff;
  for (int r = 0; r < RS_ROUNDS; r++) {
    const int64_t i = base + r * RS_T + tid;
    const bool valid = i < n;
    uint64_t k = 0;
    int64_t v = 0;
    int dig = RS_DIG;  // sentinel for invalid lanes
    if (valid) {
      k = kin[i];
      v = vin[i];
      dig = (int)((k >> shift) & (RS_DIG - 1));
    }
#pragma unroll
    for (int w = 0; w < RS_T / 32; w++) wcnt[w][tid] = 0;
    __syncthreads();
    const unsigned peers = __match_any_sync(0xffffffffu, dig);
    const int leader = __ffs(peers) - 1;
    const int rank_in_warp = __popc(peers & ((1u << lane) - 1u));
    if (valid && lane == leader) wcnt[wid][dig] = __popc(peers);
    __syncthreads();
    {
      int32_t acc = run[tid];
#pragma unroll
      for (int w = 0; w < RS_T / 32; w++) {
        const int32_t c = wcnt[w][tid];
        wcnt[w][tid] = acc;
        acc += c;
      }
      run[tid] = acc;
    }
    __syncthreads();
    if (valid) {
      const int64_t pos = s_toff[dig] + wcnt[wid][dig] + rank_in_warp;
      kout[pos] = k;
      vout[pos] = v;
    }
    __syncthreads();
  }
}

// Two-kernel exclusive scan for larger n: per-tile totals, then every tile scans its own
// elements after summing the totals of the tiles before it (fixed order, deterministic).
constexpr int SC_T = 512, SC_PER = 4, SC_TILE = SC_T * SC_PER;

__global__ void __launch_bounds__(SC_T) tile_sum_kernel(const int32_t* __restrict__ in, int64_t n,
                                                       int64_t* __restrict__ tsum) {
  __shared__ int64_t red[SC_T / 32];
  const int64_t base = (int64_t)blockIdx.x * SC_TILE;
  int64_t v = 0;
#pragma unroll
  for (int k = 0; k < SC_PER; k++) {
    const int64_t i = base + k * SC_T + threadIdx.x;
    if (i < n) v += in[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < SC_T / 32; w++) t += red[w];
    tsum[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(SC_T) tile_scan_kernel(const int32_t* __restrict__ in, int64_t n,
                                                        const int64_t* __restrict__ tsum,
                                                        int64_t* __restrict__ out) {
  __shared__ int64_t wsum[SC_T / 32];
  __shared__ int64_t s_off;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid == 0) {  // offset = sum of the preceding tiles' totals
    int64_t o = 0;
    for (int b = lane; b < (int)blockIdx.x; b += 32) o += tsum[b];
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) o += __shfl_xor_sync(0xffffffffu, o, k);
    if (lane == 0) s_off = o;
  }
  // each thread owns SC_PER consecutive elements
  const int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_PER;
  int32_t x[SC_PER];
  int64_t loc = 0;
#pragma unroll
  for (int k = 0; k < SC_PER; k++) {
    x[k] = (base + k < n) ? in[base + k] : 0;
    loc += x[k];
  }
  int64_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int64_t t = lane < SC_T / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    if (lane < SC_T / 32) wsum[lane] = t;
  }
  __syncthreads();
  int64_t run = s_off + (wid ? wsum[wid - 1] : 0) + incl - loc;
#pragma unroll
  for (int k = 0; k < SC_PER; k++) {
    if (base + k < n) out[base + k] = run;
    run += x[k];
  }
}

}  // namespace

namespace ks {

int scan_exclusive_i32(cudaStream_t st, const int32_t* in, int64_t n, int64_t* out);

// Stable sort of n (key, value) pairs on the low `bits` bits of the key.  Result in
// (keys, vals) (the input buffers are overwritten).
int radix_sort_pairs(cudaStream_t st, uint64_t* keys, int64_t* vals, int64_t n, int bits) {
  if (n <= 1 || bits <= 0) return KS_OK;
  const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
  Scratch<uint64_t> k2(n, st);
  Scratch<int64_t> v2(n, st);
  Scratch<int32_t> hist(ntiles * RS_DIG, st);
  Scratch<int64_t> offs(ntiles * RS_DIG, st);
  KS_REQUIRE(k2.p && v2.p && hist.p && offs.p, KS_ECUDA, "scratch allocation failed");
  uint64_t* ka = keys; int64_t* va = vals;
  uint64_t* kb = k2.p; int64_t* vb = v2.p;
  const int passes = (bits + RS_BITS - 1) / RS_BITS;
  for (int p = 0; p < passes; p++) {
    const int shift = p * RS_BITS;
    rs_hist_kernel<<<(unsigned)ntiles, RS_T, 0, st>>>(ka, n, shift, ntiles, hist.p);
    KS_CHECK_LAUNCH();
    int rc = scan_exclusive_i32(st, hist.p, ntiles * RS_DIG, offs.p);
    if (rc) return rc;
    rs_scatter_kernel<<<(unsigned)ntiles, RS_T, 0, st>>>(ka, va, n, shift, ntiles, offs.p, kb, vb);
    KS_CHECK_LAUNCH();
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (ka != keys) {
    KS_TRY_CUDA(cudaMemcpyAsync(keys, ka, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    KS_TRY_CUDA(cudaMemcpyAsync(vals, va, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  }
  return KS_OK;
}

int scan_exclusive_i32(cudaStream_t st, const int32_t* in, int64_t n, int64_t* out) {
  if (n <= 0) return KS_OK;
  if (n <= 4096) {
    scan_small_kernel<<<1, 1024, 0, st>>>(in, n, out);
    KS_CHECK_LAUNCH();
    return KS_OK;
  }
  const int64_t tiles = (n + SC_TILE - 1) / SC_TILE;
  Scratch<int64_t> tsum(tiles, st);
  KS_REQUIRE(tsum.p, KS_ECUDA, "scratch allocation failed");
  tile_sum_kernel<<<(unsigned)tiles, SC_T, 0, st>>>(in, n, tsum.p);
  KS_CHECK_LAUNCH();
  tile_scan_kernel<<<(unsigned)tiles, SC_T, 0, st>>>(in, n, tsum.p, out);
  KS_CHECK_LAUNCH();
  return KS_OK;
}

}  // namespace ks
