// Shared helpers for the kronsolve B200 library (sm_100a, FP64).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>

#include "../../include/kronsolve_b200.h"

namespace ks {

void set_error(const char* fmt, ...);

// Diagnostic switches (environment variables), read ONCE per process on
// first use: no getenv on the solve path, and a captured graph cannot disagree with later calls.
enum EnvSwitch { ENV_TALL, ENV_KRON2, ENV_RICHARDSON, ENV_NO_EIGBASIS, ENV_GRAM_SCALAR, ENV_GATHER_BLOCKS, ENV_TSQR, ENV_JACOBI_FP32, ENV_JACOBI_GENERIC, ENV_RICH_OLD, ENV_NO_DEFLATE, ENV_NO_OA, ENV_SKETCH_SORT, ENV_TALL_OLD, ENV_TABLES_ONE_CTA, ENV_COUNT };
const char* env(EnvSwitch id);
int cuda_status(cudaError_t e, const char* what);

// Stream-ordered scratch allocation (default mempool, release threshold raised
// once so repeated solves reuse the same HBM).
void* scratch_alloc(size_t bytes, cudaStream_t s);
void scratch_free(void* p, cudaStream_t s);

inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <typename T>
struct Scratch {
  T* p = nullptr;
  cudaStream_t s;
  Scratch(size_t n, cudaStream_t st) : s(st) { p = n ? (T*)scratch_alloc(n * sizeof(T), st) : nullptr; }
  ~Scratch() { if (p) scratch_free(p, s); }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
};

}  // namespace ks

#define KS_TRY_CUDA(expr)                                         \
  do {                                                            \
    cudaError_t _e = (expr);                                      \
    if (_e != cudaSuccess) return ks::cuda_status(_e, #expr);     \
  } while (0)

#define KS_CHECK_LAUNCH() KS_TRY_CUDA(cudaGetLastError())

#define KS_REQUIRE(cond, code, ...)     \
  do {                                  \
    if (!(cond)) {                      \
      ks::set_error(__VA_ARGS__);       \
      return (code);                    \
    }                                   \
  } while (0)

// ---- device helpers -------------------------------------------------------

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum in a fixed order (deterministic).  `red` needs blockDim/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// Block-wide maximum (same pattern as block_sum).
__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// Asynchronous global->shared copies (LDGSTS): issued back to back without touching registers,
// so the L2/HBM latencies of a whole staging loop overlap.  (Plain load/store staging loops get
// serialised by ptxas under register pressure.)  Zero-fill variant for out-of-range elements.
__device__ __forceinline__ void ks_cp_async8(void* dst, const void* src, bool valid = true) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void ks_cp_async16z(void* dst, const void* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void ks_cp_async4(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void ks_cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__host__ __device__ __forceinline__ int64_t ks_min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t ks_max64(int64_t a, int64_t b) { return a > b ? a : b; }

static inline unsigned ceil_div_u(long long a, long long b) { return (unsigned)((a + b - 1) / b); }
