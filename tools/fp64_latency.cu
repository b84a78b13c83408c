// Calibration: dependent-chain latency of FP64 ops (DFMA, DADD, DMUL, sqrt, div, rcp) on one warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double* c, double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// CHAINS independent accumulators per warp, WARPS warps per block
template <int CHAINS>
__global__ void dmma_kernel(int n, double* out, long long* cyc) {
  double c[CHAINS][4] = {};
  const double a0 = 1e-3 * threadIdx.x, a1 = 2e-3, b0 = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int k = 0; k < CHAINS; k++) dmma(c[k], a0, a1, b0);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = (t1 - t0);
  double s = 0;
  for (int k = 0; k < CHAINS; k++) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DFMA throughput: CH independent chains per thread, W warps
template <int CH>
__global__ void dfma_tp_kernel(int n, double* out, long long* cyc) {
  double a[CH];
#pragma unroll
  for (int k = 0; k < CH; k++) a[k] = threadIdx.x * 1e-9 + k;
  const double b = 1.0000001, c = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
#pragma unroll
    for (int k = 0; k < CH; k++) a[k] = fma(a[k], b, c);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = (t1 - t0);
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; k++) s += a[k];
  out[threadIdx.x] = s;
}

template <int OP>
__global__ void lat_kernel(int n, double x0, double* out, long long* cyc) {
  double a = x0 + threadIdx.x * 1e-9, b = 1.0000001, c = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    if (OP == 0) a = fma(a, b, c);
    if (OP == 1) a = a + c;
    if (OP == 2) a = a * b;
    if (OP == 3) a = sqrt(a) + 1.0;
    if (OP == 4) a = 1.0 / a + 1.0;
    if (OP == 5) a = __drcp_rn(a) + 1.0;
    if (OP == 6) a = rsqrt(a) + 1.0;
    if (OP == 7) { float f = (float)a; a = (double)(f * 1.0000001f + 1e-7f); }
    if (OP == 8) a = __shfl_xor_sync(0xffffffffu, a, 1) + c;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = (t1 - t0);
  out[threadIdx.x] = a;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 8);
  const char* names[] = {"dfma", "dadd", "dmul", "sqrt+add", "div+add", "drcp_rn+add", "rsqrt+add", "f32 fma via cvt",
                         "shfl64+dadd"};
  const int n = 4096;
#define RUN(OP)                                                      \
  lat_kernel<OP><<<1, 32>>>(n, 1.5, out, cyc);                       \
  cudaDeviceSynchronize();                                           \
  lat_kernel<OP><<<1, 32>>>(n, 1.5, out, cyc);                       \
  cudaDeviceSynchronize();                                           \
  printf("%-16s %6.1f cycles/op\n", names[OP], (double)*cyc / n);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8)
#define DM(CH, W)                                                              \
  dmma_kernel<CH><<<1, 32 * W>>>(1024, out, cyc);                              \
  cudaDeviceSynchronize();                                                     \
  dmma_kernel<CH><<<1, 32 * W>>>(1024, out, cyc);                              \
  cudaDeviceSynchronize();                                                     \
  printf("dmma chains %d warps %2d: %6.1f cycles per dmma-step (per warp), %5.2f cycles/dmma/SM\n", CH, W, \
         (double)*cyc / 1024, (double)*cyc / 1024 / (CH * W));
  DM(1, 1) DM(2, 1) DM(4, 1) DM(8, 1) DM(1, 4) DM(4, 4) DM(1, 8) DM(4, 8) DM(8, 8) DM(4, 16)
#define TP(CH, W)                                                              \
  dfma_tp_kernel<CH><<<1, 32 * W>>>(4096, out, cyc);                           \
  cudaDeviceSynchronize();                                                     \
  dfma_tp_kernel<CH><<<1, 32 * W>>>(4096, out, cyc);                           \
  cudaDeviceSynchronize();                                                     \
  printf("dfma chains %d warps %2d: %6.2f cycles per warp-dfma per SM (%.1f lanes/clk)\n", CH, W,   \
         (double)*cyc / (4096.0 * CH * W), 32.0 * 4096.0 * CH * W / (double)*cyc);
  TP(8, 1) TP(8, 4) TP(8, 8) TP(8, 16) TP(8, 32)
  return 0;
}
