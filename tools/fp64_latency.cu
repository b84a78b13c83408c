// Calibration: dependent-chain latency of FP64 ops (DFMA, DADD, DMUL, sqrt, div, rcp) on one warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

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
  return 0;
}
