// Calibration: cost of a block-wide barrier step (512 threads) with and without a serial
// sqrt/div on one thread between barriers.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void bar_kernel(int steps, int mode, double* out, long long* cyc) {
  __shared__ double buf[2][64];
  __shared__ double piv[2];
  const int tid = threadIdx.x;
  double a = tid * 1e-3 + 1.0;
  long long t0 = clock64();
  for (int k = 0; k < steps; k++) {
    const int b = k & 1;
    if (tid < 64) buf[b][tid] = a;
    if (mode >= 1 && tid == (k & 63)) {
      const double l = sqrt(a + 2.0);
      piv[b] = 1.0 / l;
    }
    __syncthreads();
    const double rl = mode >= 1 ? piv[b] : 1.0;
    if (mode >= 2) {
#pragma unroll
      for (int m = 0; m < 8; m++) a = fma(-(buf[b][(tid + m) & 63] * rl), buf[b][tid & 63], a);
    } else {
      a += buf[b][tid & 63] * rl;
    }
  }
  long long t1 = clock64();
  if (tid == 0) *cyc = (t1 - t0) / steps;
  out[tid] = a;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 8);
  for (int threads : {128, 256, 512, 1024})
    for (int mode = 0; mode < 3; mode++) {
      bar_kernel<<<1, threads>>>(64, mode, out, cyc);
      cudaDeviceSynchronize();
      bar_kernel<<<1, threads>>>(64, mode, out, cyc);
      cudaDeviceSynchronize();
      printf("threads %4d mode %d: %lld cycles/step\n", threads, mode, *cyc);
    }
  return 0;
}
