// FP64 peak microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64) issue throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m16n8k4_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = 0.5, b0 = 0.25;
  double c[4][4];
#pragma unroll
  for (int j = 0; j < 4; j++)
#pragma unroll
    for (int i = 0; i < 4; i++) c[j][i] = 0.0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a0), "d"(a1), "d"(b0));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; j++)
#pragma unroll
    for (int i = 0; i < 4; i++) s += c[j][i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m16n8k16_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; i++) b[i] = 0.5 + i;
  double c[4][4];
#pragma unroll
  for (int j = 0; j < 4; j++)
#pragma unroll
    for (int i = 0; i < 4; i++) c[j][i] = 0.0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; j++)
#pragma unroll
    for (int i = 0; i < 4; i++) s += c[j][i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m8n8k4_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, b0 = 0.25;
  double c[4][2];
#pragma unroll
  for (int j = 0; j < 4; j++) { c[j][0] = 0; c[j][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a0), "d"(b0));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int sustained(double seconds) {
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 4, bs = 256, iters = 4000;
  const double flops1 = 2.0 * 16 * 8 * 4 * 4 * iters * (double)grid * (bs / 32);
  dmma_m16n8k4_kernel<<<grid, bs>>>(out, 100); CK(cudaDeviceSynchronize());
  int launches = 0; float total_ms = 0;
  cudaEventRecord(e0);
  while (total_ms < seconds * 1e3) {
    for (int i = 0; i < 20; i++) dmma_m16n8k4_kernel<<<grid, bs>>>(out, iters);
    launches += 20;
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&total_ms, e0, e1);
  }
  printf("{\"kind\": \"dmma_sustained\", \"seconds\": %.2f, \"tflops\": %.3f}\n", total_ms / 1e3,
         flops1 * launches / (total_ms * 1e-3) / 1e12);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1) return sustained(atof(argv[1]));
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  for (int bs : {128, 256, 512}) for (int per_sm : {1, 2, 4, 8}) {
    int iters = 20000; int grid = sms * per_sm;
    dfma_kernel<<<grid, bs>>>(out, 100, 0.999, 1e-3);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_kernel<<<grid, bs>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)grid * bs;
    printf("{\"kind\": \"dfma\", \"block\": %d, \"grid\": %d, \"tflops\": %.3f}\n", bs, grid, flops / ms / 1e9);
  }
  for (int bs : {128, 256, 512}) for (int per_sm : {1, 2, 4}) {
    int iters = 4000; int grid = sms * per_sm;
    dmma_m16n8k4_kernel<<<grid, bs>>>(out, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_m16n8k4_kernel<<<grid, bs>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 4 * 4 * iters * (double)grid * (bs / 32);
    printf("{\"kind\": \"dmma_m16n8k4\", \"block\": %d, \"grid\": %d, \"tflops\": %.3f}\n", bs, grid, flops / ms / 1e9);
  }
  for (int bs : {128, 256, 512}) for (int per_sm : {1, 2, 4}) {
    int iters = 1000; int grid = sms * per_sm;
    dmma_m16n8k16_kernel<<<grid, bs>>>(out, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_m16n8k16_kernel<<<grid, bs>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 4 * iters * (double)grid * (bs / 32);
    printf("{\"kind\": \"dmma_m16n8k16\", \"block\": %d, \"grid\": %d, \"tflops\": %.3f}\n", bs, grid, flops / ms / 1e9);
  }
  for (int bs : {128, 256}) for (int per_sm : {2, 4}) {
    int iters = 4000; int grid = sms * per_sm;
    dmma_m8n8k4_kernel<<<grid, bs>>>(out, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_m8n8k4_kernel<<<grid, bs>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 4 * iters * (double)grid * (bs / 32);
    printf("{\"kind\": \"dmma_m8n8k4\", \"block\": %d, \"grid\": %d, \"tflops\": %.3f}\n", bs, grid, flops / ms / 1e9);
  }
  {
    size_t n = (size_t)1 << 27;  // 2 GiB per buffer (double2 = 16 B)
    double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    cudaMemset(a, 0, n * 16);
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0);
      copy_kernel<<<sms * 8, 512>>>(a, b, n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"kind\": \"copy\", \"gbs\": %.1f}\n", 2.0 * n * 16 / ms / 1e6);
    }
  }
  return 0;
}
