// Grid-wide barrier cost on B200: cooperative_groups grid.sync() vs a release/acquire counter barrier.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync_bench gridsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void cg_sync_kernel(int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// monotone counter barrier: arrival i of round r waits until counter >= (r+1)*G
__global__ void counter_sync_kernel(int iters, unsigned* counter, long long* out) {
  const unsigned G = gridDim.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
      const unsigned target = (unsigned)(i + 1) * G;
      while (ld_acquire(counter) < target) {
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* out;
  unsigned* counter;
  cudaMalloc(&out, 8);
  cudaMalloc(&counter, 4);
  int iters = 1000;
  for (int rep = 0; rep < 2; rep++) {
    void* a1[] = {&iters, &out};
    cudaLaunchCooperativeKernel((void*)cg_sync_kernel, sms, 256, a1, 0, 0);
    long long h;
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("{\"kind\": \"cg_grid_sync\", \"ctas\": %d, \"cycles_per_sync\": %.0f}\n", sms, (double)h / iters);
    cudaMemset(counter, 0, 4);
    void* a2[] = {&iters, &counter, &out};
    cudaLaunchCooperativeKernel((void*)counter_sync_kernel, sms, 256, a2, 0, 0);
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("{\"kind\": \"counter_sync\", \"ctas\": %d, \"cycles_per_sync\": %.0f}\n", sms, (double)h / iters);
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
