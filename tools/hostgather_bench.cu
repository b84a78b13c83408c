// Random 8-byte reads from page-locked (mapped) host memory: how fast can 38k sampled b entries be
// gathered over PCIe, by loads in flight per thread and block size.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hostgather_bench hostgather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

template <int ILP>
__global__ void gather_kernel(const double* __restrict__ b, const int64_t* __restrict__ idx, int64_t s,
                              double* __restrict__ out) {
  const int64_t q0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * ILP;
  double v[ILP];
#pragma unroll
  for (int k = 0; k < ILP; k++) v[k] = q0 + k < s ? b[idx[q0 + k]] : 0.0;
#pragma unroll
  for (int k = 0; k < ILP; k++)
    if (q0 + k < s) out[q0 + k] = v[k];
}

template <int ILP>
float run(const double* b, const int64_t* idx, int64_t s, double* out, int bs) {
  const int64_t thr = (s + ILP - 1) / ILP;
  const int grid = (int)((thr + bs - 1) / bs);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 7; r++) {
    cudaEventRecord(e0);
    gather_kernel<ILP><<<grid, bs>>>(b, idx, s, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;
  }
  return best * 1e3f;
}

int main() {
  const int64_t n2 = 16384LL * 16384LL, s = 38045;
  double* hb;
  if (cudaHostAlloc(&hb, n2 * 8, cudaHostAllocMapped) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  for (int64_t i = 0; i < n2; i += 512) hb[i] = 1.0;  // touch every page
  std::vector<int64_t> hidx(s);
  uint64_t x = 88172645463325252ULL;
  for (auto& v : hidx) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = (int64_t)(x % (uint64_t)n2); }
  int64_t* didx; double* dout; double* db;
  cudaMalloc(&didx, s * 8); cudaMalloc(&dout, s * 8);
  cudaMemcpy(didx, hidx.data(), s * 8, cudaMemcpyHostToDevice);
  cudaHostGetDevicePointer(&db, hb, 0);
  for (int bs : {128, 256, 512}) {
    printf("{\"block\": %d, \"ilp1_us\": %.1f, \"ilp2_us\": %.1f, \"ilp4_us\": %.1f, \"ilp8_us\": %.1f}\n", bs,
           run<1>(db, didx, s, dout, bs), run<2>(db, didx, s, dout, bs), run<4>(db, didx, s, dout, bs),
           run<8>(db, didx, s, dout, bs));
  }
  // sorted indices (same pages visited in address order)
  std::vector<int64_t> sidx = hidx;
  std::qsort(sidx.data(), s, 8, [](const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b; return (x > y) - (x < y); });
  cudaMemcpy(didx, sidx.data(), s * 8, cudaMemcpyHostToDevice);
  printf("{\"sorted\": true, \"block\": 128, \"ilp1_us\": %.1f, \"ilp4_us\": %.1f}\n", run<1>(db, didx, s, dout, 128),
         run<4>(db, didx, s, dout, 128));
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
