// Sustained HBM copy on one B200: the best copy kernel of tools/copybench.cu
// (4 x double2 per thread, grid-stride) over 2 x 8 GiB, run back to back for
// ~3 s so the GPU settles at its power cap; prints the rate of each 100-copy
// block (read + write bytes / time).  Context for the c3 step kernel's
// sustained roofline fraction, not a peak of record.
#include <cstdio>
#include <cuda_runtime.h>
template <int U>
__global__ void copy_unroll(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t base = (blockIdx.x * (size_t)blockDim.x) * U + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (; base < n; base += stride) {
    double2 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t i = base + u * blockDim.x; if (i < n) r[u] = __ldg(a + i); }
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t i = base + u * blockDim.x; if (i < n) b[i] = r[u]; }
  }
}
int main() {
  const size_t n = (size_t)1 << 29;  // 8 GiB per buffer
  double2 *a, *b;
  if (cudaMalloc(&a, n * sizeof(double2)) != cudaSuccess || cudaMalloc(&b, n * sizeof(double2)) != cudaSuccess) return 1;
  cudaMemset(a, 0, n * sizeof(double2));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const dim3 grid(sms * 8), block(256);
  for (int blk = 0; blk < 12; ++blk) {
    cudaEventRecord(e0);
    for (int k = 0; k < 100; ++k) copy_unroll<4><<<grid, block>>>(k & 1 ? b : a, k & 1 ? a : b, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"block\": %d, \"copy_gbs\": %.1f, \"ms_per_copy\": %.4f}\n", blk, 100.0 * 2 * n * sizeof(double2) / (ms * 1e-3) / 1e9,
           ms / 100);
    fflush(stdout);
  }
  return 0;
}
