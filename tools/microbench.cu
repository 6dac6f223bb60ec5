// FP64 pipe and HBM copy microbenchmarks on one B200 (roofline denominators).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void fp64_kernel(double* out, double a, double b, int iters) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = a + threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) x[k] = fma(x[k], b, a);
      if (OP == 1) x[k] = __dadd_rn(x[k], b);
      if (OP == 2) x[k] = __dmul_rn(x[k], b);
    }
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  const char* names[3] = {"DFMA", "DADD", "DMUL"};
  for (int op = 0; op < 3; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (op == 0) fp64_kernel<0><<<blocks, threads>>>(out, 1.0, 0.999999, iters);
      if (op == 1) fp64_kernel<1><<<blocks, threads>>>(out, 1.0, 1e-9, iters);
      if (op == 2) fp64_kernel<2><<<blocks, threads>>>(out, 1.0, 0.999999, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 8;
      if (rep == 1) printf("%s: %.3f T instr/s (%.1f per SM per clock at 1.965 GHz)\n", names[op], ops / ms / 1e9, ops / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  size_t n = (size_t)1 << 28;  // 4 GiB per buffer in double2
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16);
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    copy_kernel<<<148 * 16, 256>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0) printf("copy 2x%.1f GB: %.1f GB/s (read+write)\n", n * 16 / 1e9, 2.0 * n * 16 / (ms * 1e-3) / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
