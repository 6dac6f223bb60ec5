// HBM copy variants on one B200: what access pattern reaches the copy roof
// (MEASURED_PEAKS hbm_gbs = torch copy_).  Read+write bytes / time.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void copy_v2(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void copy_v2_cs(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}
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
// double (8 B) per lane, like the stencil's rows
__global__ void copy_d(const double* __restrict__ a, double* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  size_t n = (size_t)1 << 29;  // 8 GiB per buffer (double2)
  double2 *a, *b;
  cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep && ms < best) best = ms;
    }
    printf("%-28s %8.1f GB/s\n", name, 2.0 * n * 16 / (best * 1e-3) / 1e9);
  };
  for (int g : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
    char nm[64];
    snprintf(nm, 64, "v2 grid %d", g); run(nm, [&] { copy_v2<<<g, 256>>>(a, b, n); });
    snprintf(nm, 64, "v2 .cs grid %d", g); run(nm, [&] { copy_v2_cs<<<g, 256>>>(a, b, n); });
    snprintf(nm, 64, "v2 unroll4 grid %d", g); run(nm, [&] { copy_unroll<4><<<g, 256>>>(a, b, n); });
    snprintf(nm, 64, "d grid %d", g); run(nm, [&] { copy_d<<<g, 256>>>((const double*)a, (double*)b, 2 * n); });
  }
  run("cudaMemcpy D2D", [&] { cudaMemcpyAsync(b, a, n * 16, cudaMemcpyDeviceToDevice); });
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
