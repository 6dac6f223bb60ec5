// Does the stencil's access shape cost DRAM bandwidth?  Copy 16384 x 16384 x 4
// doubles row by row like the pair kernel: each warp owns 64 columns of a strip
// of rows and per row reads/writes (a) 4 variable rows 128 KB apart
// ("row-interleaved SoA", the library's layout) or (b) one contiguous 2 KB
// chunk (pair-interleaved [j][i/2][v][2]).  Read+write bytes / time.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NX = 16384, NY = 16384, NV = 4, ROWS = 128;
__global__ void soa_rows(const double2* __restrict__ in, double2* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * 4 + (threadIdx.x >> 5));
  const int c = warp * 64 + 2 * lane;
  if (c >= NX) return;
  const long long rs = (long long)NX * NV;  // doubles per cell row
  for (int r = blockIdx.y * ROWS; r < (blockIdx.y + 1) * ROWS; ++r) {
    double2 v[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = in[(r * rs + (long long)k * NX + c) / 2];
#pragma unroll
    for (int k = 0; k < NV; ++k) out[(r * rs + (long long)k * NX + c) / 2] = v[k];
  }
}
__global__ void pair_rows(const double2* __restrict__ in, double2* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * 4 + (threadIdx.x >> 5));
  const int c = warp * 64 + 2 * lane;
  if (c >= NX) return;
  const long long rs = (long long)NX * NV;
  for (int r = blockIdx.y * ROWS; r < (blockIdx.y + 1) * ROWS; ++r) {
    double2 v[NV];
    const long long base = r * rs + (long long)c * NV;  // this lane's 2 cells x 4 vars, contiguous
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = in[base / 2 + k];
#pragma unroll
    for (int k = 0; k < NV; ++k) out[base / 2 + k] = v[k];
  }
}
int main() {
  const size_t n = (size_t)NX * NY * NV;
  double2 *a, *b;
  cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8); cudaMemset(b, 0, n * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  dim3 grid(NX / 64 / 4, NY / ROWS);
  for (int variant = 0; variant < 2; ++variant) {
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (variant == 0) soa_rows<<<grid, 128>>>(a, b); else pair_rows<<<grid, 128>>>(a, b);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep && ms < best) best = ms;
    }
    printf("%-40s %8.1f GB/s\n", variant == 0 ? "row-interleaved SoA (4 streams/warp)" : "pair-interleaved (1 stream/warp)",
           2.0 * n * 8 / (best * 1e-3) / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
