// HBM probe: in-place read-modify-write (u += c) vs out-of-place (out = in + c), 16-byte vectors,
// 1.08 GB FP64 arrays, grid = 4 x 148 x 8 CTAs of 256 threads, grid-stride.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void inplace(double2* u, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double2 v = u[i];
    v.x += 1.0;
    v.y += 1.0;
    u[i] = v;
  }
}
__global__ void outplace(const double2* __restrict__ a, double2* __restrict__ b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double2 v = a[i];
    v.x += 1.0;
    v.y += 1.0;
    b[i] = v;
  }
}
int main() {
  const long long n = 513LL * 513 * 513 / 2;  // double2 elements ~ 1.08 GB
  double2 *a, *b;
  cudaMalloc(&a, n * sizeof(double2));
  cudaMalloc(&b, n * sizeof(double2));
  cudaMemset(a, 0, n * sizeof(double2));
  cudaMemset(b, 0, n * sizeof(double2));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * 8 * 4;
  for (int rep = 0; rep < 2; rep++) {
    for (int mode = 0; mode < 2; mode++) {
      for (int w = 0; w < 3; w++) mode ? outplace<<<grid, 256>>>(a, b, n) : inplace<<<grid, 256>>>(a, n);
      cudaEventRecord(e0);
      for (int k = 0; k < 20; k++) mode ? outplace<<<grid, 256>>>(a, b, n) : inplace<<<grid, 256>>>(a, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 20;
      printf("%s %.4f ms %.0f GB/s\n", mode ? "out-of-place" : "in-place", ms, 2.0 * n * 16 / ms / 1e6);
    }
  }
  return 0;
}
