// microbenchmark: cost of barrier.cluster (release/acquire) for cluster sizes 1..16, 512 threads
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) k(long long* out, int n, int mode) {
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    if (mode == 0)
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else if (mode == 1)
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
    else
      __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) for (int mode = 0; mode < 3; mode++) {
    cudaLaunchConfig_t c = {}; c.gridDim = dim3(cs); c.blockDim = dim3(512);
    cudaLaunchAttribute a; a.id = cudaLaunchAttributeClusterDimension; a.val.clusterDim.x = cs; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
    c.attrs = &a; c.numAttrs = 1;
    const int n = 2000;
    for (int rep = 0; rep < 2; rep++) cudaLaunchKernelEx(&c, k, d, n, mode);
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("cluster %2d mode %s: %.0f cycles per barrier (%s)\n", cs, mode == 0 ? "release/acquire" : mode == 1 ? "relaxed" : "syncthreads", h / (double)n, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
