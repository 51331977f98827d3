// standalone TMA box-load probe (debug tool)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_1406_5369_b200/csrc/tma.cuh"
using namespace mg;
template <typename T>
__global__ void k(const __grid_constant__ CUtensorMap tm, int bx, int by, T* out, int x0, int y0, int z0) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = (uint64_t*)(sm + 65536);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) { mbar_expect_tx(bar, bx * by * sizeof(T)); tma_load_3d(sm, &tm, x0, y0, z0, bar); }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < bx * by; i += blockDim.x) out[i] = ((T*)sm)[i];
}
template <typename T>
int run(int bx, int by, int nx, int rows, int planes, int pitch, int dtype_override = -1, int c0 = -2) {
  T* g; cudaMalloc(&g, sizeof(T) * pitch * rows * planes);
  T* h = (T*)malloc(sizeof(T) * pitch * rows * planes);
  for (int i = 0; i < pitch * rows * planes; i++) h[i] = (T)i;
  cudaMemcpy(g, h, sizeof(T) * pitch * rows * planes, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t str[2] = {(cuuint64_t)(pitch * sizeof(T)), (cuuint64_t)(pitch * rows * sizeof(T))};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
  CUtensorMapDataType dty = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  if (dtype_override >= 0) dty = (CUtensorMapDataType)dtype_override;
  CUresult r = cuTensorMapEncodeTiled(&tm, dty,
      3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  T* out; cudaMalloc(&out, sizeof(T) * bx * by);
  cudaFuncSetAttribute(k<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
  k<T><<<1, 128, 65536 + 64>>>(tm, bx, by, out, c0, c0, 1);
  cudaError_t e = cudaDeviceSynchronize();
  T* ho = (T*)malloc(sizeof(T) * bx * by);
  int bad = -1;
  if (e == cudaSuccess) {
    cudaMemcpy(ho, out, sizeof(T) * bx * by, cudaMemcpyDeviceToHost);
    bad = 0;
    for (int y = 0; y < by; y++) for (int x = 0; x < bx; x++) {
      int gx = x + c0, gy = y + c0;
      T ref = (gx >= 0 && gx < nx && gy >= 0 && gy < rows) ? (T)(1 * pitch * rows + gy * pitch + gx) : (T)0;
      if (ho[y * bx + x] != ref) bad++;
    }
  }
  printf("esz=%d box=%dx%d encode=%d launch=%s bad=%d\n", (int)sizeof(T), bx, by, (int)r, cudaGetErrorString(e), bad);
  return e != cudaSuccess;
}
int main(int argc, char** argv) {
  int which = atoi(argv[1]);
  if (which == 0) run<double>(68, 12, 65, 65, 65, 80);
  if (which == 1) run<float>(68, 12, 65, 65, 65, 96);
  if (which == 2) run<float>(72, 12, 65, 65, 65, 96);
  if (which == 3) run<float>(64, 12, 65, 65, 65, 96);
  if (which == 4) run<float>(68, 12, 65, 65, 65, 128);
  if (which == 5) run<float>(132, 12, 129, 129, 65, 160);
  if (which == 6) run<float>(68, 12, 65, 65, 65, 96, CU_TENSOR_MAP_DATA_TYPE_UINT32);
  if (which == 7) run<float>(68, 12, 65, 65, 65, 96, CU_TENSOR_MAP_DATA_TYPE_INT32);
  if (which == 8) run<float>(68, 12, 65, 65, 65, 96, -1, 0);
  if (which == 10) run<float>(68, 12, 65, 65, 65, 96, -1, -4);
  if (which == 11) run<float>(68, 12, 65, 65, 65, 96, -1, 2);
  if (which == 12) run<float>(68, 12, 65, 65, 65, 96, -1, 1);
  if (which == 13) run<double>(68, 12, 65, 65, 65, 80, -1, -1);
  if (which == 14) run<float>(68, 12, 65, 65, 65, 96, -1, -1);
  if (which == 9) run<double>(68, 12, 65, 65, 65, 80, CU_TENSOR_MAP_DATA_TYPE_UINT64);
  return 0;
}
