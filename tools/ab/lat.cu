// microbenchmarks: dependent-chain latencies on this GPU (one thread)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, const double* gsrc, int n) {
  __shared__ double sh[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = 1.0 + i * 1e-9;
  __syncthreads();
  if (threadIdx.x) return;
  double a = out[0], b = out[1];
  long long t0 = clock64();
  for (int i = 0; i < n; i++) { a = __dadd_rn(a, b); a = __dadd_rn(a, b); a = __dadd_rn(a, b); a = __dadd_rn(a, b); }
  long long t1 = clock64();
  for (int i = 0; i < n; i++) { a = __dmul_rn(a, b); a = __dmul_rn(a, b); a = __dmul_rn(a, b); a = __dmul_rn(a, b); }
  long long t2 = clock64();
  double bb = 1.0000001 + b; for (int i = 0; i < n; i++) { a = __ddiv_rn(a, bb); }
  long long t3 = clock64();
  // dependent LDS chain (index from loaded value)
  int idx = 0;
  for (int i = 0; i < n; i++) { idx = (int)sh[idx & 1023] & 1023; idx = (int)sh[idx] & 1023; }
  long long t4 = clock64();
  // generic pointer to shared
  volatile double* gp = (volatile double*)(out[2] > 0 ? (double*)sh : (double*)gsrc);
  for (int i = 0; i < n; i++) { idx = (int)gp[idx & 1023] & 1023; idx = (int)gp[idx] & 1023; }
  long long t5 = clock64();
  float fa = (float)a, fb = (float)b;
  for (int i = 0; i < n; i++) { fa = __fadd_rn(fa, fb); fa = __fadd_rn(fa, fb); fa = __fadd_rn(fa, fb); fa = __fadd_rn(fa, fb); }
  long long t6 = clock64();
  out[3] = a + idx + fa;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
}
int main() {
  double h[4] = {1.0, 1e-17, 1.0, 0}; double* d; long long* c; double* g;
  cudaMalloc(&d, 32); cudaMalloc(&c, 64); cudaMalloc(&g, 8192);
  cudaMemcpy(d, h, 32, cudaMemcpyHostToDevice);
  const int n = 1000;
  for (int rep = 0; rep < 2; rep++) {
    k<<<1, 128>>>(d, c, g, n);
    long long hc[6]; cudaMemcpy(hc, c, 48, cudaMemcpyDeviceToHost);
    printf("DADD %.1f  DMUL %.1f  DDIV %.1f  LDS %.1f  LD.generic->smem %.1f  FADD %.1f cycles\n", hc[0] / (4.0 * n), hc[1] / (4.0 * n), hc[2] / (1.0 * n),
           hc[3] / (2.0 * n), hc[4] / (2.0 * n), hc[5] / (4.0 * n));
  }
  return 0;
}
