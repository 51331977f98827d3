#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double div_rn_via(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double q = __fma_rn(__fma_rn(-b, q0, a), y, q0);
  const double r = __fma_rn(-b, q, a);
  const long long bits = __double_as_longlong(q);
  const int e = (int)((bits >> 52) & 0x7ff);
  if (e > 60 && e < 2040) {
    const double hu = __longlong_as_double((long long)(e - 53) << 52);  // half an ulp of q
    const bool below = (r < 0.0) != (b < 0.0);                         // a / b < q
    const bool pow2 = (bits & 0xfffffffffffffll) == 0;
    const double h = __dmul_rn(below && pow2 ? 0.5 * hu : hu, fabs(b));
    if (h > 0x1p-960 && fabs(r) < h) return q;
  }
  return __ddiv_rn(a, b);
}

__device__ unsigned long long mix(unsigned long long x) { x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x; }
__global__ void k(unsigned long long seed, int mode, unsigned long long* bad, unsigned long long* fallback) {
  unsigned long long id = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  unsigned long long nb = 0, nf = 0;
  for (int it = 0; it < 64; it++) {
    unsigned long long x = mix(seed ^ (id * 64 + it)), z = mix(x + 0x9e3779b97f4a7c15ull);
    double a, b;
    if (mode == 0) {  // random mantissas, exponents in a moderate range
      a = __longlong_as_double((x & 0x800fffffffffffffull) | ((unsigned long long)(1023 - 40 + (x >> 53) % 80) << 52));
      b = __longlong_as_double((z & 0x000fffffffffffffull) | ((unsigned long long)(1023 - 40 + (z >> 53) % 80) << 52));
    } else if (mode == 1) {  // b near powers of two, a near multiples (hard cases)
      a = __longlong_as_double(((x & 0xfull) | (x & 0x8000000000000000ull)) | ((unsigned long long)(1023 + (x >> 60)) << 52)) ;
      b = __longlong_as_double(((z & 0x3ull) ^ ((z >> 2) & 1 ? 0xfffffffffffffull : 0)) | ((unsigned long long)(1023 - 3 + (z >> 61)) << 52));
    } else {  // full exponent range
      a = __longlong_as_double(x); b = __longlong_as_double(z);
      if (!isfinite(a) || !isfinite(b) || b == 0.0) continue;
    }
    double y = __drcp_rn(b);
    double q1 = div_rn_via(a, b, y), q2 = __ddiv_rn(a, b);
    if (__double_as_longlong(q1) != __double_as_longlong(q2) && !(isnan(q1) && isnan(q2))) nb++;
  }
  atomicAdd(bad, nb);
}
int main() {
  unsigned long long *d; cudaMalloc(&d, 16);
  for (int mode = 0; mode < 3; mode++) {
    cudaMemset(d, 0, 16);
    for (int rep = 0; rep < 16; rep++) k<<<4096, 256>>>(rep * 1234567ull + mode, mode, d, d + 1);
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mode %d: %llu pairs, mismatches %llu\n", mode, 16ull * 4096 * 256 * 64, h[0]);
  }
  return 0;
}
