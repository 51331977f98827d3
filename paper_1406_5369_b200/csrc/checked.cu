// checked.cu — guard-banded allocations of the CHECKED build (see checked.h).  Compiled into
// the product library as an empty translation unit.
#ifdef MG_CHECKED
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <vector>

namespace mg {

static constexpr size_t kGuard = 64 * 1024;
static constexpr unsigned char kPattern = 0xA5;
static std::mutex g_mu;
static std::map<void*, std::pair<char*, size_t>> g_live;  // user pointer -> (base, bytes)
static long long g_failures = 0;

static bool guard_ok(const char* base, size_t bytes) {
  std::vector<unsigned char> h(2 * kGuard);
  if (cudaMemcpy(h.data(), base, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(h.data() + kGuard, base + kGuard + bytes, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  for (unsigned char c : h)
    if (c != kPattern) return false;
  return true;
}

cudaError_t checked_malloc(void** p, size_t bytes) {
  char* base = nullptr;
  cudaError_t e = (cudaMalloc)(reinterpret_cast<void**>(&base), bytes + 2 * kGuard);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemset(base, kPattern, kGuard)) != cudaSuccess ||
      (e = cudaMemset(base + kGuard + bytes, kPattern, kGuard)) != cudaSuccess) {
    (cudaFree)(base);
    return e;
  }
  *p = base + kGuard;
  std::lock_guard<std::mutex> lk(g_mu);
  g_live[*p] = {base, bytes};
  return cudaSuccess;
}

cudaError_t checked_free(void* p) {
  if (!p) return cudaSuccess;
  std::pair<char*, size_t> a;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_live.find(p);
    if (it == g_live.end()) return (cudaFree)(p);
    a = it->second;
    g_live.erase(it);
  }
  cudaDeviceSynchronize();
  if (!guard_ok(a.first, a.second)) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_failures++;
  }
  return (cudaFree)(a.first);
}

}  // namespace mg

// number of corrupted guard bands: of the buffers freed so far plus a scan of the live ones
extern "C" long long mg_checked_guard_failures(void) {
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(mg::g_mu);
  long long n = mg::g_failures;
  for (auto& kv : mg::g_live)
    if (!mg::guard_ok(kv.second.first, kv.second.second)) n++;
  return n;
}
#endif
