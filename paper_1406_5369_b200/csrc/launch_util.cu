// launch_util.cu — see launch_util.h.
#include "launch_util.h"

#include <map>
#include <mutex>
#include <tuple>

namespace mg {

static std::mutex g_mu;

int sm_count() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  static std::map<int, int> cache;
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms < 1) sms = 1;
  cache[dev] = sms;
  return sms;
}

int resident_ctas(const void* kernel, int threads, int smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = sm_count();
  std::lock_guard<std::mutex> lk(g_mu);
  static std::map<std::tuple<int, const void*, int, int>, int> cache;
  const auto key = std::make_tuple(dev, kernel, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
  const int r = (occ < 1 ? 1 : occ) * sms;
  cache[key] = r;
  return r;
}

int per_device_once(const void* key, int (*probe)()) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  static std::map<std::pair<int, const void*>, int> cache;
  const auto k = std::make_pair(dev, key);
  auto it = cache.find(k);
  if (it != cache.end()) return it->second;
  const int r = probe();
  cache[k] = r;
  return r;
}

}  // namespace mg
