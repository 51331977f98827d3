// launch_util.h — per-kernel launch facts shared by the launchers, cached thread-safely
// (several solvers may launch from several host threads, e.g. the loopback ranks).
#pragma once
#include <cuda_runtime.h>

namespace mg {
// multiprocessors of the current device
int sm_count();
// CTAs of `kernel` (`threads` per CTA, `smem` dynamic bytes) resident on the whole current
// device; opts the kernel in to `smem` > 48 KB first
int resident_ctas(const void* kernel, int threads, int smem);
// once per (current device, key): run probe() (which may set function attributes: those are
// per device context) and cache its result
int per_device_once(const void* key, int (*probe)());
}  // namespace mg
