// checked.h — the CHECKED build (make checked -> libmgb200_checked.so, -DMG_CHECKED): the
// substitute for compute-sanitizer, which is closed on this pool.  Not part of
// the product library: without MG_CHECKED this header declares nothing.
//  - every device buffer the library allocates gets guard bands of kGuard bytes on both sides,
//    filled with a pattern and verified when the buffer is freed and by
//    mg_checked_guard_failures() (catches out-of-bounds writes of every kernel into the
//    library's own arrays; the tests guard the caller's arrays themselves);
//  - mbarrier waits are bounded and trap instead of spinning forever (tma.cuh), so a broken
//    TMA/mbarrier ring shows as a CUDA error instead of a hung GPU.
#pragma once
#ifdef MG_CHECKED
#include <cuda_runtime.h>

#include <cstddef>

namespace mg {
cudaError_t checked_malloc(void** p, size_t bytes);
cudaError_t checked_free(void* p);
}  // namespace mg

#define cudaMalloc(p, n) ::mg::checked_malloc(reinterpret_cast<void**>(p), (n))
#define cudaFree(p) ::mg::checked_free(reinterpret_cast<void*>(p))
#endif
