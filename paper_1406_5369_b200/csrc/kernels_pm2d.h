// kernels_pm2d.h — launchers of the warp-marching kernels for 2D levels
// (kernels_pm2d.cu).  Reached through the pm:: launchers, which dispatch on
// Geom::three_d.
#pragma once
#include "mg_common.cuh"

namespace mg {
namespace pm2 {
bool supported(const Geom& g, int min_nx);
template <typename T>
cudaError_t launch_sweep(const Geom& g, const Coef<T>& c, bool rbgs, const T* uin, const T* f, T* uout, bool zero_in,
                         cudaStream_t st, double* partial, int* npartial);
template <typename T>
int sweep_partials(const Geom& g, bool rbgs);
// K (2, or 3 in FP32) omega-Jacobi sweeps in one pass: bitwise equal to K single sweeps.
// partial != nullptr: also the norm partials of uin's residual (*npartial of them; not
// with zero_in).  e != nullptr: the passes start from uin + P e (coarse correction e on
// level *gc fused in; uin is not modified).  fc != nullptr (rr_fusable(K)): also the
// full-weighting restriction of the result's residual into fc on level *gc (as
// launch_resid_restrict; not with e)
template <typename T>
cudaError_t launch_jacobi_k(const Geom& g, const Coef<T>& c, int K, const T* uin, const T* f, T* uout, bool zero_in,
                            cudaStream_t st, double* partial = nullptr, int* npartial = nullptr,
                            const T* e = nullptr, const Geom* gc = nullptr, T* fc = nullptr);
// whether a K-sweep pass can carry the residual + restriction (r exact on the stored columns)
template <typename T>
bool rr_fusable(int K);
template <typename T>
cudaError_t launch_norm(const Geom& g, const Coef<T>& c, const T* u, const T* f, double* partial, int* npartial,
                        cudaStream_t st);
template <typename T>
int norm_partials(const Geom& g);
template <typename T>
cudaError_t launch_resid_restrict(const Geom& gf, const Geom& gc, const Coef<T>& c, const T* u, const T* f, T* fc,
                                  cudaStream_t st);
// uout = uin + P e (in place when uout == uin; out of place, uout's boundary holds the data)
template <typename T>
cudaError_t launch_prolong(const Geom& gf, const Geom& gc, const T* e, const T* uin, T* uout, cudaStream_t st);
}  // namespace pm2
}  // namespace mg
