// kernels_pm.h — launchers of the plane-marching kernels: TMA-staged tiles for 3D levels
// (kernels_pm.cu), warp-marching strips for 2D levels (kernels_pm2d.cu, dispatched here).
#pragma once
#include "mg_common.cuh"

#include <cuda.h>

namespace mg {
namespace pm {
// cuTensorMapEncodeTiled (through the runtime's driver entry point): element type FP64/FP32,
// dims/strides (bytes, dims 1..rank-1)/box of a rank-`rank` tensor, no swizzle, zero OOB fill
CUresult encode_tiled(CUtensorMap* tm, bool fp64, int rank, const void* base, const unsigned long long* dims,
                      const unsigned long long* strides, const unsigned* box);
// true when a level is large enough for the plane-marching kernels
bool supported(const Geom& g, int min_nx);
// residual partials a sweep writes when `partial` is given (3D levels):
//  SN_INPUT      ||f - A u_in||^2 of every interior node
//  SN_INPUT_RED  the same, red nodes only (RBGS)
//  SN_OUT_BLACK  ||f - A u_out||^2 of the black nodes (RBGS; with SN_INPUT_RED of the next sweep
//                of the same u and f, this is the norm of u_out, node by node bitwise)
enum SweepNorm { SN_INPUT = 1, SN_INPUT_RED = 2, SN_OUT_BLACK = 3 };
// one RBGS (rbgs=true) or Jacobi sweep u_out = S(u_in); zero_in: u_in is taken as 0 (not read)
// partial != nullptr: also write residual partials (`nm`; one per CTA, *npartial of them)
// ecoarse != nullptr: the input is u_in + P ecoarse (prolongation + correction fused, 3D)
template <typename T>
cudaError_t launch_sweep(const Geom& g, const Coef<T>& c, bool rbgs, const T* uin, const T* f, T* uout, bool zero_in,
                         cudaStream_t st, double* partial = nullptr, int* npartial = nullptr,
                         const T* ecoarse = nullptr, const Geom* gcoarse = nullptr, SweepNorm nm = SN_INPUT);
// upper bound of the partials a sweep of level g writes
template <typename T>
int sweep_partials(const Geom& g, bool rbgs);
// exactly the partials a non-fused 3D sweep of level g writes (its CTA count)
template <typename T>
int sweep_items(const Geom& g, bool rbgs);
// fc (coarse interior) = FW(f - A u) ; coarse boundary untouched
template <typename T>
cudaError_t launch_resid_restrict(const Geom& gf, const Geom& gc, const Coef<T>& c, const T* u, const T* f, T* fc,
                                  cudaStream_t st);
// residual-norm partials (one double per CTA); *npartial = count written
template <typename T>
cudaError_t launch_norm(const Geom& g, const Coef<T>& c, const T* u, const T* f, double* partial, int* npartial,
                        cudaStream_t st);
template <typename T>
int norm_partials(const Geom& g);
// u += P e (3D, interior fine nodes)
template <typename T>
cudaError_t launch_prolong(const Geom& gf, const Geom& gc, const T* e, T* u, cudaStream_t st);
}  // namespace pm
}  // namespace mg
