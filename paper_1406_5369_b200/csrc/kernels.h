// kernels.h — host-side launchers of the level-operator kernels.
// Every launcher enqueues exactly one kernel on `st` and returns
// cudaGetLastError().  Templates are instantiated for float and double.
#pragma once
#include "mg_common.cuh"

namespace mg {

// --- op-by-op ("baseline") kernels: one thread per node, any level size ---
template <typename T>
cudaError_t launch_jacobi(const Geom& g, const Coef<T>& c, const T* uin, const T* f, T* uout, cudaStream_t st);
template <typename T>
cudaError_t launch_rbgs_colour(const Geom& g, const Coef<T>& c, T* u, const T* f, int colour, cudaStream_t st);
// one hyperplane i + j + global plane = s of a lexicographic omega-GS sweep (in place)
template <typename T>
cudaError_t launch_gs_lex_plane(const Geom& g, const Coef<T>& c, T* u, const T* f, int s, cudaStream_t st);
// first / last hyperplane index of a level's interior
inline int gs_lex_smin(const Geom& g) { return 1 + (g.three_d ? 1 : 0) + g.p_lo + g.p_glob0; }
inline int gs_lex_smax(const Geom& g) { return (g.nx - 1) + (g.three_d ? g.ny - 1 : 0) + g.p_hi - 1 + g.p_glob0; }
template <typename T>
cudaError_t launch_residual(const Geom& g, const Coef<T>& c, const T* u, const T* f, T* r, cudaStream_t st);
template <typename T>
cudaError_t launch_restrict(const Geom& gf, const Geom& gc, const T* r, T* fc, cudaStream_t st);
template <typename T>
cudaError_t launch_prolong_correct(const Geom& gf, const Geom& gc, const T* e, T* u, cudaStream_t st);
template <typename T>
cudaError_t launch_copy_boundary(const Geom& g, const T* src, T* dst, cudaStream_t st);
// residual-norm partials: one double per block of a fixed decomposition; returns #partials
template <typename T>
int norm_num_partials(const Geom& g);
template <typename T>
cudaError_t launch_norm_partial(const Geom& g, const Coef<T>& c, const T* u, const T* f, double* partial,
                                cudaStream_t st);
cudaError_t launch_norm_final(const double* partial, int n, double* out, cudaStream_t st, bool take_sqrt = true);
cudaError_t launch_norm_combine(const double* sums, int P, double* out, cudaStream_t st);

// --- coarsest level direct solve (Cholesky factor computed once at setup) ---
// A assembled from the stencil (interior unknowns, x fastest), factor L (m x m, row major)
cudaError_t launch_cholesky_factor(const Geom& g, double cx, double cy, double cz, double D, double* L, int m,
                                   int* status, cudaStream_t st);
template <typename T>
cudaError_t launch_coarse_direct(const Geom& g, double D, const double* L, int m, const T* f, T* e, double* work,
                                 cudaStream_t st);

// --- synthetic inputs (SplitMix64 of the global unpadded node index) ---
template <typename T>
cudaError_t launch_workload_fill(const Geom& g, uint64_t seed, double lo, double hi, T* dst, cudaStream_t st);

}  // namespace mg
