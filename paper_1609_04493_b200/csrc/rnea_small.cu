// rnea_small.cu -- dispatch of the register-resident THREAD kernel (rnea_small.cuh)
// by link count; the kernels are instantiated in rnea_small_f64.cu / _f32a.cu / _f32b.cu.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_small.h"

namespace rd {

bool small_kernel_has_n(int n, bool fp64, int64_t B) {
  if (n < 1) return false;
  if (!fp64) return n <= small_max_n<float>() && !small_f32_cliff(n);
  return n <= kSmallMaxN64Any || (n <= small_max_n<double>() && B <= kSmallCapBatch);
}

template <typename T, int N>
static cudaError_t dispatch_n(int n, const LinkDHc<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                              const T* qd, const T* qdd, T* tau, cudaStream_t st, uint32_t prism,
                              const StateBoundary<T>* sb) {
  if (n == N) return small_launch_n<T, N>(L_host, bnd, B, q, qd, qdd, tau, st, prism, sb);
  if constexpr (N > 1) return dispatch_n<T, N - 1>(n, L_host, bnd, B, q, qd, qdd, tau, st, prism, sb);
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t launch_rnea_small(int n, const LinkDHc<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                              const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                              uint32_t prism_mask, const StateBoundary<T>* sb) {
  if (n < 1 || n > small_max_n<T>()) return cudaErrorInvalidValue;
  ++*launches;
  return dispatch_n<T, small_max_n<T>()>(n, L_host, bnd, B, q, qd, qdd, tau, st, prism_mask, sb);
}
template cudaError_t launch_rnea_small<double>(int, const LinkDHc<double>*, const Boundary<double>&, int64_t,
                                               const double*, const double*, const double*, double*, cudaStream_t,
                                               int*, uint32_t, const StateBoundary<double>*);
template cudaError_t launch_rnea_small<float>(int, const LinkDHc<float>*, const Boundary<float>&, int64_t,
                                              const float*, const float*, const float*, float*, cudaStream_t, int*,
                                              uint32_t, const StateBoundary<float>*);

}  // namespace rd
