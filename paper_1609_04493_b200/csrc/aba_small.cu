// aba_small.cu -- dispatch of the register-resident ABA kernel (aba_small.cuh) by
// link count; the kernels are instantiated in aba_small_f64.cu / aba_small_f32.cu.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"

namespace rd {

// Longest chain per precision, measured against the workspace kernel
// (profiles/r02/ab_aba_small_long.csv, device time at 1e5 / 1e6 states): fp64 n = 16
// 54.9 / 523 vs 65.8 / 556 us; fp32 n = 18 32.1 / 282 vs 49.3 / 409 us, n = 20
// 48.5 / 454 vs 54.6 / 452 us, n = 22 loses (80 / 797 vs 60 / 495 us: spills).
template <typename T>
constexpr int aba_small_max_n() { return sizeof(T) == 8 ? 16 : 20; }

template <typename T, int N>
cudaError_t aba_small_launch_n(const LinkDH<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                               const T* qd, const T* tau, T* qdd, cudaStream_t st, int32_t* status,
                               uint32_t prism, const StateBoundary<T>* sb);

bool aba_small_has_n(int n, bool fp64) {
  return n >= 1 && n <= (fp64 ? aba_small_max_n<double>() : aba_small_max_n<float>());
}

template <typename T, int N>
static cudaError_t dispatch_n(int n, const LinkDH<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                              const T* qd, const T* tau, T* qdd, cudaStream_t st, int32_t* status, uint32_t prism,
                              const StateBoundary<T>* sb) {
  if (n == N) return aba_small_launch_n<T, N>(L_host, bnd, B, q, qd, tau, qdd, st, status, prism, sb);
  if constexpr (N > 1) return dispatch_n<T, N - 1>(n, L_host, bnd, B, q, qd, tau, qdd, st, status, prism, sb);
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t launch_aba_small(int n, const LinkDH<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                             const T* qd, const T* tau, T* qdd, cudaStream_t st, int* launches, int32_t* status,
                             uint32_t prism_mask, const StateBoundary<T>* sb) {
  if (n < 1 || n > aba_small_max_n<T>()) return cudaErrorInvalidValue;
  ++*launches;
  return dispatch_n<T, aba_small_max_n<T>()>(n, L_host, bnd, B, q, qd, tau, qdd, st, status, prism_mask, sb);
}
template cudaError_t launch_aba_small<double>(int, const LinkDH<double>*, const Boundary<double>&, int64_t,
                                              const double*, const double*, const double*, double*, cudaStream_t,
                                              int*, int32_t*, uint32_t, const StateBoundary<double>*);
template cudaError_t launch_aba_small<float>(int, const LinkDH<float>*, const Boundary<float>&, int64_t,
                                             const float*, const float*, const float*, float*, cudaStream_t, int*,
                                             int32_t*, uint32_t, const StateBoundary<float>*);

}  // namespace rd
