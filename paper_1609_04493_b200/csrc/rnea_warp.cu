// rnea_warp.cu -- placeholder; replaced by the warp-scan strategy.
#include <cuda_runtime.h>
#include "rd_internal.h"
namespace rd {
template <typename T>
cudaError_t launch_rnea_warp(int, const LinkConst<T>*, const Boundary<T>&, int64_t, const T*, const T*, const T*,
                             T*, cudaStream_t, int*, bool* supported) {
  *supported = false;
  return cudaSuccess;
}
template cudaError_t launch_rnea_warp<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                              const double*, const double*, const double*, double*, cudaStream_t,
                                              int*, bool*);
template cudaError_t launch_rnea_warp<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                             const float*, const float*, const float*, float*, cudaStream_t, int*,
                                             bool*);
}  // namespace rd
