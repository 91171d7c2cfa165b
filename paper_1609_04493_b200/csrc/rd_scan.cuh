// rd_scan.cuh -- warp-level scan building blocks shared by the scan kernels
// (product path): composition of affine maps x -> L x + b (6x6 L) across lanes.
#pragma once
#include "rd_internal.h"

namespace rd {

// (L, b) := (L, b) o (Lp, bp) = (L Lp, L bp + b) with (Lp, bp) of lane `src`;
// every lane takes part in the shuffles, `take` selects who keeps the result.
template <typename T, bool DOWN>
__device__ __forceinline__ void compose_shfl(T (&Lm)[36], T (&bv)[6], int d, bool take) {
  T nL[36], nb[6];
#pragma unroll
  for (int i = 0; i < 36; ++i) nL[i] = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i) nb[i] = bv[i];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    T row[6];
#pragma unroll
    for (int j = 0; j < 6; ++j)
      row[j] = DOWN ? __shfl_down_sync(0xffffffffu, Lm[6 * k + j], d) : __shfl_up_sync(0xffffffffu, Lm[6 * k + j], d);
    const T bk = DOWN ? __shfl_down_sync(0xffffffffu, bv[k], d) : __shfl_up_sync(0xffffffffu, bv[k], d);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const T lik = Lm[6 * i + k];
#pragma unroll
      for (int j = 0; j < 6; ++j) nL[6 * i + j] = fma(lik, row[j], nL[6 * i + j]);
      nb[i] = fma(lik, bk, nb[i]);
    }
  }
  if (take) {
#pragma unroll
    for (int i = 0; i < 36; ++i) Lm[i] = nL[i];
#pragma unroll
    for (int i = 0; i < 6; ++i) bv[i] = nb[i];
  }
}

}  // namespace rd
