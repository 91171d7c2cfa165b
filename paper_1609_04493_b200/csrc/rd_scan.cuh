// rd_scan.cuh -- warp-level scan building blocks shared by the scan kernels
// (product path): composition of affine maps x -> L x + b (6x6 L) across lanes.
#pragma once
#include "rd_internal.h"
#include "rd_math.cuh"

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

// Backward half of the literal scan kernels (lane = link l, n <= 32): the Eq. (16)
// affine scan F_l = L_l F_{l+1} + Fhat_l, L_l = Ad^T_{f_{l+1}^{-1}} = [[R', 0], [[p']R', R']]
// from link l+1's (R', p') (lagged torque row dropped, A5; link n-1:
// F_{n-1} = Fhat + F_{n+1}, f_{n,n+1} = I), as a Kogge-Stone suffix scan of
// (6x6, offset) operators; returns tau_l = S_l^T F_l, S = (beta e_z, alpha e_z).
template <typename T>
__device__ __forceinline__ T eq16_backward_torque(int lane, int n, bool act, const Rot<T>& R, T p0, T p1, T p2,
                                                  const T (&Fh)[6], const T (&Ftip)[6], T alpha, T beta) {
  const unsigned f = 0xffffffffu;
  const T nR[9] = {__shfl_down_sync(f, R.r00, 1), __shfl_down_sync(f, R.r01, 1), __shfl_down_sync(f, R.r02, 1),
                   __shfl_down_sync(f, R.r10, 1), __shfl_down_sync(f, R.r11, 1), __shfl_down_sync(f, R.r12, 1),
                   __shfl_down_sync(f, R.r20, 1), __shfl_down_sync(f, R.r21, 1), __shfl_down_sync(f, R.r22, 1)};
  const T np0 = __shfl_down_sync(f, p0, 1), np1 = __shfl_down_sync(f, p1, 1), np2 = __shfl_down_sync(f, p2, 1);
  T Lm[36], bv[6];
  const bool has_child = lane + 1 < n;
#pragma unroll
  for (int i = 0; i < 36; ++i) Lm[i] = 0;
  if (has_child) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        Lm[6 * i + j] = nR[3 * i + j];
        Lm[6 * (3 + i) + 3 + j] = nR[3 * i + j];
      }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const T x0 = nR[j], x1 = nR[3 + j], x2 = nR[6 + j];
      Lm[6 * 3 + j] = np1 * x2 - np2 * x1;
      Lm[6 * 4 + j] = np2 * x0 - np0 * x2;
      Lm[6 * 5 + j] = np0 * x1 - np1 * x0;
    }
  } else if (!act) {
#pragma unroll
    for (int i = 0; i < 6; ++i) Lm[7 * i] = 1;        // padding lanes: identity operator
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) bv[k] = (act ? Fh[k] : T(0)) + ((lane == n - 1) ? Ftip[k] : T(0));
#pragma unroll
  for (int dd = 1; dd < 32; dd <<= 1) compose_shfl<T, true>(Lm, bv, dd, lane + dd < 32);
  return fma(beta, bv[2], alpha * bv[5]);
}

}  // namespace rd
