// rnea_generic.cu -- one thread per state, serial RNEA (Eq. 1-2) for ANY
// n and any mix of revolute / screw / prismatic joints (runtime loop).
//
// Model constants are read from a device array (uniform across the warp: one
// broadcast transaction per value, L1-resident).  The per-link stash
// (sin, cos, d = beta q, Fhat) = 9 scalars lives in a global workspace laid out
// slot-contiguous, ws[(i*9 + k) * slots + slot], so every access is a coalesced
// 256 B (fp64) warp transaction that stays in L1/L2 between the forward and the
// backward sweep.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"

namespace rd {

constexpr int kGenPerLink = 9;
constexpr int kGenThreads = 128;

int generic_ws_per_link() { return kGenPerLink; }

int64_t generic_ws_slots(int64_t B) {
  const int64_t max_slots = (int64_t)num_sms() * 8 * kGenThreads;   // 8 CTAs of 128 per SM
  const int64_t want = ((B + kGenThreads - 1) / kGenThreads) * kGenThreads;
  return want < max_slots ? want : max_slots;
}

template <typename T, bool SB>
__global__ void __launch_bounds__(kGenThreads)
rnea_generic_kernel(int n, const LinkConst<T>* __restrict__ L, const Boundary<T> bnd, int64_t B,
                    const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ qdd,
                    T* __restrict__ tau, T* __restrict__ ws, int64_t slots,
                    const typename SBArg<T, SB>::type sb) {
  const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= slots) return;
  for (int64_t b = slot; b < B; b += slots) {
    T V[6], Vd[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) { V[k] = bnd.V0[k]; Vd[k] = bnd.Vd0[k]; }
    if constexpr (SB) {                              // per-state V_0, Vdot_0 (NEXT-4)
      if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, V);
      if (sb.Vd0) sb_vec(sb.Vd0, sb.A0, B, b, Vd);
    }
    for (int i = 0; i < n; ++i) {
      const LinkConst<T> C = L[i];
      const T qi = __ldg(q + (int64_t)i * B + b);
      T s, c;
      rd_sincos(C.alpha * qi, &s, &c);
      const T d = C.beta * qi;
      const Rot<T> R = make_rot(C, s, c);
      const T p0 = fma(d, C.Rm[2], C.pm[0]), p1 = fma(d, C.Rm[5], C.pm[1]), p2 = fma(d, C.Rm[8], C.pm[2]);
      T Vn[6], Vdn[6], Fh[6];
      fwd_step<T, false>(C, R, p0, p1, p2, __ldg(qd + (int64_t)i * B + b), __ldg(qdd + (int64_t)i * B + b),
                         V, Vd, Vn, Vdn);
      bias_force(C, Vn, Vdn, Fh);
      T* w = ws + (int64_t)i * kGenPerLink * slots + slot;
      w[0] = s;
      w[slots] = c;
      w[2 * slots] = d;
#pragma unroll
      for (int k = 0; k < 6; ++k) w[(3 + k) * slots] = Fh[k];
#pragma unroll
      for (int k = 0; k < 6; ++k) { V[k] = Vn[k]; Vd[k] = Vdn[k]; }
    }
    // Backward, Eq. (2): F_i = Fhat_i + Ad^T_{f_{i,i+1}^{-1}} F_{i+1}, tau_i = S_i^T F_i.
    T F[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) F[k] = bnd.Ftip[k];
    if constexpr (SB) {
      if (sb.Ft) sb_vec(sb.Ft, sb.At, B, b, F);
    }
    bool tip = true;
    Rot<T> Rn;
    T pn0 = 0, pn1 = 0, pn2 = 0;
    for (int i = n - 1; i >= 0; --i) {
      const T* w = ws + (int64_t)i * kGenPerLink * slots + slot;
      T Fh[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) Fh[k] = w[(3 + k) * slots];
      if (tip) {
#pragma unroll
        for (int k = 0; k < 6; ++k) F[k] = Fh[k] + F[k];
        tip = false;
      } else {
        T Fo[6];
        bwd_step(Rn, pn0, pn1, pn2, F, Fh, Fo);
#pragma unroll
        for (int k = 0; k < 6; ++k) F[k] = Fo[k];
      }
      const LinkConst<T> C = L[i];
      tau[(int64_t)i * B + b] = fma(C.beta, F[2], C.alpha * F[5]);
      const T s = w[0], c = w[slots], d = w[2 * slots];
      Rn = make_rot(C, s, c);
      pn0 = fma(d, C.Rm[2], C.pm[0]);
      pn1 = fma(d, C.Rm[5], C.pm[1]);
      pn2 = fma(d, C.Rm[8], C.pm[2]);
    }
  }
}

template <typename T>
cudaError_t launch_rnea_generic(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B,
                                const T* q, const T* qd, const T* qdd, T* tau, T* ws, int64_t ws_slots,
                                cudaStream_t st, int* launches, const StateBoundary<T>* sb) {
  const int64_t grid = (ws_slots + kGenThreads - 1) / kGenThreads;
  if (sb)
    rnea_generic_kernel<T, true><<<(unsigned)grid, kGenThreads, 0, st>>>(n, L_dev, bnd, B, q, qd, qdd, tau, ws,
                                                                          ws_slots, *sb);
  else
    rnea_generic_kernel<T, false><<<(unsigned)grid, kGenThreads, 0, st>>>(n, L_dev, bnd, B, q, qd, qdd, tau, ws,
                                                                           ws_slots, NoStateBoundary{});
  ++*launches;
  return cudaGetLastError();
}

template cudaError_t launch_rnea_generic<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                                 const double*, const double*, const double*, double*, double*,
                                                 int64_t, cudaStream_t, int*, const StateBoundary<double>*);
template cudaError_t launch_rnea_generic<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                                const float*, const float*, const float*, float*, float*,
                                                int64_t, cudaStream_t, int*, const StateBoundary<float>*);

}  // namespace rd
