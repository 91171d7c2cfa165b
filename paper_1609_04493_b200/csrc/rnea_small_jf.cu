// rnea_small_jf.cu -- the register-resident THREAD kernel in JOINT frames: one thread per
// state, the whole recursion of Eq. (1)-(2) in registers, link loops unrolled
// at compile time, for short chains of ANY joint type (revolute, prismatic, screw:
// S_i = (beta e_z, alpha e_z)).
//
// The DH-frame register kernel (rnea_small.cuh) needs a well-conditioned DH model;
// screw joints and calibrated arms with nearly parallel consecutive axes (capi.cu
// build_dh) ran REVERSE / GENERIC instead.  Same structure in the joint frames of
// LinkConst: f_i = (Rm Rz(alpha q), pm + beta q Rm e_z), the general Ad maps
// (fwd_step / bwd_step, rd_math.cuh), Fhat_i = J_i Vdot_i - ad^T_{V_i} J_i V_i
// with J about the joint origin, per-link (sin, cos) and Fhat kept in registers.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"
#include "rd_aba.cuh"

namespace rd {

namespace {

constexpr int kJfSmallThreads = 128;

template <typename T, int N>
struct SmallJfParams {
  LinkConst<T> L[N];
  Boundary<T> bnd;
};

template <typename T, int N, bool SB>
__global__ void __launch_bounds__(kJfSmallThreads)
rnea_small_jf_kernel(const __grid_constant__ SmallJfParams<T, N> P, int64_t B, const T* __restrict__ q,
                     const T* __restrict__ qd, const T* __restrict__ qdd, T* __restrict__ tau,
                     const __grid_constant__ typename SBArg<T, SB>::type sb) {
  const int64_t b = (int64_t)blockIdx.x * kJfSmallThreads + threadIdx.x;
  if (b >= B) return;
  T cq[N], cqd[N], cqa[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    cq[k] = __ldg(q + (int64_t)k * B + b);
    cqd[k] = __ldg(qd + (int64_t)k * B + b);
    cqa[k] = __ldg(qdd + (int64_t)k * B + b);
  }
  // forward sweep, Eq. (1); (sin, cos) and Fhat of every link stay in registers
  T V[6], Vd[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) { V[k] = P.bnd.V0[k]; Vd[k] = P.bnd.Vd0[k]; }
  if constexpr (SB) {
    if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, V);
    if (sb.Vd0) sb_vec(sb.Vd0, sb.A0, B, b, Vd);
  }
  T ss[N], sc[N], Fh[N][6];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const LinkConst<T>& C = P.L[k];
    Rot<T> R;
    T p0, p1, p2, s, c, d;
    link_transform(C, cq[k], R, p0, p1, p2, s, c, d);
    T Vn[6], Vdn[6];
    fwd_step<T, false>(C, R, p0, p1, p2, cqd[k], cqa[k], V, Vd, Vn, Vdn);
    bias_force(C, Vn, Vdn, Fh[k]);
    ss[k] = s; sc[k] = c;
#pragma unroll
    for (int j = 0; j < 6; ++j) { V[j] = Vn[j]; Vd[j] = Vdn[j]; }
  }
  // backward sweep, Eq. (2): F_i = Fhat_i + Ad^T_{f_{i,i+1}^-1} F_{i+1}, tau_i = S_i^T F_i;
  // f_{n,n+1} = I (A5)
  T F[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) F[k] = P.bnd.Ftip[k];
  if constexpr (SB) {
    if (sb.Ft) sb_vec(sb.Ft, sb.At, B, b, F);
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    T Fo[6];
    if (i == N - 1) {
#pragma unroll
      for (int k = 0; k < 6; ++k) Fo[k] = Fh[i][k] + F[k];
    } else {
      const LinkConst<T>& Cc = P.L[i + 1];
      const Rot<T> R = make_rot(Cc, ss[i + 1], sc[i + 1]);
      const T d = Cc.beta * cq[i + 1];
      bwd_step(R, fma(d, Cc.Rm[2], Cc.pm[0]), fma(d, Cc.Rm[5], Cc.pm[1]), fma(d, Cc.Rm[8], Cc.pm[2]), F, Fh[i], Fo);
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) F[k] = Fo[k];
    tau[(int64_t)i * B + b] = fma(P.L[i].alpha, F[5], P.L[i].beta * F[2]);
  }
}

template <typename T, int N>
cudaError_t jf_launch_n(const LinkConst<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q, const T* qd,
                        const T* qdd, T* tau, cudaStream_t st, const StateBoundary<T>* sb) {
  SmallJfParams<T, N> P;
  for (int i = 0; i < N; ++i) P.L[i] = L_host[i];
  P.bnd = bnd;
  const unsigned grid = (unsigned)((B + kJfSmallThreads - 1) / kJfSmallThreads);
  if (sb)
    rnea_small_jf_kernel<T, N, true><<<grid, kJfSmallThreads, 0, st>>>(P, B, q, qd, qdd, tau, *sb);
  else
    rnea_small_jf_kernel<T, N, false><<<grid, kJfSmallThreads, 0, st>>>(P, B, q, qd, qdd, tau, NoStateBoundary{});
  return cudaGetLastError();
}

template <typename T, int N>
cudaError_t jf_dispatch(int n, const LinkConst<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                        const T* qd, const T* qdd, T* tau, cudaStream_t st, const StateBoundary<T>* sb) {
  if (n == N) return jf_launch_n<T, N>(L_host, bnd, B, q, qd, qdd, tau, st, sb);
  if constexpr (N > 1) return jf_dispatch<T, N - 1>(n, L_host, bnd, B, q, qd, qdd, tau, st, sb);
  return cudaErrorInvalidValue;
}

template <typename T>
constexpr int small_jf_max_n() { return sizeof(T) == 8 ? 8 : 12; }

}  // namespace

bool small_jf_has_n(int n, bool fp64) { return n >= 1 && n <= (fp64 ? small_jf_max_n<double>() : small_jf_max_n<float>()); }

template <typename T>
cudaError_t launch_rnea_small_jf(int n, const LinkConst<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                                 const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                                 const StateBoundary<T>* sb) {
  if (!small_jf_has_n(n, sizeof(T) == 8)) return cudaErrorInvalidValue;
  ++*launches;
  return jf_dispatch<T, small_jf_max_n<T>()>(n, L_host, bnd, B, q, qd, qdd, tau, st, sb);
}

template cudaError_t launch_rnea_small_jf<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                                  const double*, const double*, const double*, double*,
                                                  cudaStream_t, int*, const StateBoundary<double>*);
template cudaError_t launch_rnea_small_jf<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                                 const float*, const float*, const float*, float*, cudaStream_t,
                                                 int*, const StateBoundary<float>*);

}  // namespace rd
