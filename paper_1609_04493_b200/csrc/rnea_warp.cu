// rnea_warp.cu -- one WARP per state, lane = link: the paper's parallel ID
// (Alg. 1) as Kogge-Stone shuffle scans across the links of one
// robot (strategy WARP_SCAN, n <= 32, any joint type).
//
// The two forward scans of Alg. 1 (InclusiveVelScan, InclusiveAccScan: Ad-affine
// semigroup elements (f^-1, xi), Eq. 12-13 with the A4 operand order) are
// evaluated in the BASE frame, where their non-commutative part is one SE(3)
// prefix product and the rest are plain vector prefix sums (DESIGN.md A-base):
//   g_{0,l}   = f_1 f_2 ... f_l                     (SE(3) scan, 5 shuffle rounds)
//   S0_l      = Ad_{g_{0,l}} S_l                     (joint axis in the base frame)
//   V0_l      = V_0 + sum_{k<=l} S0_k qd_k           (= Ad_{g_{0,l}} V_l)
//   Vd0_l     = Vd_0 + sum_{k<=l} (S0_k qdd_k + ad_{V0_k} S0_k qd_k)
// then the bias wrench per lane ("perfectly parallel") in the body frame,
// moved to the base frame, and the backward InclusiveForceScan (Eq. 16) becomes
// a suffix sum: F0_l = Ad^T_{g_{0,n}^{-1}} F_{n+1} + sum_{k>=l} Ad^T_{g_{0,k}^{-1}} Fhat_k;
// tau_l = S0_l . F0_l (CalcTorque).  Each identity is pinned in the oracle tests
// (scan == recursion) and by GPU parity.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"

namespace rd {

constexpr int kWarpCta = 8;          // warps (states) per CTA

template <typename T>
__device__ __forceinline__ T shup(T v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
template <typename T>
__device__ __forceinline__ T shdn(T v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }

template <typename T, bool SB>
__global__ void __launch_bounds__(kWarpCta * 32)
rnea_warp_kernel(int n, const LinkConst<T>* __restrict__ Lg, const Boundary<T> bnd, int64_t B,
                 const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ qdd,
                 T* __restrict__ tau, T* __restrict__ fhat, const typename SBArg<T, SB>::type sb) {
  // per-link constants in shared memory, structure-of-arrays [field][32] (lane-contiguous)
  constexpr int NF = sizeof(LinkConst<T>) / sizeof(T);
  __shared__ T sc[NF][32];
  for (int idx = threadIdx.x; idx < NF * 32; idx += blockDim.x) {
    const int f = idx / 32, l = idx % 32;
    T v = 0;
    if (l < n) v = reinterpret_cast<const T*>(Lg + l)[f];
    else if (f == 0 || f == 4 || f == 8) v = 1;     // padding link: Rm = I, everything else 0
    sc[f][l] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const bool act = lane < n;
  auto c = [&](int f) { return sc[f][lane]; };
  LinkConst<T> C;
#pragma unroll
  for (int f = 0; f < 9; ++f) C.Rm[f] = c(f);
#pragma unroll
  for (int f = 0; f < 3; ++f) C.pm[f] = c(9 + f);
  C.m = c(12);
#pragma unroll
  for (int f = 0; f < 3; ++f) C.h[f] = c(13 + f);
#pragma unroll
  for (int f = 0; f < 6; ++f) C.I[f] = c(16 + f);
  C.alpha = c(22);
  C.beta = c(23);

  for (int64_t b = (int64_t)blockIdx.x * kWarpCta + warp; b < B; b += (int64_t)gridDim.x * kWarpCta) {
    T qi = 0, qdi = 0, qddi = 0;
    if (act) {
      qi = __ldg(q + (int64_t)lane * B + b);
      qdi = __ldg(qd + (int64_t)lane * B + b);
      qddi = qdd ? __ldg(qdd + (int64_t)lane * B + b) : T(0);   // qdd == nullptr: qdd = 0 (tau_bias, Eq. 5)
    }
    // CalcTransform: f_l = (Rm Rz(alpha q), pm + beta q Rm e_z)
    T s, cc;
    rd_sincos(C.alpha * qi, &s, &cc);
    Rot<T> R = make_rot(C, s, cc);
    const T d = C.beta * qi;
    T p0 = fma(d, C.Rm[2], C.pm[0]), p1 = fma(d, C.Rm[5], C.pm[1]), p2 = fma(d, C.Rm[8], C.pm[2]);
    // SE(3) inclusive scan g_{0,l} = g_{0,l-1} f_l (earlier element on the left)
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const T e00 = shup(R.r00, dd), e01 = shup(R.r01, dd), e02 = shup(R.r02, dd);
      const T e10 = shup(R.r10, dd), e11 = shup(R.r11, dd), e12 = shup(R.r12, dd);
      const T e20 = shup(R.r20, dd), e21 = shup(R.r21, dd), e22 = shup(R.r22, dd);
      const T ep0 = shup(p0, dd), ep1 = shup(p1, dd), ep2 = shup(p2, dd);
      if (lane >= dd) {
        Rot<T> Rn;
        Rn.r00 = fma(e00, R.r00, fma(e01, R.r10, e02 * R.r20));
        Rn.r01 = fma(e00, R.r01, fma(e01, R.r11, e02 * R.r21));
        Rn.r02 = fma(e00, R.r02, fma(e01, R.r12, e02 * R.r22));
        Rn.r10 = fma(e10, R.r00, fma(e11, R.r10, e12 * R.r20));
        Rn.r11 = fma(e10, R.r01, fma(e11, R.r11, e12 * R.r21));
        Rn.r12 = fma(e10, R.r02, fma(e11, R.r12, e12 * R.r22));
        Rn.r20 = fma(e20, R.r00, fma(e21, R.r10, e22 * R.r20));
        Rn.r21 = fma(e20, R.r01, fma(e21, R.r11, e22 * R.r21));
        Rn.r22 = fma(e20, R.r02, fma(e21, R.r12, e22 * R.r22));
        const T n0 = fma(e00, p0, fma(e01, p1, fma(e02, p2, ep0)));
        const T n1 = fma(e10, p0, fma(e11, p1, fma(e12, p2, ep1)));
        const T n2 = fma(e20, p0, fma(e21, p1, fma(e22, p2, ep2)));
        R = Rn;
        p0 = n0; p1 = n1; p2 = n2;
      }
    }
    // S0_l = Ad_{g_{0,l}} (beta e_z, alpha e_z) = (beta z + alpha p x z, alpha z), z = R e_z
    const T z0 = R.r02, z1 = R.r12, z2 = R.r22;
    T S0[6];
    S0[0] = fma(C.beta, z0, C.alpha * (p1 * z2 - p2 * z1));
    S0[1] = fma(C.beta, z1, C.alpha * (p2 * z0 - p0 * z2));
    S0[2] = fma(C.beta, z2, C.alpha * (p0 * z1 - p1 * z0));
    S0[3] = C.alpha * z0;
    S0[4] = C.alpha * z1;
    S0[5] = C.alpha * z2;
    // V0 = V_0 + inclusive prefix sum of S0 qd
    T V[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) V[k] = S0[k] * qdi;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const T o = shup(V[k], dd);
        if (lane >= dd) V[k] += o;
      }
    }
    {
      T v0[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) v0[k] = bnd.V0[k];
      if constexpr (SB) {                            // per-state V_0 (NEXT-4)
        if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, v0);
      }
#pragma unroll
      for (int k = 0; k < 6; ++k) V[k] += v0[k];
    }
    // Vd0 = Vd_0 + prefix sum of S0 qdd + ad_{V0}(S0 qd)
    T A[6];
    {
      const T x0 = S0[0] * qdi, x1 = S0[1] * qdi, x2 = S0[2] * qdi;
      const T y0 = S0[3] * qdi, y1 = S0[4] * qdi, y2 = S0[5] * qdi;
      // ad_{(v,w)}(x, y) = (w x x + v x y, w x y)
      A[0] = fma(S0[0], qddi, (V[4] * x2 - V[5] * x1) + (V[1] * y2 - V[2] * y1));
      A[1] = fma(S0[1], qddi, (V[5] * x0 - V[3] * x2) + (V[2] * y0 - V[0] * y2));
      A[2] = fma(S0[2], qddi, (V[3] * x1 - V[4] * x0) + (V[0] * y1 - V[1] * y0));
      A[3] = fma(S0[3], qddi, V[4] * y2 - V[5] * y1);
      A[4] = fma(S0[4], qddi, V[5] * y0 - V[3] * y2);
      A[5] = fma(S0[5], qddi, V[3] * y1 - V[4] * y0);
    }
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const T o = shup(A[k], dd);
        if (lane >= dd) A[k] += o;
      }
    }
    {
      T a0[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) a0[k] = bnd.Vd0[k];
      if constexpr (SB) {
        if (sb.Vd0) sb_vec(sb.Vd0, sb.A0, B, b, a0);
      }
#pragma unroll
      for (int k = 0; k < 6; ++k) A[k] += a0[k];
    }
    // body-frame V_l, Vdot_l = Ad_{g^-1}(.), bias wrench Fhat_l, back to the base frame
    T Vb[6], Ab[6], Fh[6];
    ad_finv(R, p0, p1, p2, V, Vb);
    ad_finv(R, p0, p1, p2, A, Ab);
    bias_force(C, Vb, Ab, Fh);
    if (fhat && act) {                               // Fhat_l (joint frame) for the merged FD scan, [n][6][B]
#pragma unroll
      for (int k = 0; k < 6; ++k) fhat[((int64_t)lane * 6 + k) * B + b] = Fh[k];
    }
    T F[6];
    const T zero6[6] = {0, 0, 0, 0, 0, 0};
    bwd_step(R, p0, p1, p2, Fh, zero6, F);          // F0hat = Ad^T_{g^-1} Fhat = (R f, p x R f + R m)
    if (!act) {
#pragma unroll
      for (int k = 0; k < 6; ++k) F[k] = 0;
    }
    T ftip[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) ftip[k] = bnd.Ftip[k];
    if constexpr (SB) {
      if (sb.Ft) sb_vec(sb.Ft, sb.At, B, b, ftip);
    }
    if (lane == n - 1) {                             // tip wrench F_{n+1} (frame n) to the base frame
      T Ft[6];
      bwd_step(R, p0, p1, p2, ftip, zero6, Ft);
#pragma unroll
      for (int k = 0; k < 6; ++k) F[k] += Ft[k];
    }
    // backward scan (Eq. 16) = suffix sum in the base frame
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const T o = shdn(F[k], dd);
        if (lane + dd < 32) F[k] += o;
      }
    }
    // CalcTorque: tau_l = S0_l . F0_l
    T t = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) t = fma(S0[k], F[k], t);
    if (act && tau) tau[(int64_t)lane * B + b] = t;
  }
}

template <typename T>
cudaError_t launch_rnea_warp(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                             const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                             bool* supported, T* fhat, const StateBoundary<T>* sb) {
  *supported = n >= 1 && n <= 32;
  if (!*supported) return cudaSuccess;
  int64_t grid = (B + kWarpCta - 1) / kWarpCta;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (grid > cap) grid = cap;
  if (sb)
    rnea_warp_kernel<T, true><<<(unsigned)grid, kWarpCta * 32, 0, st>>>(n, L_dev, bnd, B, q, qd, qdd, tau, fhat,
                                                                         *sb);
  else
    rnea_warp_kernel<T, false><<<(unsigned)grid, kWarpCta * 32, 0, st>>>(n, L_dev, bnd, B, q, qd, qdd, tau, fhat,
                                                                          NoStateBoundary{});
  ++*launches;
  return cudaGetLastError();
}

template cudaError_t launch_rnea_warp<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                              const double*, const double*, const double*, double*, cudaStream_t,
                                              int*, bool*, double*, const StateBoundary<double>*);
template cudaError_t launch_rnea_warp<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                             const float*, const float*, const float*, float*, cudaStream_t, int*,
                                             bool*, float*, const StateBoundary<float>*);

}  // namespace rd
