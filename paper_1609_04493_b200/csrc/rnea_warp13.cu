// rnea_warp13.cu -- the paper's scan operators taken literally (strategy
// WARP_SCAN_EQ13, n <= 32, any joints): one warp per state,
// lane = link, BODY-frame scans.
//   forward:  ONE Kogge-Stone scan of the Eq. (13) semigroup elements
//             a_l = (f_l^{-1}, S_l qdd_l, S_l qd_l) in SE(3) x se(3)^2
//             -- the synchronous V/Vdot scan of Eq. (12), not split as
//             in Alg. 1 --, prefixes P_l = a_l (+) P_{l-1} (A4), seed A_0 = (I, Vdot_0, V_0);
//             V_l = xi2(P_l), Vdot_l = xi1(P_l);
//   bias:     Fhat_l = J_l Vdot_l - ad^T_{V_l}(J_l V_l) per lane;
//   backward: the Eq. (16) affine scan F_l = Ad^T_{f_{l+1}^{-1}} F_{l+1} + Fhat_l
//             (lagged torque row dropped, A5) as a Kogge-Stone suffix
//             scan of (6x6, offset) operators, seed F_{n+1};
//   torque:   tau_l = S_l^T F_l (Alg. 1 line 5).
// Compared against the base-frame rnea_warp.cu (one SE(3) scan + vector sums),
// this carries 24 scalars per forward element and a 6x6 operator per backward
// element; it exists to measure the paper's own operators.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"
#include "rd_scan.cuh"

namespace rd {

constexpr int kW13Cta = 4;

// Eq. (13) element: g = (R, p) in SE(3), xi1, xi2 in se(3)
template <typename T>
struct VA {
  Rot<T> R;
  T p[3];
  T x1[6], x2[6];
};

// Ad_g x = (R x_v + p x (R x_w), R x_w)
template <typename T>
__device__ __forceinline__ void Ad_g(const Rot<T>& R, const T* p, const T* x, T* y) {
  T w0, w1, w2, v0, v1, v2;
  rot_n(R, x[3], x[4], x[5], w0, w1, w2);
  rot_n(R, x[0], x[1], x[2], v0, v1, v2);
  y[0] = fma(p[1], w2, fma(-p[2], w1, v0));
  y[1] = fma(p[2], w0, fma(-p[0], w2, v1));
  y[2] = fma(p[0], w1, fma(-p[1], w0, v2));
  y[3] = w0; y[4] = w1; y[5] = w2;
}

// a (+) b = (g_a g_b, Ad_{g_a} xi1_b + xi1_a - ad_{xi2_a}(Ad_{g_a} xi2_b), Ad_{g_a} xi2_b + xi2_a)
template <typename T>
__device__ __forceinline__ VA<T> oplus(const VA<T>& a, const VA<T>& b) {
  VA<T> r;
  const Rot<T>& A = a.R;
  r.R.r00 = fma(A.r00, b.R.r00, fma(A.r01, b.R.r10, A.r02 * b.R.r20));
  r.R.r01 = fma(A.r00, b.R.r01, fma(A.r01, b.R.r11, A.r02 * b.R.r21));
  r.R.r02 = fma(A.r00, b.R.r02, fma(A.r01, b.R.r12, A.r02 * b.R.r22));
  r.R.r10 = fma(A.r10, b.R.r00, fma(A.r11, b.R.r10, A.r12 * b.R.r20));
  r.R.r11 = fma(A.r10, b.R.r01, fma(A.r11, b.R.r11, A.r12 * b.R.r21));
  r.R.r12 = fma(A.r10, b.R.r02, fma(A.r11, b.R.r12, A.r12 * b.R.r22));
  r.R.r20 = fma(A.r20, b.R.r00, fma(A.r21, b.R.r10, A.r22 * b.R.r20));
  r.R.r21 = fma(A.r20, b.R.r01, fma(A.r21, b.R.r11, A.r22 * b.R.r21));
  r.R.r22 = fma(A.r20, b.R.r02, fma(A.r21, b.R.r12, A.r22 * b.R.r22));
  r.p[0] = fma(A.r00, b.p[0], fma(A.r01, b.p[1], fma(A.r02, b.p[2], a.p[0])));
  r.p[1] = fma(A.r10, b.p[0], fma(A.r11, b.p[1], fma(A.r12, b.p[2], a.p[1])));
  r.p[2] = fma(A.r20, b.p[0], fma(A.r21, b.p[1], fma(A.r22, b.p[2], a.p[2])));
  T y1[6], y2[6];
  Ad_g(a.R, a.p, b.x1, y1);
  Ad_g(a.R, a.p, b.x2, y2);
  // ad_{(v,w)}(x, y) = (w x x + v x y, w x y), (v, w) = xi2_a, (x, y) = y2
  const T* s = a.x2;
  const T ad0 = (s[4] * y2[2] - s[5] * y2[1]) + (s[1] * y2[5] - s[2] * y2[4]);
  const T ad1 = (s[5] * y2[0] - s[3] * y2[2]) + (s[2] * y2[3] - s[0] * y2[5]);
  const T ad2 = (s[3] * y2[1] - s[4] * y2[0]) + (s[0] * y2[4] - s[1] * y2[3]);
  const T ad3 = s[4] * y2[5] - s[5] * y2[4];
  const T ad4 = s[5] * y2[3] - s[3] * y2[5];
  const T ad5 = s[3] * y2[4] - s[4] * y2[3];
  r.x1[0] = y1[0] + a.x1[0] - ad0;
  r.x1[1] = y1[1] + a.x1[1] - ad1;
  r.x1[2] = y1[2] + a.x1[2] - ad2;
  r.x1[3] = y1[3] + a.x1[3] - ad3;
  r.x1[4] = y1[4] + a.x1[4] - ad4;
  r.x1[5] = y1[5] + a.x1[5] - ad5;
#pragma unroll
  for (int k = 0; k < 6; ++k) r.x2[k] = y2[k] + a.x2[k];
  return r;
}

template <typename T>
__device__ __forceinline__ VA<T> va_shfl_up(const VA<T>& a, int d) {
  VA<T> o;
  const unsigned f = 0xffffffffu;
  o.R.r00 = __shfl_up_sync(f, a.R.r00, d); o.R.r01 = __shfl_up_sync(f, a.R.r01, d); o.R.r02 = __shfl_up_sync(f, a.R.r02, d);
  o.R.r10 = __shfl_up_sync(f, a.R.r10, d); o.R.r11 = __shfl_up_sync(f, a.R.r11, d); o.R.r12 = __shfl_up_sync(f, a.R.r12, d);
  o.R.r20 = __shfl_up_sync(f, a.R.r20, d); o.R.r21 = __shfl_up_sync(f, a.R.r21, d); o.R.r22 = __shfl_up_sync(f, a.R.r22, d);
#pragma unroll
  for (int k = 0; k < 3; ++k) o.p[k] = __shfl_up_sync(f, a.p[k], d);
#pragma unroll
  for (int k = 0; k < 6; ++k) { o.x1[k] = __shfl_up_sync(f, a.x1[k], d); o.x2[k] = __shfl_up_sync(f, a.x2[k], d); }
  return o;
}

template <typename T>
__global__ void __launch_bounds__(kW13Cta * 32)
rnea_warp13_kernel(int n, const LinkConst<T>* __restrict__ Lg, const Boundary<T> bnd, int64_t B,
                   const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ qdd,
                   T* __restrict__ tau) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool act = lane < n;
  LinkConst<T> C;
  if (act) {
    C = Lg[lane];
  } else {
#pragma unroll
    for (int k = 0; k < 9; ++k) C.Rm[k] = (k % 4 == 0) ? T(1) : T(0);
#pragma unroll
    for (int k = 0; k < 3; ++k) { C.pm[k] = 0; C.h[k] = 0; }
#pragma unroll
    for (int k = 0; k < 6; ++k) C.I[k] = 0;
    C.m = 0; C.alpha = 0; C.beta = 0;
  }
  for (int64_t b = (int64_t)blockIdx.x * kW13Cta + warp; b < B; b += (int64_t)gridDim.x * kW13Cta) {
    T qi = 0, qdi = 0, qddi = 0;
    if (act) {
      qi = __ldg(q + (int64_t)lane * B + b);
      qdi = __ldg(qd + (int64_t)lane * B + b);
      qddi = __ldg(qdd + (int64_t)lane * B + b);
    }
    // f_l = (R, p) (joint frames); the operand is (f_l^{-1}, S qdd, S qd), f^{-1} = (R^T, -R^T p)
    T s, c;
    rd_sincos(C.alpha * qi, &s, &c);
    const Rot<T> R = make_rot(C, s, c);
    const T d = C.beta * qi;
    const T p0 = fma(d, C.Rm[2], C.pm[0]), p1 = fma(d, C.Rm[5], C.pm[1]), p2 = fma(d, C.Rm[8], C.pm[2]);
    VA<T> a;
    a.R = Rot<T>{R.r00, R.r10, R.r20, R.r01, R.r11, R.r21, R.r02, R.r12, R.r22};
    a.p[0] = -fma(R.r00, p0, fma(R.r10, p1, R.r20 * p2));
    a.p[1] = -fma(R.r01, p0, fma(R.r11, p1, R.r21 * p2));
    a.p[2] = -fma(R.r02, p0, fma(R.r12, p1, R.r22 * p2));
#pragma unroll
    for (int k = 0; k < 6; ++k) { a.x1[k] = 0; a.x2[k] = 0; }
    a.x1[2] = C.beta * qddi; a.x1[5] = C.alpha * qddi;
    a.x2[2] = C.beta * qdi;  a.x2[5] = C.alpha * qdi;
    // Kogge-Stone: P_l = a_l (+) P_{l-d}
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const VA<T> e = va_shfl_up(a, dd);
      const VA<T> r = oplus(a, e);
      if (lane >= dd) a = r;
    }
    // apply the seed A_0 = (I, Vdot_0, V_0): V_l = xi2(P_l (+) A_0), Vdot_l = xi1(P_l (+) A_0)
    VA<T> seed;
    seed.R = Rot<T>{1, 0, 0, 0, 1, 0, 0, 0, 1};
    seed.p[0] = seed.p[1] = seed.p[2] = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) { seed.x1[k] = bnd.Vd0[k]; seed.x2[k] = bnd.V0[k]; }
    const VA<T> P = oplus(a, seed);
    T Fh[6];
    bias_force(C, P.x2, P.x1, Fh);
    if (!act) {
#pragma unroll
      for (int k = 0; k < 6; ++k) Fh[k] = 0;
    }
    const T t = eq16_backward_torque(lane, n, act, R, p0, p1, p2, Fh, bnd.Ftip, C.alpha, C.beta);
    if (act) tau[(int64_t)lane * B + b] = t;
  }
}

template <typename T>
cudaError_t launch_rnea_warp13(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                               const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                               bool* supported) {
  *supported = n >= 1 && n <= 32;
  if (!*supported) return cudaSuccess;
  int64_t grid = (B + kW13Cta - 1) / kW13Cta;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (grid > cap) grid = cap;
  rnea_warp13_kernel<T><<<(unsigned)grid, kW13Cta * 32, 0, st>>>(n, L_dev, bnd, B, q, qd, qdd, tau);
  ++*launches;
  return cudaGetLastError();
}

template cudaError_t launch_rnea_warp13<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                                const double*, const double*, const double*, double*, cudaStream_t,
                                                int*, bool*);
template cudaError_t launch_rnea_warp13<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                               const float*, const float*, const float*, float*, cudaStream_t, int*,
                                               bool*);

}  // namespace rd
