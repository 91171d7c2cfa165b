// rd_math.cuh -- per-link RNEA arithmetic in joint frames (product path).
//
// Notation follows PAPER.md Eq. (1)-(2): V_i, Vdot_i (twists, (v,w)),
// Fhat_i = J_i Vdot_i - ad^T_{V_i}(J_i V_i), F_i (wrench, (f,m)),
// tau_i = S_i^T F_i.  In the joint frame of link i, f_{i-1,i} = (R, p) with
// R = Rm Rz(alpha q), p = pm + beta q Rm e_z, and S_i = (beta e_z, alpha e_z)
// (DESIGN.md "Joint frames").  Lean forms:
//   Ad_{f^-1}(v, w)       = (R^T (v + w x p), R^T w)
//   ad_V(S qd)            = qd (beta w x e_z + alpha v x e_z, alpha w x e_z)
//   -ad^T_V (P_f, P_m)    = (w x P_f, v x P_f + w x P_m)
//   J (v, w)              = (m v - h x w, h x v + I w)
//   Ad^T_{f^-1}(f, m)     = (R f, p x (R f) + R m)
#pragma once
#include "rd_internal.h"
#include "rd_f32x2.cuh"

namespace rd {

template <typename T>
struct Rot {
  T r00, r01, r02, r10, r11, r12, r20, r21, r22;
};

// sin/cos of a joint angle, branch-free (one basic block, so the scheduler can
// interleave it with the V/Vdot chains).  Quadrant k = rint(2x/pi) by the
// 1.5*2^52 rounding trick; Cody-Waite reduction with pi/2 split in two doubles
// (each FMA rounds once, the split carries ~107 bits of pi/2, so the reduced
// argument is accurate to ~1 ulp for |x| up to ~1e9); fdlibm minimax
// polynomials (__kernel_sin / __kernel_cos coefficients) on [-pi/4, pi/4].
// Measured against the host libm in tests/test_gpu_parity.py (large-angle case).
// Coefficients in the constant bank so the DFMAs take them as c[][] operands
// (double literals would be rebuilt with two UMOVs each, every call).
static __constant__ double kSinCosD[16] = {
    6755399441055744.0,            // 0: 1.5 * 2^52 (round-to-integer shifter)
    0.63661977236758138,           // 1: 2/pi
    1.5707963267948966,            // 2: pi/2 (hi)
    6.123233995736766e-17,         // 3: pi/2 (lo)
    1.58969099521155010221e-10,    // 4..9: fdlibm __kernel_sin S6..S1
    -2.50507602534068634195e-08,
    2.75573137070700676789e-06,
    -1.98412698298579493134e-04,
    8.33333333332248946124e-03,
    -1.66666666666666324348e-01,
    -1.13596475577881948265e-11,   // 10..15: fdlibm __kernel_cos C6..C1
    2.08757232129817482790e-09,
    -2.75573143513906633035e-07,
    2.48015872894767294178e-05,
    -1.38888888888741095749e-03,
    4.16666666666666019037e-02,
};

__device__ __forceinline__ void rd_sincos(double x, double* sp, double* cp) {
  const double t = fma(x, kSinCosD[1], kSinCosD[0]);
  const int quad = __double2loint(t);
  const double k = t - kSinCosD[0];
  double r = fma(-k, kSinCosD[2], x);
  r = fma(-k, kSinCosD[3], r);
  const double z = r * r;
  double ps = fma(z, kSinCosD[4], kSinCosD[5]);
  ps = fma(z, ps, kSinCosD[6]);
  ps = fma(z, ps, kSinCosD[7]);
  ps = fma(z, ps, kSinCosD[8]);
  ps = fma(z, ps, kSinCosD[9]);
  const double sn = fma(z * r, ps, r);
  double pc = fma(z, kSinCosD[10], kSinCosD[11]);
  pc = fma(z, pc, kSinCosD[12]);
  pc = fma(z, pc, kSinCosD[13]);
  pc = fma(z, pc, kSinCosD[14]);
  pc = fma(z, pc, kSinCosD[15]);
  const double cs = fma(z * z, pc, fma(-0.5, z, 1.0));
  // sin(x) = [s, c, -s, -c][quad & 3], cos(x) = [c, -s, -c, s][quad & 3];
  // the negations flip the sign bit of the high word.
  const bool swap = quad & 1;
  const double a = swap ? cs : sn;
  const double b = swap ? sn : cs;
  const unsigned sa = ((unsigned)quad & 2u) << 30, sb = ((unsigned)(quad + 1) & 2u) << 30;
  *sp = __hiloint2double(__double2hiint(a) ^ (int)sa, __double2loint(a));
  *cp = __hiloint2double(__double2hiint(b) ^ (int)sb, __double2loint(b));
}
// fp32: three-float Cody-Waite split of pi/2 (accurate for |x| up to ~1e4) and
// Cephes minimax polynomials; branch-free.
__device__ __forceinline__ void rd_sincos(float x, float* sp, float* cp) {
  {
    const float k = rintf(x * 0.636619772f);
    const int quad = (int)k;
    float r = fmaf(-k, 1.57079637f, x);                 // pi/2 in three floats (Cody-Waite)
    r = fmaf(-k, -4.37113883e-08f, r);
    r = fmaf(-k, -1.71512489e-15f, r);
    const float z = r * r;
    // minimax on [-pi/4, pi/4] (Cephes sinf/cosf coefficients)
    const float sn = fmaf(z * r, fmaf(z, fmaf(z, -1.9515295891e-4f, 8.3321608736e-3f), -1.6666654611e-1f), r);
    const float cs = fmaf(z * z, fmaf(z, fmaf(z, 2.443315711809948e-5f, -1.388731625493765e-3f),
                                       4.166664568298827e-2f), fmaf(-0.5f, z, 1.0f));
    const float a = (quad & 1) ? cs : sn;
    const float b = (quad & 1) ? sn : cs;
    *sp = (quad & 2) ? -a : a;
    *cp = ((quad + 1) & 2) ? -b : b;
  }
}

// R = Rm * Rz(theta) from (s, c) = (sin theta, cos theta): only the first two
// columns change, R[:,2] = Rm[:,2].
template <typename T>
__device__ __forceinline__ Rot<T> make_rot(const LinkConst<T>& C, T s, T c) {
  Rot<T> R;
  R.r00 = fma(C.Rm[0], c, C.Rm[1] * s);
  R.r10 = fma(C.Rm[3], c, C.Rm[4] * s);
  R.r20 = fma(C.Rm[6], c, C.Rm[7] * s);
  R.r01 = fma(C.Rm[1], c, -(C.Rm[0] * s));
  R.r11 = fma(C.Rm[4], c, -(C.Rm[3] * s));
  R.r21 = fma(C.Rm[7], c, -(C.Rm[6] * s));
  R.r02 = C.Rm[2];
  R.r12 = C.Rm[5];
  R.r22 = C.Rm[8];
  return R;
}

// y = R^T x
template <typename T>
__device__ __forceinline__ void rot_t(const Rot<T>& R, T x0, T x1, T x2, T& y0, T& y1, T& y2) {
  y0 = fma(R.r00, x0, fma(R.r10, x1, R.r20 * x2));
  y1 = fma(R.r01, x0, fma(R.r11, x1, R.r21 * x2));
  y2 = fma(R.r02, x0, fma(R.r12, x1, R.r22 * x2));
}
// y = R x
template <typename T>
__device__ __forceinline__ void rot_n(const Rot<T>& R, T x0, T x1, T x2, T& y0, T& y1, T& y2) {
  y0 = fma(R.r00, x0, fma(R.r01, x1, R.r02 * x2));
  y1 = fma(R.r10, x0, fma(R.r11, x1, R.r12 * x2));
  y2 = fma(R.r20, x0, fma(R.r21, x1, R.r22 * x2));
}

// out = Ad_{f^-1} in, with f = (R, p):  (R^T (v + w x p), R^T w)
template <typename T>
__device__ __forceinline__ void ad_finv(const Rot<T>& R, T p0, T p1, T p2, const T* in, T* out) {
  const T x0 = fma(in[4], p2, fma(-in[5], p1, in[0]));
  const T x1 = fma(in[5], p0, fma(-in[3], p2, in[1]));
  const T x2 = fma(in[3], p1, fma(-in[4], p0, in[2]));
  rot_t(R, x0, x1, x2, out[0], out[1], out[2]);
  rot_t(R, in[3], in[4], in[5], out[3], out[4], out[5]);
}

// Fhat = J Vd + (w x P_f, v x P_f + w x P_m), P = J V
// CT: any per-link constant struct with m, h[3], I[6] (LinkConst or LinkDH).
template <typename T, typename CT>
__device__ __forceinline__ void bias_force(const CT& C, const T* V, const T* Vd, T* Fh) {
  const T m = C.m, h0 = C.h[0], h1 = C.h[1], h2 = C.h[2];
  const T Ixx = C.I[0], Iyy = C.I[1], Izz = C.I[2], Ixy = C.I[3], Ixz = C.I[4], Iyz = C.I[5];
  // P = J V
  const T Pf0 = fma(m, V[0], fma(-h1, V[5], h2 * V[4]));
  const T Pf1 = fma(m, V[1], fma(-h2, V[3], h0 * V[5]));
  const T Pf2 = fma(m, V[2], fma(-h0, V[4], h1 * V[3]));
  const T Pm0 = fma(h1, V[2], fma(-h2, V[1], fma(Ixx, V[3], fma(Ixy, V[4], Ixz * V[5]))));
  const T Pm1 = fma(h2, V[0], fma(-h0, V[2], fma(Ixy, V[3], fma(Iyy, V[4], Iyz * V[5]))));
  const T Pm2 = fma(h0, V[1], fma(-h1, V[0], fma(Ixz, V[3], fma(Iyz, V[4], Izz * V[5]))));
  // A = J Vd, then add the gyroscopic terms
  T Af0 = fma(m, Vd[0], fma(-h1, Vd[5], h2 * Vd[4]));
  T Af1 = fma(m, Vd[1], fma(-h2, Vd[3], h0 * Vd[5]));
  T Af2 = fma(m, Vd[2], fma(-h0, Vd[4], h1 * Vd[3]));
  T Am0 = fma(h1, Vd[2], fma(-h2, Vd[1], fma(Ixx, Vd[3], fma(Ixy, Vd[4], Ixz * Vd[5]))));
  T Am1 = fma(h2, Vd[0], fma(-h0, Vd[2], fma(Ixy, Vd[3], fma(Iyy, Vd[4], Iyz * Vd[5]))));
  T Am2 = fma(h0, Vd[1], fma(-h1, Vd[0], fma(Ixz, Vd[3], fma(Iyz, Vd[4], Izz * Vd[5]))));
  const T w0 = V[3], w1 = V[4], w2 = V[5], v0 = V[0], v1 = V[1], v2 = V[2];
  Fh[0] = fma(w1, Pf2, fma(-w2, Pf1, Af0));
  Fh[1] = fma(w2, Pf0, fma(-w0, Pf2, Af1));
  Fh[2] = fma(w0, Pf1, fma(-w1, Pf0, Af2));
  Fh[3] = fma(v1, Pf2, fma(-v2, Pf1, fma(w1, Pm2, fma(-w2, Pm1, Am0))));
  Fh[4] = fma(v2, Pf0, fma(-v0, Pf2, fma(w2, Pm0, fma(-w0, Pm2, Am1))));
  Fh[5] = fma(v0, Pf1, fma(-v1, Pf0, fma(w0, Pm1, fma(-w1, Pm0, Am2))));
}

// Fhat = J Vd - ad^T_V (J V) evaluated at the centre of mass c, where J
// is block diagonal (Newton-Euler form; C: LinkDHc):
//   v_c = v + w x c,  a_c = vd + wd x c,  f = m (a_c + w x v_c),
//   n_c = I_c wd + w x (I_c w),  Fhat = (f, n_c + c x f)
// 51 FP64 instructions instead of the 66 of bias_force.
template <typename T, typename CT>
__device__ __forceinline__ void bias_force_com(const CT& C, const T* V, const T* Vd, T* Fh) {
  const T c0 = C.c[0], c1 = C.c[1], c2 = C.c[2];
  const T w0 = V[3], w1 = V[4], w2 = V[5];
  const T dw0 = Vd[3], dw1 = Vd[4], dw2 = Vd[5];
  const T vc0 = fma(w1, c2, fma(-w2, c1, V[0]));
  const T vc1 = fma(w2, c0, fma(-w0, c2, V[1]));
  const T vc2 = fma(w0, c1, fma(-w1, c0, V[2]));
  const T ac0 = fma(dw1, c2, fma(-dw2, c1, Vd[0]));
  const T ac1 = fma(dw2, c0, fma(-dw0, c2, Vd[1]));
  const T ac2 = fma(dw0, c1, fma(-dw1, c0, Vd[2]));
  const T f0 = C.m * fma(w1, vc2, fma(-w2, vc1, ac0));
  const T f1 = C.m * fma(w2, vc0, fma(-w0, vc2, ac1));
  const T f2 = C.m * fma(w0, vc1, fma(-w1, vc0, ac2));
  const T Ixx = C.Ic[0], Iyy = C.Ic[1], Izz = C.Ic[2], Ixy = C.Ic[3], Ixz = C.Ic[4], Iyz = C.Ic[5];
  const T L0 = fma(Ixx, w0, fma(Ixy, w1, Ixz * w2));
  const T L1 = fma(Ixy, w0, fma(Iyy, w1, Iyz * w2));
  const T L2 = fma(Ixz, w0, fma(Iyz, w1, Izz * w2));
  Fh[0] = f0; Fh[1] = f1; Fh[2] = f2;
  Fh[3] = fma(c1, f2, fma(-c2, f1, fma(w1, L2, fma(-w2, L1, fma(Ixx, dw0, fma(Ixy, dw1, Ixz * dw2))))));
  Fh[4] = fma(c2, f0, fma(-c0, f2, fma(w2, L0, fma(-w0, L2, fma(Ixy, dw0, fma(Iyy, dw1, Iyz * dw2))))));
  Fh[5] = fma(c0, f1, fma(-c1, f0, fma(w0, L1, fma(-w1, L0, fma(Ixz, dw0, fma(Iyz, dw1, Izz * dw2))))));
}

// Fh = Pc - ad^T_V (J V) = Pc + (w x P_f, v x P_f + w x P_m), P = J V: the bias
// wrench of a link with Vdot = 0 (the ABA's p_i) plus the wrench Pc
// carried from the child, Pc seeding the FMA chains (42 FP64 instructions; the
// general bias_force with a zero Vdot would spend 24 more on J 0).
template <typename T, typename CT>
__device__ __forceinline__ void bias_force_v(const CT& C, const T* V, const T* Pc, T* Fh) {
  const T m = C.m, h0 = C.h[0], h1 = C.h[1], h2 = C.h[2];
  const T Ixx = C.I[0], Iyy = C.I[1], Izz = C.I[2], Ixy = C.I[3], Ixz = C.I[4], Iyz = C.I[5];
  const T Pf0 = fma(m, V[0], fma(-h1, V[5], h2 * V[4]));
  const T Pf1 = fma(m, V[1], fma(-h2, V[3], h0 * V[5]));
  const T Pf2 = fma(m, V[2], fma(-h0, V[4], h1 * V[3]));
  const T Pm0 = fma(h1, V[2], fma(-h2, V[1], fma(Ixx, V[3], fma(Ixy, V[4], Ixz * V[5]))));
  const T Pm1 = fma(h2, V[0], fma(-h0, V[2], fma(Ixy, V[3], fma(Iyy, V[4], Iyz * V[5]))));
  const T Pm2 = fma(h0, V[1], fma(-h1, V[0], fma(Ixz, V[3], fma(Iyz, V[4], Izz * V[5]))));
  const T w0 = V[3], w1 = V[4], w2 = V[5], v0 = V[0], v1 = V[1], v2 = V[2];
  Fh[0] = fma(w1, Pf2, fma(-w2, Pf1, Pc[0]));
  Fh[1] = fma(w2, Pf0, fma(-w0, Pf2, Pc[1]));
  Fh[2] = fma(w0, Pf1, fma(-w1, Pf0, Pc[2]));
  Fh[3] = fma(v1, Pf2, fma(-v2, Pf1, fma(w1, Pm2, fma(-w2, Pm1, Pc[3]))));
  Fh[4] = fma(v2, Pf0, fma(-v0, Pf2, fma(w2, Pm0, fma(-w0, Pm2, Pc[4]))));
  Fh[5] = fma(v0, Pf1, fma(-v1, Pf0, fma(w0, Pm1, fma(-w1, Pm0, Pc[5]))));
}

// One forward step of Eq. (1) for link with constants C:
//   V  = Ad_{f^-1} Vp + S qd
//   Vd = Ad_{f^-1} Vdp + S qdd + ad_V (S qd)      (= ... - ad_{S qd} Ad_{f^-1} Vp)
// REV: alpha = 1, beta = 0 known at compile time.
template <typename T, bool REV>
__device__ __forceinline__ void fwd_step(const LinkConst<T>& C, const Rot<T>& R, T p0, T p1, T p2,
                                         T qd, T qdd, const T* Vp, const T* Vdp, T* V, T* Vd) {
  ad_finv(R, p0, p1, p2, Vp, V);
  ad_finv(R, p0, p1, p2, Vdp, Vd);
  if (REV) {
    V[5] += qd;
    Vd[5] += qdd;
    // ad_V(e_z qd) = qd (v x e_z, w x e_z),  a x e_z = (a1, -a0, 0)
    Vd[0] = fma(qd, V[1], Vd[0]);
    Vd[1] = fma(-qd, V[0], Vd[1]);
    Vd[3] = fma(qd, V[4], Vd[3]);
    Vd[4] = fma(-qd, V[3], Vd[4]);
  } else {
    const T a = C.alpha, b = C.beta;
    V[2] = fma(b, qd, V[2]);
    V[5] = fma(a, qd, V[5]);
    Vd[2] = fma(b, qdd, Vd[2]);
    Vd[5] = fma(a, qdd, Vd[5]);
    const T aq = a * qd, bq = b * qd;
    Vd[0] = fma(bq, V[4], fma(aq, V[1], Vd[0]));
    Vd[1] = fma(-bq, V[3], fma(-aq, V[0], Vd[1]));
    Vd[3] = fma(aq, V[4], Vd[3]);
    Vd[4] = fma(-aq, V[3], Vd[4]);
  }
}

// One backward step of Eq. (2): F = Fhat + Ad^T_{f_{i,i+1}^{-1}} Fn
// where (R, p) is the transform of link i+1.
template <typename T>
__device__ __forceinline__ void bwd_step(const Rot<T>& R, T p0, T p1, T p2, const T* Fn, const T* Fh, T* F) {
  T y0, y1, y2, z0, z1, z2;
  rot_n(R, Fn[0], Fn[1], Fn[2], y0, y1, y2);
  rot_n(R, Fn[3], Fn[4], Fn[5], z0, z1, z2);
  F[0] = Fh[0] + y0;
  F[1] = Fh[1] + y1;
  F[2] = Fh[2] + y2;
  F[3] = fma(p1, y2, fma(-p2, y1, Fh[3] + z0));
  F[4] = fma(p2, y0, fma(-p0, y2, Fh[4] + z1));
  F[5] = fma(p0, y1, fma(-p1, y0, Fh[5] + z2));
}

// ---------------------------------------------------------------- DH frames
// f = Rx(alpha) Tx(a) Rz(theta) Tz(d) (modified DH), so R = Rx(alpha) Rz(theta)
// and p = (a, -sa d, ca d).  Every map below is applied as the product of its
// four elementary factors (plane rotations and single-axis shifts, each 2-8
// FP64 instructions), never through R and p: Ad_{f^-1} costs 20 instructions
// per twist (22 with the general p x w form), the backward Ad^T with Fhat folded
// into its last factor 20 (28).  DESIGN.md "DH frames" derives the factors;
// the GPU parity suite checks every kernel that uses them against the oracle.
// out = Ad_{f^-1} in = Ad_{Tz^-1} Ad_{Rz^-1} Ad_{Tx^-1} Ad_{Rx^-1} in.
template <typename T>
__device__ __forceinline__ void dh_ad_finv(T ca, T sa, T a, T d, T s, T c, const T* in, T* out) {
  // Rx^T (x0, ca x1 + sa x2, -sa x1 + ca x2) on v and w
  T v1 = fma(ca, in[1], sa * in[2]), v2 = fma(ca, in[2], -(sa * in[1]));
  const T w1 = fma(ca, in[4], sa * in[5]), w2 = fma(ca, in[5], -(sa * in[4]));
  // Tx(a)^-1: v += w x (a e_x) = a (0, w2, -w1)
  v1 = fma(a, w2, v1);
  v2 = fma(-a, w1, v2);
  // Rz^T (c y0 + s y1, -s y0 + c y1, y2)
  const T W0 = fma(c, in[3], s * w1), W1 = fma(c, w1, -(s * in[3]));
  const T V0 = fma(c, in[0], s * v1), V1 = fma(c, v1, -(s * in[0]));
  // Tz(d)^-1: v += w x (d e_z) = d (w1, -w0, 0)
  out[0] = fma(d, W1, V0);
  out[1] = fma(-d, W0, V1);
  out[2] = v2;
  out[3] = W0; out[4] = W1; out[5] = w2;
}
template <typename T, typename CT>
__device__ __forceinline__ void dh_ad_finv(const CT& C, T s, T c, const T* in, T* out) {
  dh_ad_finv(C.ca, C.sa, C.a, C.d, s, c, in, out);
}

// F = Fh + Ad^T_{f^-1} Fn, Ad^T_{f^-1} = Ad^T_{Rx^-1} Ad^T_{Tx^-1} Ad^T_{Rz^-1} Ad^T_{Tz^-1}
// (a translation t acts as (f, m) -> (f, m + t x f)), with (ca, sa, a, d, s, c) of
// the child link (identity for the tip, A5); Fh is added inside the last factor.
template <typename T>
__device__ __forceinline__ void dh_bwd(T ca, T sa, T a, T d, T s, T c, const T* Fn, const T* Fh, T* F) {
  // Tz(d): m += d e_z x f = d (-f1, f0, 0)
  const T m0 = fma(-d, Fn[1], Fn[3]), m1 = fma(d, Fn[0], Fn[4]);
  // Rz: (c y0 - s y1, s y0 + c y1, y2); the x rows are final (Rx fixes e_x)
  F[0] = fma(c, Fn[0], fma(-s, Fn[1], Fh[0]));
  F[3] = fma(c, m0, fma(-s, m1, Fh[3]));
  const T f1 = fma(s, Fn[0], c * Fn[1]);
  T n1 = fma(s, m0, c * m1);
  // Tx(a): m += a e_x x f = a (0, -f2, f1)
  n1 = fma(-a, Fn[2], n1);
  const T n2 = fma(a, f1, Fn[5]);
  // Rx: (z0, ca z1 - sa z2, sa z1 + ca z2), + Fh
  F[1] = fma(ca, f1, fma(-sa, Fn[2], Fh[1]));
  F[2] = fma(sa, f1, fma(ca, Fn[2], Fh[2]));
  F[4] = fma(ca, n1, fma(-sa, n2, Fh[4]));
  F[5] = fma(sa, n1, fma(ca, n2, Fh[5]));
}

// out = Ad_f in = Ad_{Rx} Ad_{Tx} Ad_{Rz} Ad_{Tz} in (a translation t acts as
// (v, w) -> (v + t x w, w)): the inverse of dh_ad_finv (used to re-derive
// V_{i-1}, Vdot_{i-1} from V_i, Vdot_i).
template <typename T>
__device__ __forceinline__ void dh_ad_f(T ca, T sa, T a, T d, T s, T c, const T* in, T* out) {
  // Tz(d): v += d e_z x w = d (-w1, w0, 0)
  const T v0 = fma(-d, in[4], in[0]), v1 = fma(d, in[3], in[1]);
  // Rz: (c y0 - s y1, s y0 + c y1, y2)
  const T W0 = fma(c, in[3], -(s * in[4])), W1 = fma(s, in[3], c * in[4]);
  T V1 = fma(s, v0, c * v1);
  out[0] = fma(c, v0, -(s * v1));
  // Tx(a): v += a e_x x w = a (0, -w2, w1)
  V1 = fma(-a, in[5], V1);
  const T V2 = fma(a, W1, in[2]);
  // Rx: (z0, ca z1 - sa z2, sa z1 + ca z2)
  out[1] = fma(ca, V1, -(sa * V2));
  out[2] = fma(sa, V1, ca * V2);
  out[3] = W0;
  out[4] = fma(ca, W1, -(sa * in[5]));
  out[5] = fma(sa, W1, ca * in[5]);
}
template <typename T>
__device__ __forceinline__ void dh_ad_f(const LinkDH<T>& C, T s, T c, const T* in, T* out) {
  dh_ad_f(C.ca, C.sa, C.a, C.d, s, c, in, out);
}

// (sin, cos) of theta and the translation d of link C: revolute theta = th0 + q;
// prismatic (PR && prism) theta = th0, d = d0 + q.
// fp32: kSc32Pair evaluates the sin and cos polynomials as one FFMA2 pair (sincos_f32x2,
// bit-identical to rd_sincos(float)), opt-in where it measured faster (REVERSE fp32;
// the register ABA lost 1.4-1.8x, ab_f32_sc2*); kSc32Mufu: sincos_mufu.
// fp32 sin/cos on the special-function unit: reduction to [-pi, pi] with 2 pi split in
// two floats, then sin.approx / cos.approx (PTX: max abs error 2^-20.9 there, ~8x the
// polynomial's; used where the fp32 error stays far inside 1e-4: the register ID
// kernel, n <= 32: 4.8e-6 at n = 30; REVERSE's inverse recursion amplified it to
// 5.5e-5 at n = 200, so REVERSE keeps the polynomial; profiles/r02/ab_f32_mufu.txt).
__device__ __forceinline__ void sincos_mufu(float x, float* sp, float* cp) {
  const float k = rintf(x * 0.159154943f);
  float r = fmaf(-k, 6.28318548f, x);
  r = fmaf(-k, -1.74845553e-7f, r);
  *sp = __sinf(r);
  *cp = __cosf(r);
}
// fp32 sin/cos evaluation of dh_link (fp64 always uses rd_sincos).
enum SinCos32 { kSc32Poly = 0, kSc32Pair = 1, kSc32Mufu = 2 };
template <bool PR, int SC = kSc32Poly, typename T, typename CT>
__device__ __forceinline__ void dh_link(const CT& C, bool prism, T qi, T* s, T* c, T* d) {
  const T qa = (PR && prism) ? T(0) : qi;
  if constexpr (sizeof(T) == 8) {
    rd_sincos(qa + C.th0, s, c);
  } else {
    T s0, c0;
    if constexpr (SC == kSc32Mufu) sincos_mufu(qa, &s0, &c0);
    else if constexpr (SC == kSc32Pair) sincos_f32x2(qa, &s0, &c0);
    else rd_sincos(qa, &s0, &c0);
    *s = fma(s0, C.cth0, c0 * C.sth0);
    *c = fma(c0, C.cth0, -(s0 * C.sth0));
  }
  *d = (PR && prism) ? C.d + qi : C.d;
}

// Per-state boundary vector of state b: out = A u, u = p[k*B + b] (k = 0..5).
template <typename T>
__device__ __forceinline__ void sb_vec(const T* __restrict__ p, const T* A, int64_t B, int64_t b, T* out) {
  T u[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) u[k] = __ldg(p + (int64_t)k * B + b);
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    T acc = A[6 * r] * u[0];
#pragma unroll
    for (int c = 1; c < 6; ++c) acc = fma(A[6 * r + c], u[c], acc);
    out[r] = acc;
  }
}

}  // namespace rd
