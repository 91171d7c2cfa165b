// rd_f32x2.cuh -- the fp32 per-link algebra on packed pairs (sm_100a f32x2:
// FFMA2 / FMUL2 run two FP32 FMAs per lane per instruction, the same FP32 pipe
// rate as FFMA at half the issue slots; measured 74 TFLOP/s, tools/ffma2_peak.cu).
// The forward Ad acts on (V_k, Vdot_k) pairs, the bias wrench on (v_c, a_c) and
// (I_c w, I_c wd) pairs, the backward Ad^T on (f_k, m_k) pairs, sin/cos as one
// polynomial pair.  Shared by the stash (rnea_thread.cu) and register
// (rnea_small.cu) THREAD kernels.
#pragma once
#include <cuda_runtime.h>

namespace rd {

__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// Cephes sinf / cosf coefficient pairs (S3, C3), (S2, C2), (S1, C1) as constant-bank
// operands of FFMA2 (immediates would be rebuilt into register pairs every link)
static __constant__ float2 kSinCos32x2[3] = {{-1.9515295891e-4f, 2.443315711809948e-5f},
                                             {8.3321608736e-3f, -1.388731625493765e-3f},
                                             {-1.6666654611e-1f, 4.166664568298827e-2f}};
// (sin, cos) of q (fp32, as rd_sincos) with the two polynomials evaluated as one pair
__device__ __forceinline__ void sincos_f32x2(float x, float* sp, float* cp) {
  const float k = rintf(x * 0.636619772f);
  const int quad = (int)k;
  float r = fmaf(-k, 1.57079637f, x);
  r = fmaf(-k, -4.37113883e-08f, r);
  r = fmaf(-k, -1.71512489e-15f, r);
  const float z = r * r;
  const float2 Z = f2(z);
  float2 P = fma2(Z, kSinCos32x2[0], kSinCos32x2[1]);
  P = fma2(Z, P, kSinCos32x2[2]);
  const float2 SC = fma2(mul2(Z, make_float2(r, z)), P, make_float2(r, fmaf(-0.5f, z, 1.0f)));
  const float sn = SC.x, cs = SC.y;
  const float a = (quad & 1) ? cs : sn;
  const float b = (quad & 1) ? sn : cs;
  *sp = (quad & 2) ? -a : a;
  *cp = ((quad + 1) & 2) ? -b : b;
}

// Ad_{f^-1} of dh_ad_finv (rd_math.cuh) on the pair (V, Vdot), lane-wise
__device__ __forceinline__ void dh_ad_finv_x2(float ca, float sa, float a, float d, float s, float c,
                                              const float2* in, float2* out) {
  const float2 CA = f2(ca), SA = f2(sa), NSA = f2(-sa), C = f2(c), S = f2(s), NS = f2(-s);
  float2 v1 = fma2(CA, in[1], mul2(SA, in[2])), v2 = fma2(CA, in[2], mul2(NSA, in[1]));
  const float2 w1 = fma2(CA, in[4], mul2(SA, in[5])), w2 = fma2(CA, in[5], mul2(NSA, in[4]));
  v1 = fma2(f2(a), w2, v1);
  v2 = fma2(f2(-a), w1, v2);
  const float2 W0 = fma2(C, in[3], mul2(S, w1)), W1 = fma2(C, w1, mul2(NS, in[3]));
  const float2 V0 = fma2(C, in[0], mul2(S, v1)), V1 = fma2(C, v1, mul2(NS, in[0]));
  out[0] = fma2(f2(d), W1, V0);
  out[1] = fma2(f2(-d), W0, V1);
  out[2] = v2; out[3] = W0; out[4] = W1; out[5] = w2;
}

// Fhat at the centre of mass (bias_force_com, rd_math.cuh) from the pairs (V, Vdot);
// out = (f0, n0, f1, n1, f2, n2), the (f, m) pair order of the backward sweep
template <typename CT>
__device__ __forceinline__ void bias_force_com_x2(const CT& C, const float2* VV, float* out) {
  const float c0 = C.c[0], c1 = C.c[1], c2 = C.c[2];
  // (v_c, a_c) = (v, vd) + (w, wd) x c
  const float2 P0 = fma2(VV[4], f2(c2), fma2(VV[5], f2(-c1), VV[0]));
  const float2 P1 = fma2(VV[5], f2(c0), fma2(VV[3], f2(-c2), VV[1]));
  const float2 P2 = fma2(VV[3], f2(c1), fma2(VV[4], f2(-c0), VV[2]));
  const float w0 = VV[3].x, w1 = VV[4].x, w2 = VV[5].x;
  const float f0 = C.m * fmaf(w1, P2.x, fmaf(-w2, P1.x, P0.y));
  const float f1 = C.m * fmaf(w2, P0.x, fmaf(-w0, P2.x, P1.y));
  const float f2v = C.m * fmaf(w0, P1.x, fmaf(-w1, P0.x, P2.y));
  // (I_c w, I_c wd)
  const float Ixx = C.Ic[0], Iyy = C.Ic[1], Izz = C.Ic[2], Ixy = C.Ic[3], Ixz = C.Ic[4], Iyz = C.Ic[5];
  const float2 L0 = fma2(f2(Ixx), VV[3], fma2(f2(Ixy), VV[4], mul2(f2(Ixz), VV[5])));
  const float2 L1 = fma2(f2(Ixy), VV[3], fma2(f2(Iyy), VV[4], mul2(f2(Iyz), VV[5])));
  const float2 L2 = fma2(f2(Ixz), VV[3], fma2(f2(Iyz), VV[4], mul2(f2(Izz), VV[5])));
  out[0] = f0; out[2] = f1; out[4] = f2v;
  out[1] = fmaf(c1, f2v, fmaf(-c2, f1, fmaf(w1, L2.x, fmaf(-w2, L1.x, L0.y))));
  out[3] = fmaf(c2, f0, fmaf(-c0, f2v, fmaf(w2, L0.x, fmaf(-w0, L2.x, L1.y))));
  out[5] = fmaf(c0, f1, fmaf(-c1, f0, fmaf(w0, L1.x, fmaf(-w1, L0.x, L2.y))));
}

// F <- Fh + Ad^T_{f^-1} F of dh_bwd (rd_math.cuh) on the pairs FF[k] = (f_k, m_k),
// updated in place (lane updates, so no pair is re-assembled); Fh in the pair
// order (f0, n0, f1, n1, f2, n2)
__device__ __forceinline__ void dh_bwd_x2(float ca, float sa, float a, float d, float s, float c,
                                          float2* FF, const float* Fh) {
  // Tz(d): m += d e_z x f = d (-f1, f0, 0)   (m lanes)
  FF[0].y = fmaf(-d, FF[1].x, FF[0].y);
  FF[1].y = fmaf(d, FF[0].x, FF[1].y);
  // Rz; the x rows are final
  const float2 F0 = fma2(f2(c), FF[0], fma2(f2(-s), FF[1], make_float2(Fh[0], Fh[1])));
  float2 g1 = fma2(f2(s), FF[0], mul2(f2(c), FF[1]));
  // Tx(a): m += a e_x x f = a (0, -f2, f1)
  g1.y = fmaf(-a, FF[2].x, g1.y);
  FF[2].y = fmaf(a, g1.x, FF[2].y);
  // Rx, + Fh
  const float2 F1 = fma2(f2(ca), g1, fma2(f2(-sa), FF[2], make_float2(Fh[2], Fh[3])));
  const float2 F2 = fma2(f2(sa), g1, fma2(f2(ca), FF[2], make_float2(Fh[4], Fh[5])));
  FF[0] = F0; FF[1] = F1; FF[2] = F2;
}


}  // namespace rd
