// rd_aba.cuh -- articulated-body helpers shared by the ABA kernels (product path):
// symmetric 6x6 spatial inertias in 3x3 blocks, the congruence X^T K X for
// X = Ad_{f^-1}, the link inertia and transform in joint frames.
#pragma once
#include "rd_internal.h"
#include "rd_math.cuh"

namespace rd {

// Symmetric 6x6 K = [[A, B], [B^T, C]]: A, C symmetric (xx yy zz xy xz yz), B general row-major.
template <typename T>
struct Sym6 {
  T a[6], b[9], c[6];
};

// y = K x
template <typename T>
__device__ __forceinline__ void sym6_mv(const Sym6<T>& K, const T* x, T* y) {
  const T* A = K.a;
  const T* Bm = K.b;
  const T* C = K.c;
  y[0] = A[0] * x[0] + A[3] * x[1] + A[4] * x[2] + Bm[0] * x[3] + Bm[1] * x[4] + Bm[2] * x[5];
  y[1] = A[3] * x[0] + A[1] * x[1] + A[5] * x[2] + Bm[3] * x[3] + Bm[4] * x[4] + Bm[5] * x[5];
  y[2] = A[4] * x[0] + A[5] * x[1] + A[2] * x[2] + Bm[6] * x[3] + Bm[7] * x[4] + Bm[8] * x[5];
  y[3] = Bm[0] * x[0] + Bm[3] * x[1] + Bm[6] * x[2] + C[0] * x[3] + C[3] * x[4] + C[4] * x[5];
  y[4] = Bm[1] * x[0] + Bm[4] * x[1] + Bm[7] * x[2] + C[3] * x[3] + C[1] * x[4] + C[5] * x[5];
  y[5] = Bm[2] * x[0] + Bm[5] * x[1] + Bm[8] * x[2] + C[4] * x[3] + C[5] * x[4] + C[2] * x[5];
}

// K -= u u^T / D
template <typename T>
__device__ __forceinline__ void sym6_rank1_sub(Sym6<T>& K, const T* u, T invD) {
  T w[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) w[k] = u[k] * invD;
  K.a[0] -= w[0] * u[0]; K.a[1] -= w[1] * u[1]; K.a[2] -= w[2] * u[2];
  K.a[3] -= w[0] * u[1]; K.a[4] -= w[0] * u[2]; K.a[5] -= w[1] * u[2];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) K.b[3 * i + j] -= w[i] * u[3 + j];
  K.c[0] -= w[3] * u[3]; K.c[1] -= w[4] * u[4]; K.c[2] -= w[5] * u[5];
  K.c[3] -= w[3] * u[4]; K.c[4] -= w[3] * u[5]; K.c[5] -= w[4] * u[5];
}

// Full 3x3 from symmetric storage.
template <typename T>
__device__ __forceinline__ void sym_full(const T* s, T* M) {
  M[0] = s[0]; M[1] = s[3]; M[2] = s[4];
  M[3] = s[3]; M[4] = s[1]; M[5] = s[5];
  M[6] = s[4]; M[7] = s[5]; M[8] = s[2];
}

// out = R M R^T (M general 3x3 row-major)
template <typename T>
__device__ __forceinline__ void rot_conj(const Rot<T>& R, const T* M, T* out) {
  const T r[9] = {R.r00, R.r01, R.r02, R.r10, R.r11, R.r12, R.r20, R.r21, R.r22};
  T t[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) t[3 * i + j] = r[3 * i] * M[j] + r[3 * i + 1] * M[3 + j] + r[3 * i + 2] * M[6 + j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) out[3 * i + j] = t[3 * i] * r[3 * j] + t[3 * i + 1] * r[3 * j + 1] + t[3 * i + 2] * r[3 * j + 2];
}

// Congruence X^T K X with X = Ad_{f^-1}, f = (R, p) (derivation in DESIGN.md):
//   A' = R A R^T, B' = R B R^T, C' = R C R^T, P = [p]
//   A_new = A',  B_new = B' - A' P,  C_new = C' + P B' + (P B')^T - P A' P.
template <typename T>
__device__ __forceinline__ void congruence(const Rot<T>& R, T p0, T p1, T p2, const Sym6<T>& K, Sym6<T>& out) {
  T Af[9], Cf[9], Ap[9], Bp[9], Cp[9];
  sym_full(K.a, Af);
  sym_full(K.c, Cf);
  rot_conj(R, Af, Ap);
  rot_conj(R, K.b, Bp);
  rot_conj(R, Cf, Cp);
  // A'P: column j = A' (p x e_j); p x e_0 = (0, p2, -p1), p x e_1 = (-p2, 0, p0), p x e_2 = (p1, -p0, 0)
  T AP[9];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    AP[3 * i + 0] = Ap[3 * i + 1] * p2 - Ap[3 * i + 2] * p1;
    AP[3 * i + 1] = Ap[3 * i + 2] * p0 - Ap[3 * i + 0] * p2;
    AP[3 * i + 2] = Ap[3 * i + 0] * p1 - Ap[3 * i + 1] * p0;
  }
  // P X for a 3x3 X: column j = p x X[:, j]
  T PB[9], PAP[9];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const T x0 = Bp[j], x1 = Bp[3 + j], x2 = Bp[6 + j];
    PB[j] = p1 * x2 - p2 * x1;
    PB[3 + j] = p2 * x0 - p0 * x2;
    PB[6 + j] = p0 * x1 - p1 * x0;
    const T y0 = AP[j], y1 = AP[3 + j], y2 = AP[6 + j];
    PAP[j] = p1 * y2 - p2 * y1;
    PAP[3 + j] = p2 * y0 - p0 * y2;
    PAP[6 + j] = p0 * y1 - p1 * y0;
  }
  out.a[0] = Ap[0]; out.a[1] = Ap[4]; out.a[2] = Ap[8];
  out.a[3] = Ap[1]; out.a[4] = Ap[2]; out.a[5] = Ap[5];
#pragma unroll
  for (int k = 0; k < 9; ++k) out.b[k] = Bp[k] - AP[k];
  // C_new(i,j) = C'(i,j) + PB(i,j) + PB(j,i) - PAP(i,j)   (symmetric)
  out.c[0] = Cp[0] + 2 * PB[0] - PAP[0];
  out.c[1] = Cp[4] + 2 * PB[4] - PAP[4];
  out.c[2] = Cp[8] + 2 * PB[8] - PAP[8];
  out.c[3] = Cp[1] + PB[1] + PB[3] - PAP[1];
  out.c[4] = Cp[2] + PB[2] + PB[6] - PAP[2];
  out.c[5] = Cp[5] + PB[5] + PB[7] - PAP[5];
}

template <typename T>
__device__ __forceinline__ void link_inertia(const LinkConst<T>& C, Sym6<T>& K) {
  // J = [[m I, -[h]], [[h], I]]
  K.a[0] = C.m; K.a[1] = C.m; K.a[2] = C.m; K.a[3] = 0; K.a[4] = 0; K.a[5] = 0;
  const T h0 = C.h[0], h1 = C.h[1], h2 = C.h[2];
  // -[h] = [[0, h2, -h1], [-h2, 0, h0], [h1, -h0, 0]]
  K.b[0] = 0;   K.b[1] = h2;  K.b[2] = -h1;
  K.b[3] = -h2; K.b[4] = 0;   K.b[5] = h0;
  K.b[6] = h1;  K.b[7] = -h0; K.b[8] = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) K.c[k] = C.I[k];
}

template <typename T>
__device__ __forceinline__ void link_transform(const LinkConst<T>& C, T qi, Rot<T>& R, T& p0, T& p1, T& p2,
                                               T& s, T& c, T& d) {
  rd_sincos(C.alpha * qi, &s, &c);
  d = C.beta * qi;
  R = make_rot(C, s, c);
  p0 = fma(d, C.Rm[2], C.pm[0]);
  p1 = fma(d, C.Rm[5], C.pm[1]);
  p2 = fma(d, C.Rm[8], C.pm[2]);
}

}  // namespace rd

namespace rd {

// ---------------------------------------------------------------- DH-frame congruence
// Plane rotations of the 3x3 blocks (~14 flops per symmetric block, 24 per
// general block), the rotation factors of dh_congruence below.
template <typename T>
__device__ __forceinline__ void sym_rot_plane(T* a, int i, int j, int k, T c, T s) {
  // symmetric block in (xx yy zz xy xz yz) storage; rotate the (i, j) plane, k the fixed axis
  auto idx = [](int r, int q) { return r == q ? r : 2 + r + q; };   // (0,1)->3 (0,2)->4 (1,2)->5
  const T aii = a[idx(i, i)], ajj = a[idx(j, j)], aij = a[idx(i, j)], aik = a[idx(i, k)], ajk = a[idx(j, k)];
  const T cc = c * c, ss = s * s, cs = c * s;
  a[idx(i, i)] = fma(cc, aii, fma(-2 * cs, aij, ss * ajj));
  a[idx(j, j)] = fma(ss, aii, fma(2 * cs, aij, cc * ajj));
  a[idx(i, j)] = fma(cs, aii - ajj, (cc - ss) * aij);
  a[idx(i, k)] = fma(c, aik, -(s * ajk));
  a[idx(j, k)] = fma(s, aik, c * ajk);
}
template <typename T>
__device__ __forceinline__ void gen_rot_plane(T* b, int i, int j, T c, T s) {
  // B <- R B R^T for the plane rotation R of the (i, j) plane (B general 3x3, row-major)
#pragma unroll
  for (int q = 0; q < 3; ++q) {                  // rows i, j
    const T bi = b[3 * i + q], bj = b[3 * j + q];
    b[3 * i + q] = fma(c, bi, -(s * bj));
    b[3 * j + q] = fma(s, bi, c * bj);
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {                  // columns i, j
    const T bi = b[3 * r + i], bj = b[3 * r + j];
    b[3 * r + i] = fma(c, bi, -(s * bj));
    b[3 * r + j] = fma(s, bi, c * bj);
  }
}
// Congruence by a translation t along one axis, C_t(K) = Ad_{(I,t)^-1}^T K Ad_{(I,t)^-1}:
//   B <- B - A[t],  C <- C + [t]B + ([t]B)^T - [t]A[t]     (B, the old B on the right)
// written out for t = d e_z and t = a e_x, where [t] has two non-zeros (17 FP64
// instructions each instead of ~80 for a general t).
template <typename T>
__device__ __forceinline__ void sym6_shift_z(Sym6<T>& K, T d) {
  const T* A = K.a;     // xx yy zz xy xz yz
  T* Bm = K.b;          // row-major
  T* C = K.c;
  const T dd = d * d, d2 = d + d;
  const T b00 = Bm[0], b01 = Bm[1], b02 = Bm[2], b10 = Bm[3], b11 = Bm[4], b12 = Bm[5];
  C[0] = fma(-d2, b10, fma(dd, A[1], C[0]));
  C[1] = fma(d2, b01, fma(dd, A[0], C[1]));
  C[3] = fma(-d, b11, fma(d, b00, fma(-dd, A[3], C[3])));
  C[4] = fma(-d, b12, C[4]);
  C[5] = fma(d, b02, C[5]);
  // B(:, 0) -= d A(:, 1);  B(:, 1) += d A(:, 0)
  Bm[0] = fma(-d, A[3], b00); Bm[1] = fma(d, A[0], b01);
  Bm[3] = fma(-d, A[1], b10); Bm[4] = fma(d, A[3], b11);
  Bm[6] = fma(-d, A[5], Bm[6]); Bm[7] = fma(d, A[4], Bm[7]);
}
template <typename T>
__device__ __forceinline__ void sym6_shift_x(Sym6<T>& K, T a) {
  const T* A = K.a;
  T* Bm = K.b;
  T* C = K.c;
  const T aa = a * a, a2 = a + a;
  const T b10 = Bm[3], b11 = Bm[4], b12 = Bm[5], b20 = Bm[6], b21 = Bm[7], b22 = Bm[8];
  C[1] = fma(-a2, b21, fma(aa, A[2], C[1]));
  C[2] = fma(a2, b12, fma(aa, A[1], C[2]));
  C[5] = fma(-a, b22, fma(a, b11, fma(-aa, A[5], C[5])));
  C[3] = fma(-a, b20, C[3]);
  C[4] = fma(a, b10, C[4]);
  // B(:, 1) -= a A(:, 2);  B(:, 2) += a A(:, 1)
  Bm[1] = fma(-a, A[4], Bm[1]); Bm[2] = fma(a, A[3], Bm[2]);
  Bm[4] = fma(-a, A[5], b11);   Bm[5] = fma(a, A[1], b12);
  Bm[7] = fma(-a, A[2], b21);   Bm[8] = fma(a, A[5], b22);
}

// X^T K X for X = Ad_{f^-1}, f = Rx(alpha) Tx(a) Rz(theta) Tz(d): the congruences
// of the four factors, innermost first (C_{gh} = C_g o C_h): shift by d e_z,
// rotate by Rz(theta), shift by a e_x, rotate by Rx(alpha).
template <typename T>
__device__ __forceinline__ void dh_congruence(T ca, T sa, T a, T d, T s, T c, Sym6<T>& K) {
  sym6_shift_z(K, d);
  // Rz(theta): plane (0, 1), fixed axis 2
  sym_rot_plane(K.a, 0, 1, 2, c, s);
  gen_rot_plane(K.b, 0, 1, c, s);
  sym_rot_plane(K.c, 0, 1, 2, c, s);
  sym6_shift_x(K, a);
  // Rx(alpha): plane (1, 2), fixed axis 0
  sym_rot_plane(K.a, 1, 2, 0, ca, sa);
  gen_rot_plane(K.b, 1, 2, ca, sa);
  sym_rot_plane(K.c, 1, 2, 0, ca, sa);
}
template <typename T>
__device__ __forceinline__ void dh_congruence(const LinkDH<T>& C, T s, T c, Sym6<T>& K) {
  dh_congruence(C.ca, C.sa, C.a, C.d, s, c, K);
}

// Revolute joint in DH frames, S = e_5, U = K e_5, D = U_5: Jhat^a = K - U U^T / D has
// row and column 5 identically zero (Jhat^a S = U - U D / D = 0).  The rank-1 update
// forms only the other 15 entries and sets the zeros exactly; the z-shift and the
// Rz rotation of dh_congruence preserve the zero pattern (e_z is their axis), so
// they skip it (the x-shift and Rx rotation fill it).
template <typename T>
__device__ __forceinline__ void sym6_rank1_sub_rev(Sym6<T>& K, const T* u, T invD) {
  T w[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) w[k] = u[k] * invD;
  K.a[0] -= w[0] * u[0]; K.a[1] -= w[1] * u[1]; K.a[2] -= w[2] * u[2];
  K.a[3] -= w[0] * u[1]; K.a[4] -= w[0] * u[2]; K.a[5] -= w[1] * u[2];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    K.b[3 * i] -= w[i] * u[3];
    K.b[3 * i + 1] -= w[i] * u[4];
    K.b[3 * i + 2] = 0;
  }
  K.c[0] -= w[3] * u[3]; K.c[1] -= w[4] * u[4]; K.c[3] -= w[3] * u[4];
  K.c[2] = 0; K.c[4] = 0; K.c[5] = 0;
}
template <typename T>
__device__ __forceinline__ void dh_congruence_rev(T ca, T sa, T a, T d, T s, T c, Sym6<T>& K) {
  {                                                // shift by d e_z (B col 2, C row 2 stay 0)
    const T* A = K.a;
    T* Bm = K.b;
    T* C = K.c;
    const T dd = d * d, d2 = d + d;
    const T b00 = Bm[0], b01 = Bm[1], b10 = Bm[3], b11 = Bm[4];
    C[0] = fma(-d2, b10, fma(dd, A[1], C[0]));
    C[1] = fma(d2, b01, fma(dd, A[0], C[1]));
    C[3] = fma(-d, b11, fma(d, b00, fma(-dd, A[3], C[3])));
    Bm[0] = fma(-d, A[3], b00); Bm[1] = fma(d, A[0], b01);
    Bm[3] = fma(-d, A[1], b10); Bm[4] = fma(d, A[3], b11);
    Bm[6] = fma(-d, A[5], Bm[6]); Bm[7] = fma(d, A[4], Bm[7]);
  }
  sym_rot_plane(K.a, 0, 1, 2, c, s);               // Rz(theta)
  {
    T* b = K.b;                                    // B <- Rz B Rz^T, B(:, 2) = 0 stays 0
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const T bi = b[q], bj = b[3 + q];
      b[q] = fma(c, bi, -(s * bj));
      b[3 + q] = fma(s, bi, c * bj);
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const T bi = b[3 * r], bj = b[3 * r + 1];
      b[3 * r] = fma(c, bi, -(s * bj));
      b[3 * r + 1] = fma(s, bi, c * bj);
    }
    T* C = K.c;                                    // C <- Rz C Rz^T on the xy block only
    const T cc = c * c, ss = s * s, cs = c * s;
    const T cxx = C[0], cyy = C[1], cxy = C[3];
    C[0] = fma(cc, cxx, fma(-2 * cs, cxy, ss * cyy));
    C[1] = fma(ss, cxx, fma(2 * cs, cxy, cc * cyy));
    C[3] = fma(cs, cxx - cyy, (cc - ss) * cxy);
  }
  {                                                // shift by a e_x (sym6_shift_x with B(:, 2) = 0)
    const T* A = K.a;
    T* Bm = K.b;
    T* C = K.c;
    const T aa = a * a, a2 = a + a;
    const T b10 = Bm[3], b11 = Bm[4], b20 = Bm[6], b21 = Bm[7];
    C[1] = fma(-a2, b21, fma(aa, A[2], C[1]));
    C[2] = aa * A[1];
    C[5] = fma(a, b11, -(aa * A[5]));
    C[3] = fma(-a, b20, C[3]);
    C[4] = a * b10;
    Bm[1] = fma(-a, A[4], Bm[1]); Bm[2] = a * A[3];
    Bm[4] = fma(-a, A[5], b11);   Bm[5] = a * A[1];
    Bm[7] = fma(-a, A[2], b21);   Bm[8] = a * A[5];
  }
  sym_rot_plane(K.a, 1, 2, 0, ca, sa);             // Rx(alpha)
  gen_rot_plane(K.b, 1, 2, ca, sa);
  sym_rot_plane(K.c, 1, 2, 0, ca, sa);
}

// K += J for the link inertia J = [[m I, -[h]], [[h], I]]: only its 15 structural
// non-zeros are added.
template <typename T, typename CT>
__device__ __forceinline__ void sym6_add_inertia(const CT& C, Sym6<T>& K) {
  K.a[0] += C.m; K.a[1] += C.m; K.a[2] += C.m;
  const T h0 = C.h[0], h1 = C.h[1], h2 = C.h[2];
  K.b[1] += h2;  K.b[2] -= h1;
  K.b[3] -= h2;  K.b[5] += h0;
  K.b[6] += h1;  K.b[7] -= h0;
#pragma unroll
  for (int k = 0; k < 6; ++k) K.c[k] += C.I[k];
}

// y = y0 + K x for x with x[2] = x[5] = 0 (the ABA's c_i = ad_V(S qd), S = e_z or
// e_5), y0 seeding the chains.
template <typename T, bool R5Z = false>   // R5Z: row / column 5 of K are zero (sym6_rank1_sub_rev)
__device__ __forceinline__ void sym6_mv_xy(const Sym6<T>& K, const T* x, const T* y0, T* y) {
  const T* A = K.a;
  const T* Bm = K.b;
  const T* C = K.c;
  const T x0 = x[0], x1 = x[1], x3 = x[3], x4 = x[4];
  y[0] = fma(A[0], x0, fma(A[3], x1, fma(Bm[0], x3, fma(Bm[1], x4, y0[0]))));
  y[1] = fma(A[3], x0, fma(A[1], x1, fma(Bm[3], x3, fma(Bm[4], x4, y0[1]))));
  y[2] = fma(A[4], x0, fma(A[5], x1, fma(Bm[6], x3, fma(Bm[7], x4, y0[2]))));
  y[3] = fma(Bm[0], x0, fma(Bm[3], x1, fma(C[0], x3, fma(C[3], x4, y0[3]))));
  y[4] = fma(Bm[1], x0, fma(Bm[4], x1, fma(C[3], x3, fma(C[1], x4, y0[4]))));
  y[5] = R5Z ? y0[5] : fma(Bm[2], x0, fma(Bm[5], x1, fma(C[4], x3, fma(C[5], x4, y0[5]))));
}


template <typename T>
__device__ __forceinline__ void dh_sincos(const LinkDH<T>& C, T q, T* s, T* c) {
  if (sizeof(T) == 8) {
    rd_sincos(q + C.th0, s, c);
  } else {
    T s0, c0;
    rd_sincos(q, &s0, &c0);
    *s = fma(s0, C.cth0, c0 * C.sth0);
    *c = fma(c0, C.cth0, -(s0 * C.sth0));
  }
}

}  // namespace rd
