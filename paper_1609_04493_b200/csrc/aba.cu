// aba.cu -- batched forward dynamics qdd = FD(q, qd, tau, V_0, Vdot_0, F_{n+1})
// (Eq. 4) by the articulated-body algorithm, one thread per state.
//
// The paper's hybrid ABIA (Alg. 3) computes tau_bias with the ID
// scans, the ABI recursion Eq. (7) serially (on the CPU there), then the
// linear Eq. (18)/(19) scans.  Here all of it stays on the GPU in three sweeps
// per state:
//   1. forward  (Eq. 1 with qdd = 0): f_i, V_i, c_i = ad_{V_i}(S_i qd_i),
//      bias wrench p_i = -ad^T_{V_i} J_i V_i             (the tau_bias part, Eq. 5)
//   2. backward (Eq. 7, the unscannable Riccati step, serial per state):
//      U_i = Jhat_i S_i, D_i = S_i^T U_i (= Omega_i), u_i = tau_i - S_i^T phat_i,
//      Jhat^a = Jhat - U U^T / D,  p^a = phat + Jhat^a c + U u / D,
//      Jhat_{i-1} = J_{i-1} + X_i^T Jhat^a X_i,  phat_{i-1} = p_{i-1} + X_i^T p^a
//      (the articulated-bias recursion plays the role of Eq. (18)/(20))
//   3. forward (the role of Eq. 19): a'_i = X_i a_{i-1} + c_i (a_0 = Vdot_0),
//      qdd_i = (u_i - U_i^T a'_i) / D_i,  a_i = a'_i + S_i qdd_i.
// X_i = Ad_{f_{i-1,i}^{-1}}.  Memory-lean: sweeps 1 and 3 recompute the transforms
// and velocities instead of storing them, sweep 2 re-derives V_{i-1} from V_i by
// inverting the forward map; the only per-link scratch is Ubar = U/D and
// ubar = u/D (7 scalars) written by sweep 2 and read by sweep 3, in a
// slot-contiguous global workspace.  D_i <= 0 (A11) makes that state's qdd NaN.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"

namespace rd {

constexpr int kAbaPerLink = 7;   // Ubar = U/D (6), ubar = u/D
constexpr int kAbaThreads = 128;
int aba_ws_per_link() { return kAbaPerLink; }

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

template <typename T>
__global__ void __launch_bounds__(kAbaThreads)
aba_kernel(int n, const LinkConst<T>* __restrict__ L, const Boundary<T> bnd, int64_t B,
           const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ tau_in,
           T* __restrict__ qdd_out, T* __restrict__ ws, int64_t slots) {
  const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= slots) return;
  const T zero6[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t b = slot; b < B; b += slots) {
    // ---- sweep 1: link velocities V_i (Eq. 1), registers only; only V_n survives
    T V[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) V[k] = bnd.V0[k];
    for (int i = 0; i < n; ++i) {
      const LinkConst<T> C = L[i];
      Rot<T> R;
      T p0, p1, p2, s, c, d;
      link_transform(C, __ldg(q + (int64_t)i * B + b), R, p0, p1, p2, s, c, d);
      const T qdi = __ldg(qd + (int64_t)i * B + b);
      T Vn[6];
      ad_finv(R, p0, p1, p2, V, Vn);
      Vn[2] = fma(C.beta, qdi, Vn[2]);
      Vn[5] = fma(C.alpha, qdi, Vn[5]);
#pragma unroll
      for (int k = 0; k < 6; ++k) V[k] = Vn[k];
    }
    // ---- sweep 2 (backward): ABI Eq. (7) and articulated bias; V_i re-derived by
    //      V_{i-1} = Ad_{f_i}(V_i - S_i qd_i); stores Ubar = U/D and ubar = u/D (7 per link)
    Sym6<T> K, Kc;
    T ph[6], pc[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) pc[k] = bnd.Ftip[k];   // F_{n+1} enters link n like a bias wrench
#pragma unroll
    for (int k = 0; k < 6; ++k) { Kc.a[k] = 0; Kc.c[k] = 0; }
#pragma unroll
    for (int k = 0; k < 9; ++k) Kc.b[k] = 0;
    for (int i = n - 1; i >= 0; --i) {
      const LinkConst<T> C = L[i];
      Rot<T> R;
      T p0, p1, p2, s, c, d;
      link_transform(C, __ldg(q + (int64_t)i * B + b), R, p0, p1, p2, s, c, d);
      const T qdi = __ldg(qd + (int64_t)i * B + b);
      // c_i = ad_{V_i}(S qd) = qd (beta w x e_z + alpha v x e_z, alpha w x e_z); p_i = -ad^T_V J V
      const T aq = C.alpha * qdi, bq = C.beta * qdi;
      T cc[6];
      cc[0] = fma(bq, V[4], aq * V[1]);
      cc[1] = -fma(bq, V[3], aq * V[0]);
      cc[2] = 0;
      cc[3] = aq * V[4];
      cc[4] = -aq * V[3];
      cc[5] = 0;
      T pb[6];
      bias_force(C, V, zero6, pb);
      link_inertia(C, K);
#pragma unroll
      for (int k = 0; k < 6; ++k) { K.a[k] += Kc.a[k]; K.c[k] += Kc.c[k]; ph[k] = pb[k] + pc[k]; }
#pragma unroll
      for (int k = 0; k < 9; ++k) K.b[k] += Kc.b[k];
      // U = Jhat S, D = S^T U (= Omega), u = tau - S^T phat
      T U[6];
      {
        const T e[6] = {0, 0, C.beta, 0, 0, C.alpha};
        sym6_mv(K, e, U);
      }
      const T D = fma(C.beta, U[2], C.alpha * U[5]);
      const T u = __ldg(tau_in + (int64_t)i * B + b) - fma(C.beta, ph[2], C.alpha * ph[5]);
      const T invD = (D > (T)0) ? (T)1 / D : (T)NAN;      // A11: per-state NaN
      const T ub = u * invD;
      T* w = ws + (int64_t)i * kAbaPerLink * slots + slot;
#pragma unroll
      for (int k = 0; k < 6; ++k) w[k * slots] = U[k] * invD;
      w[6 * slots] = ub;
      if (i > 0) {
        // Jhat^a = Jhat - U U^T / D ; p^a = phat + Jhat^a c + U u / D, moved to the parent
        sym6_rank1_sub(K, U, invD);
        T Kcc[6], pa[6];
        sym6_mv(K, cc, Kcc);
#pragma unroll
        for (int k = 0; k < 6; ++k) pa[k] = ph[k] + Kcc[k] + U[k] * ub;
        congruence(R, p0, p1, p2, K, Kc);
        bwd_step(R, p0, p1, p2, pa, zero6, pc);
        // V_{i-1} = Ad_{f_i}(V_i - S qd)
        T x[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) x[k] = V[k];
        x[2] -= bq;
        x[5] -= aq;
        T vr[3], wr[3];
        rot_n(R, x[3], x[4], x[5], wr[0], wr[1], wr[2]);
        rot_n(R, x[0], x[1], x[2], vr[0], vr[1], vr[2]);
        V[0] = fma(p1, wr[2], fma(-p2, wr[1], vr[0]));
        V[1] = fma(p2, wr[0], fma(-p0, wr[2], vr[1]));
        V[2] = fma(p0, wr[1], fma(-p1, wr[0], vr[2]));
        V[3] = wr[0]; V[4] = wr[1]; V[5] = wr[2];
      }
    }
    // ---- sweep 3 (forward, the role of Eq. 19): V_i and c_i again, a'_i = X_i a_{i-1} + c_i,
    //      qdd_i = ubar_i - Ubar_i . a'_i, a_i = a'_i + S_i qdd_i
    T a[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) { a[k] = bnd.Vd0[k]; V[k] = bnd.V0[k]; }
    for (int i = 0; i < n; ++i) {
      const LinkConst<T> C = L[i];
      const T* w = ws + (int64_t)i * kAbaPerLink * slots + slot;
      T Ub[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) Ub[k] = w[k * slots];
      const T ub = w[6 * slots];
      Rot<T> R;
      T p0, p1, p2, s, c, d;
      link_transform(C, __ldg(q + (int64_t)i * B + b), R, p0, p1, p2, s, c, d);
      const T qdi = __ldg(qd + (int64_t)i * B + b);
      T Vn[6], an[6];
      ad_finv(R, p0, p1, p2, V, Vn);
      Vn[2] = fma(C.beta, qdi, Vn[2]);
      Vn[5] = fma(C.alpha, qdi, Vn[5]);
      ad_finv(R, p0, p1, p2, a, an);
      const T aq = C.alpha * qdi, bq = C.beta * qdi;
      an[0] += fma(bq, Vn[4], aq * Vn[1]);
      an[1] -= fma(bq, Vn[3], aq * Vn[0]);
      an[3] += aq * Vn[4];
      an[4] -= aq * Vn[3];
      T Ua = 0;
#pragma unroll
      for (int k = 0; k < 6; ++k) Ua = fma(Ub[k], an[k], Ua);
      const T qddi = ub - Ua;
      qdd_out[(int64_t)i * B + b] = qddi;
      an[2] = fma(C.beta, qddi, an[2]);
      an[5] = fma(C.alpha, qddi, an[5]);
#pragma unroll
      for (int k = 0; k < 6; ++k) { a[k] = an[k]; V[k] = Vn[k]; }
    }
  }
}

template <typename T>
cudaError_t launch_aba(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                       const T* qd, const T* tau, T* qdd, T* ws, int64_t ws_slots, cudaStream_t st,
                       int* launches) {
  const int64_t grid = (ws_slots + kAbaThreads - 1) / kAbaThreads;
  aba_kernel<T><<<(unsigned)grid, kAbaThreads, 0, st>>>(n, L_dev, bnd, B, q, qd, tau, qdd, ws, ws_slots);
  ++*launches;
  return cudaGetLastError();
}

template cudaError_t launch_aba<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                        const double*, const double*, const double*, double*, double*, int64_t,
                                        cudaStream_t, int*);
template cudaError_t launch_aba<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                       const float*, const float*, const float*, float*, float*, int64_t,
                                       cudaStream_t, int*);

}  // namespace rd
