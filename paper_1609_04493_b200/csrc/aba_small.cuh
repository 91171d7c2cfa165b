// aba_small.cuh -- forward dynamics (articulated-body algorithm, Eq. 7-8,
// P:104-140) for short revolute / prismatic chains in DH frames with the whole
// per-link workspace in registers (FD algorithm ABA for n <= aba_small_max_n;
// aba.cu takes longer chains).
//
// Same three sweeps and arithmetic as aba_dh_kernel (aba.cu): sweep 1 forward to
// V_n, sweep 2 backward (ABI Eq. 7 with the articulated bias, V re-derived by
// the inverse map), sweep 3 forward (accelerations, qdd).  What differs is where
// sweep 2's per-link record (Ubar = U/D, ubar = u/D) lives: in registers (the link
// loops are unrolled at compile time, template N), not in a global workspace that
// sweep 3 reads back, and the link constants are a __grid_constant__ parameter
// indexed by compile-time link numbers (constant-bank operands).  One thread per
// state, one state per thread, no tile loop.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"
#include "rd_aba.cuh"

namespace rd {

constexpr int kAbaSmallThreads = 128;

template <typename T, int N>
struct AbaSmallParams {
  LinkDH<T> L[N];
  Boundary<T> bnd;
  uint32_t prism;   // bit k: link k is prismatic (PR instantiation only)
};

template <typename T, int N, bool PR, bool SB, int MB>
__global__ void __launch_bounds__(kAbaSmallThreads, MB)
aba_small_kernel(const __grid_constant__ AbaSmallParams<T, N> P, int64_t B, const T* __restrict__ q,
                 const T* __restrict__ qd, const T* __restrict__ tau_in, T* __restrict__ qdd_out,
                 int32_t* __restrict__ status, const __grid_constant__ typename SBArg<T, SB>::type sb) {
  const int64_t b = (int64_t)blockIdx.x * kAbaSmallThreads + threadIdx.x;
  if (b >= B) return;
  const T zero6[6] = {0, 0, 0, 0, 0, 0};
  T cq[N], cqd[N], ct[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    cq[k] = __ldg(q + (int64_t)k * B + b);
    cqd[k] = __ldg(qd + (int64_t)k * B + b);
    ct[k] = __ldg(tau_in + (int64_t)k * B + b);
  }
  // ---- sweep 1: V_n (Eq. 1 with qdd = 0)
  T V[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) V[k] = P.bnd.V0[k];
  if constexpr (SB) {
    if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, V);
  }
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const LinkDH<T>& C = P.L[k];
    const bool pz = PR && ((P.prism >> k) & 1u);
    T s, c, dl, Vn[6];
    dh_link<PR>(C, pz, cq[k], &s, &c, &dl);
    dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, V, Vn);
    Vn[5] += pz ? T(0) : cqd[k];
    if (PR) Vn[2] += pz ? cqd[k] : T(0);
#pragma unroll
    for (int j = 0; j < 6; ++j) V[j] = Vn[j];
  }
  // ---- sweep 2 (backward): Eq. (7) and the articulated bias; records in registers
  constexpr int kV = PR ? 7 : 6;                   // Ubar_0..4 (+ Ubar_5 prismatic), ubar
  T rec[N][kV];
  Sym6<T> K;
  T pc[6];
  int fail = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) { pc[k] = P.bnd.Ftip[k]; K.a[k] = 0; K.c[k] = 0; }
#pragma unroll
  for (int k = 0; k < 9; ++k) K.b[k] = 0;
  if constexpr (SB) {
    if (sb.Ft) sb_vec(sb.Ft, sb.At, B, b, pc);
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    const LinkDH<T>& C = P.L[i];
    const bool pz = PR && ((P.prism >> i) & 1u);
    const T qdi = cqd[i];
    T s, c, dl;
    dh_link<PR>(C, pz, cq[i], &s, &c, &dl);
    // c_i = ad_V(S qd), S qd = (sp e_z, sr e_z)
    const T sr = pz ? T(0) : qdi, sp = pz ? qdi : T(0);
    T cc[6];
    cc[0] = PR ? fma(sp, V[4], sr * V[1]) : sr * V[1];
    cc[1] = PR ? -fma(sp, V[3], sr * V[0]) : -(sr * V[0]);
    cc[2] = 0; cc[3] = sr * V[4]; cc[4] = -sr * V[3]; cc[5] = 0;
    T ph[6];
    bias_force_v(C, V, pc, ph);                         // phat_i = p_i + X^T p^a_{i+1}
    sym6_add_inertia(C, K);                             // Jhat_i = J_i + X^T Jhat^a_{i+1} X
    T U[6] = {K.b[2], K.b[5], K.b[8], K.c[4], K.c[5], K.c[2]};   // revolute: U = K e_5
    if (PR && pz) {                                     // prismatic: U = K e_2
      U[0] = K.a[4]; U[1] = K.a[5]; U[2] = K.a[2];
      U[3] = K.b[6]; U[4] = K.b[7]; U[5] = K.b[8];
    }
    const T D = (PR && pz) ? U[2] : U[5];
    const T invD = (D > (T)0) ? (T)1 / D : (T)NAN;     // A11: per-state NaN
    if (!(D > (T)0) && fail == 0) fail = i + 1;
    const T ub = (ct[i] - ((PR && pz) ? ph[2] : ph[5])) * invD;
#pragma unroll
    for (int k = 0; k < 5; ++k) rec[i][k] = U[k] * invD;
    if constexpr (PR) rec[i][5] = U[5] * invD;
    rec[i][kV - 1] = ub;
    if (i > 0) {
      if constexpr (PR) sym6_rank1_sub(K, U, invD);     // Jhat^a
      else sym6_rank1_sub_rev(K, U, invD);
      T y0[6], pa[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) y0[k] = fma(U[k], ub, ph[k]);
      sym6_mv_xy<T, !PR>(K, cc, y0, pa);                // p^a = phat + Jhat^a c + U u / D
      if constexpr (PR) dh_congruence(C.ca, C.sa, C.a, dl, s, c, K);
      else dh_congruence_rev(C.ca, C.sa, C.a, dl, s, c, K);
      dh_bwd(C.ca, C.sa, C.a, dl, s, c, pa, zero6, pc);
      T x[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) x[k] = V[k];
      x[5] -= sr;
      if (PR) x[2] -= sp;
      dh_ad_f(C.ca, C.sa, C.a, dl, s, c, x, V);         // V_{i-1} = Ad_{f_i}(V_i - S qd)
    }
  }
  if (status) status[b] = fail;
  // ---- sweep 3 (forward, the role of Eq. 19): a'_i = X_i a_{i-1} + c_i,
  //      qdd_i = ubar_i - Ubar_i . a'_i, a_i = a'_i + S_i qdd_i
  T a[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) { a[k] = P.bnd.Vd0[k]; V[k] = P.bnd.V0[k]; }
  if constexpr (SB) {
    if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, V);
    if (sb.Vd0) sb_vec(sb.Vd0, sb.A0, B, b, a);
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const LinkDH<T>& C = P.L[i];
    const bool pz = PR && ((P.prism >> i) & 1u);
    const T qdi = cqd[i];
    const T sr = pz ? T(0) : qdi, sp = pz ? qdi : T(0);
    T s, c, dl, Vn[6], an[6];
    dh_link<PR>(C, pz, cq[i], &s, &c, &dl);
    dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, V, Vn);
    Vn[5] += sr;
    if (PR) Vn[2] += sp;
    dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, a, an);
    an[0] = fma(sr, Vn[1], PR ? fma(sp, Vn[4], an[0]) : an[0]);
    an[1] = fma(-sr, Vn[0], PR ? fma(-sp, Vn[3], an[1]) : an[1]);
    an[3] = fma(sr, Vn[4], an[3]);
    an[4] = fma(-sr, Vn[3], an[4]);
    const T Ub5 = PR ? rec[i][PR ? 5 : 0] : T(1);       // revolute: Ubar_5 = U_5 / D = 1
    T Ua = fma(Ub5, an[5], T(0));
#pragma unroll
    for (int k = 0; k < 5; ++k) Ua = fma(rec[i][k], an[k], Ua);
    const T qddi = rec[i][kV - 1] - Ua;
    qdd_out[(int64_t)i * B + b] = qddi;
    if (PR && pz) an[2] += qddi;
    else an[5] += qddi;
#pragma unroll
    for (int k = 0; k < 6; ++k) { a[k] = an[k]; V[k] = Vn[k]; }
  }
}

template <typename T, int N>
cudaError_t aba_small_launch_n(const LinkDH<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                               const T* qd, const T* tau, T* qdd, cudaStream_t st, int32_t* status,
                               uint32_t prism, const StateBoundary<T>* sb) {
  AbaSmallParams<T, N> P;
  for (int i = 0; i < N; ++i) P.L[i] = L_host[i];
  P.bnd = bnd;
  P.prism = prism;
  const unsigned grid = (unsigned)((B + kAbaSmallThreads - 1) / kAbaSmallThreads);
  // no register cap: capping fp64 at 3-4 CTAs/SM measured slower or equal from n = 6 on
  // (n = 8, 1e6: 218 us uncapped, 240 / 226 us at 3 / 4 CTAs; profiles/r02/ab_aba_small.csv)
  constexpr int MB = 1;
  if (sb) {
    if (prism)
      aba_small_kernel<T, N, true, true, MB><<<grid, kAbaSmallThreads, 0, st>>>(P, B, q, qd, tau, qdd, status, *sb);
    else
      aba_small_kernel<T, N, false, true, MB><<<grid, kAbaSmallThreads, 0, st>>>(P, B, q, qd, tau, qdd, status, *sb);
  } else {
    if (prism)
      aba_small_kernel<T, N, true, false, MB><<<grid, kAbaSmallThreads, 0, st>>>(P, B, q, qd, tau, qdd, status,
                                                                                 NoStateBoundary{});
    else
      aba_small_kernel<T, N, false, false, MB><<<grid, kAbaSmallThreads, 0, st>>>(P, B, q, qd, tau, qdd, status,
                                                                                  NoStateBoundary{});
  }
  return cudaGetLastError();
}

}  // namespace rd

#define RD_ABA_SMALL_INST(T, N)                                                                                \
  template cudaError_t aba_small_launch_n<T, N>(const LinkDH<T>*, const Boundary<T>&, int64_t, const T*,      \
                                                const T*, const T*, T*, cudaStream_t, int32_t*, uint32_t,     \
                                                const StateBoundary<T>*);
