// aba_small_jf.cu -- forward dynamics by the articulated-body algorithm (Eq. 7-8,
// P:104-140) for short chains of ANY joint type in JOINT frames, with the per-link
// records in registers (FD algorithm ABA for models without a well-conditioned DH
// form: screw joints, calibrated arms with nearly parallel axes; capi.cu build_dh).
//
// The three sweeps of aba_kernel (aba.cu, joint frames, global workspace) with the
// link loops unrolled at compile time (template N): sweep 1 forward to V_n; sweep 2
// backward (ABI Eq. 7 with the articulated bias, V re-derived by the inverse map),
// keeping Ubar = U/D and ubar = u/D of each link in registers; sweep 3 forward
// (accelerations, qdd).  Link constants are a __grid_constant__ parameter with
// compile-time indices.  D_i <= 0 (A11) makes that state's qdd NaN.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"
#include "rd_aba.cuh"

namespace rd {

namespace {

constexpr int kAbaJfThreads = 128;

template <typename T, int N>
struct AbaJfParams {
  LinkConst<T> L[N];
  Boundary<T> bnd;
};

template <typename T, int N, bool SB>
__global__ void __launch_bounds__(kAbaJfThreads)
aba_small_jf_kernel(const __grid_constant__ AbaJfParams<T, N> P, int64_t B, const T* __restrict__ q,
                    const T* __restrict__ qd, const T* __restrict__ tau_in, T* __restrict__ qdd_out,
                    int32_t* __restrict__ status, const __grid_constant__ typename SBArg<T, SB>::type sb) {
  const int64_t b = (int64_t)blockIdx.x * kAbaJfThreads + threadIdx.x;
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
    const LinkConst<T>& C = P.L[k];
    Rot<T> R;
    T p0, p1, p2, s, c, d, Vn[6];
    link_transform(C, cq[k], R, p0, p1, p2, s, c, d);
    ad_finv(R, p0, p1, p2, V, Vn);
    Vn[2] = fma(C.beta, cqd[k], Vn[2]);
    Vn[5] = fma(C.alpha, cqd[k], Vn[5]);
#pragma unroll
    for (int j = 0; j < 6; ++j) V[j] = Vn[j];
  }
  // ---- sweep 2 (backward): Eq. (7) and the articulated bias; records in registers
  T Ub[N][6], ubr[N];
  Sym6<T> K, Kc;
  T pc[6];
  int fail = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) { pc[k] = P.bnd.Ftip[k]; Kc.a[k] = 0; Kc.c[k] = 0; }
#pragma unroll
  for (int k = 0; k < 9; ++k) Kc.b[k] = 0;
  if constexpr (SB) {
    if (sb.Ft) sb_vec(sb.Ft, sb.At, B, b, pc);
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    const LinkConst<T>& C = P.L[i];
    Rot<T> R;
    T p0, p1, p2, s, c, d;
    link_transform(C, cq[i], R, p0, p1, p2, s, c, d);
    const T aq = C.alpha * cqd[i], bq = C.beta * cqd[i];
    // c_i = ad_V(S qd), p_i = -ad^T_V J V
    T cc[6];
    cc[0] = fma(bq, V[4], aq * V[1]);
    cc[1] = -fma(bq, V[3], aq * V[0]);
    cc[2] = 0;
    cc[3] = aq * V[4];
    cc[4] = -aq * V[3];
    cc[5] = 0;
    T ph[6];
    bias_force_v(C, V, pc, ph);                          // phat_i = p_i + X^T p^a_{i+1}
    link_inertia(C, K);
#pragma unroll
    for (int k = 0; k < 6; ++k) { K.a[k] += Kc.a[k]; K.c[k] += Kc.c[k]; }
#pragma unroll
    for (int k = 0; k < 9; ++k) K.b[k] += Kc.b[k];
    T U[6];
    {
      const T e[6] = {0, 0, C.beta, 0, 0, C.alpha};
      sym6_mv(K, e, U);                                  // U = Jhat S
    }
    const T D = fma(C.beta, U[2], C.alpha * U[5]);       // D = S^T U (= Omega)
    const T invD = (D > (T)0) ? (T)1 / D : (T)NAN;       // A11: per-state NaN
    if (!(D > (T)0) && fail == 0) fail = i + 1;
    const T ub = (ct[i] - fma(C.beta, ph[2], C.alpha * ph[5])) * invD;
#pragma unroll
    for (int k = 0; k < 6; ++k) Ub[i][k] = U[k] * invD;
    ubr[i] = ub;
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
    const LinkConst<T>& C = P.L[i];
    Rot<T> R;
    T p0, p1, p2, s, c, d;
    link_transform(C, cq[i], R, p0, p1, p2, s, c, d);
    T Vn[6], an[6];
    ad_finv(R, p0, p1, p2, V, Vn);
    Vn[2] = fma(C.beta, cqd[i], Vn[2]);
    Vn[5] = fma(C.alpha, cqd[i], Vn[5]);
    ad_finv(R, p0, p1, p2, a, an);
    const T aq = C.alpha * cqd[i], bq = C.beta * cqd[i];
    an[0] += fma(bq, Vn[4], aq * Vn[1]);
    an[1] -= fma(bq, Vn[3], aq * Vn[0]);
    an[3] += aq * Vn[4];
    an[4] -= aq * Vn[3];
    T Ua = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) Ua = fma(Ub[i][k], an[k], Ua);
    const T qddi = ubr[i] - Ua;
    qdd_out[(int64_t)i * B + b] = qddi;
    an[2] = fma(C.beta, qddi, an[2]);
    an[5] = fma(C.alpha, qddi, an[5]);
#pragma unroll
    for (int k = 0; k < 6; ++k) { a[k] = an[k]; V[k] = Vn[k]; }
  }
}

template <typename T, int N>
cudaError_t launch_n(const LinkConst<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q, const T* qd,
                     const T* tau, T* qdd, cudaStream_t st, int32_t* status, const StateBoundary<T>* sb) {
  AbaJfParams<T, N> P;
  for (int i = 0; i < N; ++i) P.L[i] = L_host[i];
  P.bnd = bnd;
  const unsigned grid = (unsigned)((B + kAbaJfThreads - 1) / kAbaJfThreads);
  if (sb)
    aba_small_jf_kernel<T, N, true><<<grid, kAbaJfThreads, 0, st>>>(P, B, q, qd, tau, qdd, status, *sb);
  else
    aba_small_jf_kernel<T, N, false><<<grid, kAbaJfThreads, 0, st>>>(P, B, q, qd, tau, qdd, status,
                                                                      NoStateBoundary{});
  return cudaGetLastError();
}

template <typename T, int N>
cudaError_t dispatch(int n, const LinkConst<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q, const T* qd,
                     const T* tau, T* qdd, cudaStream_t st, int32_t* status, const StateBoundary<T>* sb) {
  if (n == N) return launch_n<T, N>(L_host, bnd, B, q, qd, tau, qdd, st, status, sb);
  if constexpr (N > 1) return dispatch<T, N - 1>(n, L_host, bnd, B, q, qd, tau, qdd, st, status, sb);
  return cudaErrorInvalidValue;
}

template <typename T>
constexpr int aba_jf_max_n() { return sizeof(T) == 8 ? 8 : 12; }

}  // namespace

bool aba_small_jf_has_n(int n, bool fp64) {
  return n >= 1 && n <= (fp64 ? aba_jf_max_n<double>() : aba_jf_max_n<float>());
}

template <typename T>
cudaError_t launch_aba_small_jf(int n, const LinkConst<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                                const T* qd, const T* tau, T* qdd, cudaStream_t st, int* launches, int32_t* status,
                                const StateBoundary<T>* sb) {
  if (!aba_small_jf_has_n(n, sizeof(T) == 8)) return cudaErrorInvalidValue;
  ++*launches;
  return dispatch<T, aba_jf_max_n<T>()>(n, L_host, bnd, B, q, qd, tau, qdd, st, status, sb);
}

template cudaError_t launch_aba_small_jf<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                                 const double*, const double*, const double*, double*, cudaStream_t,
                                                 int*, int32_t*, const StateBoundary<double>*);
template cudaError_t launch_aba_small_jf<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                                const float*, const float*, const float*, float*, cudaStream_t, int*,
                                                int32_t*, const StateBoundary<float>*);

}  // namespace rd
