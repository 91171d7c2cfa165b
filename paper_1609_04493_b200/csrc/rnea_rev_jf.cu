// rnea_rev_jf.cu -- strategy REVERSE in JOINT frames: one thread per state, serial
// RNEA (Eq. 1-2) with no per-link stash, for every joint type (revolute,
// prismatic, screw: S_i = (beta e_z, alpha e_z)) and any n.
//
// The DH-frame REVERSE kernel (rnea_rev.cu) needs a DH model; screw joints, and
// chains whose DH frames are ill-conditioned (nearly parallel consecutive axes,
// capi.cu build_dh), used to fall back to GENERIC, whose per-link stash lives in a
// global workspace (~3x slower).  Same scheme as rnea_rev.cu in the joint frames
// of LinkConst: the forward sweep carries V, Vdot (Eq. 1); the backward sweep
// recomputes f_i = (R_i, p_i), Fhat_i = J_i Vdot_i - ad^T_{V_i} J_i V_i and
// Eq. (2), tau_i = S_i^T F_i, and re-derives
//   V_{i-1}    = Ad_{f_i} (V_i - S_i qd_i),
//   Vdot_{i-1} = Ad_{f_i} (Vdot_i - S_i qdd_i - ad_{V_i}(S_i qd_i)).
// Joint origins sit at the links, so the maps stay well conditioned.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"
#include "rd_aba.cuh"

namespace rd {

namespace {

constexpr int kJfThreads = 128;
constexpr int kJfMinBlocks = 4;   // resident CTAs per SM (128-register cap)
constexpr int kJfPD = 4;          // input prefetch distance (links)

// out = Ad_f in, f = (R, p): (R v + p x (R w), R w)
template <typename T>
__device__ __forceinline__ void ad_f(const Rot<T>& R, T p0, T p1, T p2, const T* in, T* out) {
  T w0, w1, w2, v0, v1, v2;
  rot_n(R, in[3], in[4], in[5], w0, w1, w2);
  rot_n(R, in[0], in[1], in[2], v0, v1, v2);
  out[0] = fma(p1, w2, fma(-p2, w1, v0));
  out[1] = fma(p2, w0, fma(-p0, w2, v1));
  out[2] = fma(p0, w1, fma(-p1, w0, v2));
  out[3] = w0; out[4] = w1; out[5] = w2;
}

template <typename T, bool SB>
__global__ void __launch_bounds__(kJfThreads, kJfMinBlocks)
rnea_rev_jf_kernel(int n, const LinkConst<T>* __restrict__ Lg, const Boundary<T> bnd, int64_t B,
                   const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ qdd,
                   T* __restrict__ tau, const typename SBArg<T, SB>::type sb) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LinkConst<T>* L = reinterpret_cast<LinkConst<T>*>(smem_raw);      // model constants, broadcast reads
  for (int i = threadIdx.x; i < n * (int)(sizeof(LinkConst<T>) / sizeof(T)); i += blockDim.x)
    reinterpret_cast<T*>(L)[i] = reinterpret_cast<const T*>(Lg)[i];
  __syncthreads();
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
    const T* pq = q + b;
    const T* pqd = qd + b;
    const T* pqa = qdd + b;
    T V[6], Vd[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) { V[k] = bnd.V0[k]; Vd[k] = bnd.Vd0[k]; }
    if constexpr (SB) {                              // per-state V_0, Vdot_0 (NEXT-4)
      if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, V);
      if (sb.Vd0) sb_vec(sb.Vd0, sb.A0, B, b, Vd);
    }
    // ---- forward sweep, Eq. (1)
    T aq[kJfPD], aqd[kJfPD], aqa[kJfPD];
#pragma unroll
    for (int j = 0; j < kJfPD; ++j) {
      const int64_t o = (int64_t)min(j, n - 1) * B;
      aq[j] = __ldg(pq + o); aqd[j] = __ldg(pqd + o); aqa[j] = __ldg(pqa + o);
    }
#pragma unroll (kJfPD)
    for (int i = 0; i < n; ++i) {
      const T qi = aq[0], qdi = aqd[0], qai = aqa[0];
#pragma unroll
      for (int j = 0; j + 1 < kJfPD; ++j) { aq[j] = aq[j + 1]; aqd[j] = aqd[j + 1]; aqa[j] = aqa[j + 1]; }
      {
        const int64_t o = (int64_t)min(i + kJfPD, n - 1) * B;
        aq[kJfPD - 1] = __ldg(pq + o); aqd[kJfPD - 1] = __ldg(pqd + o); aqa[kJfPD - 1] = __ldg(pqa + o);
      }
      const LinkConst<T>& C = L[i];
      Rot<T> R;
      T p0, p1, p2, s, c, d;
      link_transform(C, qi, R, p0, p1, p2, s, c, d);
      T Vn[6], Vdn[6];
      fwd_step<T, false>(C, R, p0, p1, p2, qdi, qai, V, Vd, Vn, Vdn);
#pragma unroll
      for (int k = 0; k < 6; ++k) { V[k] = Vn[k]; Vd[k] = Vdn[k]; }
    }
    // ---- backward sweep, Eq. (2), re-deriving V, Vdot link by link
    T F[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) F[k] = bnd.Ftip[k];
    if constexpr (SB) {
      if (sb.Ft) sb_vec(sb.Ft, sb.At, B, b, F);
    }
    Rot<T> Rc{1, 0, 0, 0, 1, 0, 0, 0, 1};             // f_{n,n+1} = I (A5)
    T c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
    for (int j = 0; j < kJfPD; ++j) {
      const int64_t o = (int64_t)max(n - 1 - j, 0) * B;
      aq[j] = __ldg(pq + o); aqd[j] = __ldg(pqd + o); aqa[j] = __ldg(pqa + o);
    }
    T tp = 0;                                        // tau of link i+1, stored during link i
#pragma unroll (kJfPD)
    for (int i = n - 1; i >= 0; --i) {
      const T qi = aq[0], qdi = aqd[0], qai = aqa[0];
#pragma unroll
      for (int j = 0; j + 1 < kJfPD; ++j) { aq[j] = aq[j + 1]; aqd[j] = aqd[j + 1]; aqa[j] = aqa[j + 1]; }
      {
        const int64_t o = (int64_t)max(i - kJfPD, 0) * B;
        aq[kJfPD - 1] = __ldg(pq + o); aqd[kJfPD - 1] = __ldg(pqd + o); aqa[kJfPD - 1] = __ldg(pqa + o);
      }
      if (i < n - 1) tau[(int64_t)(i + 1) * B + b] = tp;
      const LinkConst<T>& C = L[i];
      T Fh[6], Fo[6];
      bias_force(C, V, Vd, Fh);
      bwd_step(Rc, c0, c1, c2, F, Fh, Fo);
#pragma unroll
      for (int k = 0; k < 6; ++k) F[k] = Fo[k];
      tp = fma(C.alpha, F[5], C.beta * F[2]);        // tau_i = S_i^T F_i, S_i = (beta e_z, alpha e_z)
      Rot<T> R;
      T p0, p1, p2, s, c, d;
      link_transform(C, qi, R, p0, p1, p2, s, c, d);
      // V_{i-1} = Ad_f (V_i - S qd),  Vdot_{i-1} = Ad_f (Vdot_i - S qdd - ad_{V_i}(S qd))
      const T aqd_ = C.alpha * qdi, bqd = C.beta * qdi;
      T x[6], y[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) { x[k] = V[k]; y[k] = Vd[k]; }
      x[2] -= bqd;
      x[5] -= aqd_;
      y[2] = fma(-C.beta, qai, y[2]);
      y[5] = fma(-C.alpha, qai, y[5]);
      y[0] = fma(-bqd, V[4], fma(-aqd_, V[1], y[0]));
      y[1] = fma(bqd, V[3], fma(aqd_, V[0], y[1]));
      y[3] = fma(-aqd_, V[4], y[3]);
      y[4] = fma(aqd_, V[3], y[4]);
      ad_f(R, p0, p1, p2, x, V);
      ad_f(R, p0, p1, p2, y, Vd);
      Rc = R; c0 = p0; c1 = p1; c2 = p2;
    }
    tau[b] = tp;
  }
}

template <typename T, bool SB>
cudaError_t launch_jf(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q, const T* qd,
                      const T* qdd, T* tau, cudaStream_t st, const typename SBArg<T, SB>::type& sb) {
  const size_t smem = (size_t)n * sizeof(LinkConst<T>);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(rnea_rev_jf_kernel<T, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  int64_t grid = (B + kJfThreads - 1) / kJfThreads;
  const int64_t cap = (int64_t)num_sms() * kJfMinBlocks;
  if (grid > cap) grid = cap;
  rnea_rev_jf_kernel<T, SB><<<(unsigned)grid, kJfThreads, smem, st>>>(n, L_dev, bnd, B, q, qd, qdd, tau, sb);
  return cudaGetLastError();
}

}  // namespace

bool rev_jf_has_n(int n, bool fp64) {
  return n >= 1 && (size_t)n * (fp64 ? sizeof(LinkConst<double>) : sizeof(LinkConst<float>)) <= 200 * 1024;
}

template <typename T>
cudaError_t launch_rnea_rev_jf(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                               const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                               const StateBoundary<T>* sb) {
  if (!rev_jf_has_n(n, sizeof(T) == 8)) return cudaErrorInvalidValue;
  ++*launches;
  if (sb) return launch_jf<T, true>(n, L_dev, bnd, B, q, qd, qdd, tau, st, *sb);
  return launch_jf<T, false>(n, L_dev, bnd, B, q, qd, qdd, tau, st, NoStateBoundary{});
}

template cudaError_t launch_rnea_rev_jf<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                                const double*, const double*, const double*, double*, cudaStream_t,
                                                int*, const StateBoundary<double>*);
template cudaError_t launch_rnea_rev_jf<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                               const float*, const float*, const float*, float*, cudaStream_t, int*,
                                               const StateBoundary<float>*);

}  // namespace rd
