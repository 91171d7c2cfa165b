// rnea_small.cuh -- one thread per state with the WHOLE recursion of Eq. (1)-(2)
// in registers, for short revolute / prismatic chains in DH frames
// (n <= small_max_n<T>(); part of strategy THREAD, rnea_thread.cu takes longer chains).
//
// For a short chain the per-link stash the backward sweep needs, (sin, cos, d,
// Fhat) of every link, fits in registers, so nothing goes through TMEM or shared
// memory and the link loops are unrolled at compile time (template N):
//  * every load of the state's 3N inputs is issued up front (coalesced,
//    x[i*B + b]) and all N sincos are independent of the V chain, so one thread
//    has N-fold instruction-level parallelism where the stash kernel has two
//    chains per step;
//  * the link constants are a __grid_constant__ parameter indexed by compile-time
//    link numbers: they are constant-bank operands of the FP instructions, with no
//    loads and no address arithmetic;
//  * the grid is one thread per state (no tile loop), so the block scheduler
//    spreads a small batch evenly (the paper's 7-DoF arm, BASELINE config C2:
//    n = 7, 1e5 states, is 676 states per SM, which the stash kernel runs as one
//    full and one 32 % tile).
// Same per-link arithmetic as rnea_thread.cu (rd_math.cuh: factored DH maps,
// Newton-Euler bias wrench at the centre of mass).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>
#include "rd_internal.h"
#include "rd_math.cuh"
#include "rd_f32x2.cuh"
#include "rd_small.h"

namespace rd {

template <typename T, int N>
struct SmallParams {
  LinkDHc<T> L[N];
  Boundary<T> bnd;
  uint32_t prism;   // bit k: link k is prismatic (PR instantiation only)
};

// fp32 links on packed pairs (FFMA2) only where that measured faster: n = 7, 8
// (1e6 states: 47.5 -> 39.8 / 47.9 -> 44.7 us); elsewhere the pairs' register
// alignment costs more spills than the halved issue slots save (n = 30, 1e6:
// 0.219 -> 0.304 ms; profiles/r02/ab_small_f32_pack.csv).
__host__ __device__ constexpr bool small_f32_packed(int n) { return n == 7 || n == 8; }
// Backward sweep re-deriving (sin, cos, d) of each link from q instead of keeping
// them (two registers per link instead of six in fp64, for one more sincos per
// link).  Measured (profiles/r02/ab_small_recompute*.csv, 1e6 states): fp64 n = 12
// 66.4 -> 46.1 us at 262k states, 148.7 -> 141.8 us at 1e6 (the stash kernel:
// 148.7); the capped build from n = 7 (n = 8: 104.6 -> 86.9 us); fp32 loses at
// every n (n = 30: 0.220 -> 0.229 ms), its (sin, cos) cost one register each.
template <typename T, int N, int MB>
__host__ __device__ constexpr bool small_recompute() {
  return sizeof(T) == 8 && (N >= 9 || (MB > 1 && N >= 7));
}

// fp32 sin/cos on the SFU (dh_link kSc32Mufu): the fp32 kernel is issue-bound and the
// polynomial is ~20 instructions per link (1e6 states: n = 12 0.0696 -> 0.0663 ms, 20
// 0.1376 -> 0.1198, 30 0.2186 -> 0.2103; fp32 error 1.5e-6 -> 4.8e-6 at n = 30, contract
// 1e-4; profiles/r02/ab_f32_mufu.txt).  (Before: the polynomial pair kSc32Pair for n <= 20,
// profiles/r02/ab_small_f32_sc2.csv.)

// fp32: the same recursion on packed pairs (rd_f32x2.cuh) -- (V_k, Vdot_k) through
// the forward Ad, the ad term and the bias wrench, (f_k, m_k) through the backward
// Ad^T, sin/cos as one polynomial pair: FFMA2 / FMUL2 halve the issue slots.
template <int N, bool PR, bool SB>
__device__ __forceinline__ void small_body_f32x2(const SmallParams<float, N>& P, int64_t B, int64_t b,
                                                 const float* cq, const float* cqd, const float* cqa,
                                                 float* __restrict__ tau, const typename SBArg<float, SB>::type& sb) {
  float V[6], Vd[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) { V[k] = P.bnd.V0[k]; Vd[k] = P.bnd.Vd0[k]; }
  if constexpr (SB) {
    if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, V);
    if (sb.Vd0) sb_vec(sb.Vd0, sb.A0, B, b, Vd);
  }
  float2 VV[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) VV[k] = make_float2(V[k], Vd[k]);
  float ss[N], sc[N], sd[N], Fh[N][6];               // Fh in the pair order (f0, n0, f1, n1, f2, n2)
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const LinkDHc<float>& C = P.L[k];
    const bool prism = PR && ((P.prism >> k) & 1u);
    float s0, c0;
    // sin/cos on the SFU, theta = th0 + q by angle addition (A15); the polynomial pair
    // (sincos_f32x2) was 11 % slower at n = 7, 8 (1e6: 0.0399 / 0.0446 -> 0.0357 / 0.0399 ms)
    sincos_mufu(prism ? 0.f : cq[k], &s0, &c0);
    const float s = fmaf(s0, C.cth0, c0 * C.sth0), c = fmaf(c0, C.cth0, -(s0 * C.sth0));
    const float dl = prism ? C.d + cq[k] : C.d;
    float2 VVn[6];
    dh_ad_finv_x2(C.ca, C.sa, C.a, dl, s, c, VV, VVn);
    const float sr = prism ? 0.f : cqd[k], sp = prism ? cqd[k] : 0.f;
    const float ar = prism ? 0.f : cqa[k], ap = prism ? cqa[k] : 0.f;
    VVn[5].x += sr; VVn[5].y += ar;
    if (PR) { VVn[2].x += sp; VVn[2].y += ap; }
    VVn[0].y = fmaf(sr, VVn[1].x, PR ? fmaf(sp, VVn[4].x, VVn[0].y) : VVn[0].y);
    VVn[1].y = fmaf(-sr, VVn[0].x, PR ? fmaf(-sp, VVn[3].x, VVn[1].y) : VVn[1].y);
    VVn[3].y = fmaf(sr, VVn[4].x, VVn[3].y);
    VVn[4].y = fmaf(-sr, VVn[3].x, VVn[4].y);
    bias_force_com_x2(C, VVn, Fh[k]);
    ss[k] = s; sc[k] = c; sd[k] = dl;
#pragma unroll
    for (int j = 0; j < 6; ++j) VV[j] = VVn[j];
  }
  float F[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) F[k] = P.bnd.Ftip[k];
  if constexpr (SB) {
    if (sb.Ft) sb_vec(sb.Ft, sb.At, B, b, F);
  }
  float2 FF[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) FF[k] = make_float2(F[k], F[k + 3]);
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    if (i == N - 1) {                                // f_{n,n+1} = I (A5)
#pragma unroll
      for (int k = 0; k < 3; ++k) { FF[k].x += Fh[i][2 * k]; FF[k].y += Fh[i][2 * k + 1]; }
    } else {
      const LinkDHc<float>& Cc = P.L[i + 1];
      dh_bwd_x2(Cc.ca, Cc.sa, Cc.a, sd[i + 1], ss[i + 1], sc[i + 1], FF, Fh[i]);
    }
    const bool prism = PR && ((P.prism >> i) & 1u);
    tau[(int64_t)i * B + b] = prism ? FF[2].x : FF[2].y;
  }
}

template <typename T, int N, bool PR, int MB, bool SB>
__global__ void __launch_bounds__(kSmallThreads, MB)
rnea_small_kernel(const __grid_constant__ SmallParams<T, N> P, int64_t B, const T* __restrict__ q,
                  const T* __restrict__ qd, const T* __restrict__ qdd, T* __restrict__ tau,
                  const __grid_constant__ typename SBArg<T, SB>::type sb) {
  const int64_t b = (int64_t)blockIdx.x * kSmallThreads + threadIdx.x;
  if (b >= B) return;
  T cq[N], cqd[N], cqa[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    cq[k] = __ldg(q + (int64_t)k * B + b);
    cqd[k] = __ldg(qd + (int64_t)k * B + b);
    cqa[k] = __ldg(qdd + (int64_t)k * B + b);
  }
  if constexpr (std::is_same<T, float>::value && small_f32_packed(N)) {
    small_body_f32x2<N, PR, SB>(P, B, b, cq, cqd, cqa, tau, sb);
  } else {
    // forward sweep, Eq. (1): V, Vdot; stash (sin, cos, d, Fhat) per link in registers
    T V[6], Vd[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) { V[k] = P.bnd.V0[k]; Vd[k] = P.bnd.Vd0[k]; }
    if constexpr (SB) {                              // per-state V_0, Vdot_0 (NEXT-4)
      if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, V);
      if (sb.Vd0) sb_vec(sb.Vd0, sb.A0, B, b, Vd);
    }
    T ss[N], sc[N], sd[N], Fh[N][6];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const LinkDHc<T>& C = P.L[k];
      const bool prism = PR && ((P.prism >> k) & 1u);
      T s, c, dl;
      dh_link<PR, kSc32Mufu>(C, prism, cq[k], &s, &c, &dl);
      T Vn[6], Vdn[6];
      dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, V, Vn);
      dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, Vd, Vdn);
      // S = (0, e_z) revolute, (e_z, 0) prismatic; ad_V (sp e_z, sr e_z)
      const T sr = prism ? T(0) : cqd[k], sp = prism ? cqd[k] : T(0);
      const T ar = prism ? T(0) : cqa[k], ap = prism ? cqa[k] : T(0);
      Vn[5] += sr;
      Vdn[5] += ar;
      if (PR) { Vn[2] += sp; Vdn[2] += ap; }
      Vdn[0] = fma(sr, Vn[1], PR ? fma(sp, Vn[4], Vdn[0]) : Vdn[0]);
      Vdn[1] = fma(-sr, Vn[0], PR ? fma(-sp, Vn[3], Vdn[1]) : Vdn[1]);
      Vdn[3] = fma(sr, Vn[4], Vdn[3]);
      Vdn[4] = fma(-sr, Vn[3], Vdn[4]);
      bias_force_com(C, Vn, Vdn, Fh[k]);
      if constexpr (!small_recompute<T, N, MB>()) { ss[k] = s; sc[k] = c; sd[k] = dl; }
#pragma unroll
      for (int j = 0; j < 6; ++j) { V[j] = Vn[j]; Vd[j] = Vdn[j]; }
    }
    // backward sweep, Eq. (2): F_i = Fhat_i + Ad^T_{f_{i,i+1}^-1} F_{i+1}, tau_i = S_i^T F_i;
    // f_{n,n+1} = I (A5)
    T F[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) F[k] = P.bnd.Ftip[k];
    if constexpr (SB) {                              // per-state F_{n+1}
      if (sb.Ft) sb_vec(sb.Ft, sb.At, B, b, F);
    }
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
      T Fo[6];
      if (i == N - 1) {
#pragma unroll
        for (int k = 0; k < 6; ++k) Fo[k] = Fh[i][k] + F[k];
      } else {
        const LinkDHc<T>& Cc = P.L[i + 1];
        if constexpr (small_recompute<T, N, MB>()) {       // (sin, cos, d) of link i+1 again from q
          const bool pc = PR && ((P.prism >> (i + 1)) & 1u);
          T s1, c1, d1, qi = cq[i + 1];
          // opaque copy: without it ptxas merges this sincos with the forward one and
          // keeps (sin, cos) live across the sweeps again
          if constexpr (sizeof(T) == 8) asm volatile("mov.b64 %0, %0;" : "+d"(qi));
          else asm volatile("mov.b32 %0, %0;" : "+f"(qi));
          dh_link<PR, kSc32Mufu>(Cc, pc, qi, &s1, &c1, &d1);
          dh_bwd(Cc.ca, Cc.sa, Cc.a, d1, s1, c1, F, Fh[i], Fo);
        } else {
          dh_bwd(Cc.ca, Cc.sa, Cc.a, sd[i + 1], ss[i + 1], sc[i + 1], F, Fh[i], Fo);
        }
      }
#pragma unroll
      for (int k = 0; k < 6; ++k) F[k] = Fo[k];
      const bool prism = PR && ((P.prism >> i) & 1u);
      tau[(int64_t)i * B + b] = prism ? F[2] : F[5];
    }
  }
}

template <typename T, int N, int MB, bool SB>
static void launch_k(const SmallParams<T, N>& P, int64_t grid, int64_t B, const T* q, const T* qd, const T* qdd,
                     T* tau, cudaStream_t st, const typename SBArg<T, SB>::type& sb) {
  if (P.prism)
    rnea_small_kernel<T, N, true, MB, SB><<<(unsigned)grid, kSmallThreads, 0, st>>>(P, B, q, qd, qdd, tau, sb);
  else
    rnea_small_kernel<T, N, false, MB, SB><<<(unsigned)grid, kSmallThreads, 0, st>>>(P, B, q, qd, qdd, tau, sb);
}

template <typename T, int N>
cudaError_t small_launch_n(const LinkDHc<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                            const T* qd, const T* qdd, T* tau, cudaStream_t st, uint32_t prism,
                            const StateBoundary<T>* sb) {
  SmallParams<T, N> P;
  for (int i = 0; i < N; ++i) P.L[i] = L_host[i];
  P.bnd = bnd;
  P.prism = prism;
  const int64_t grid = (B + kSmallThreads - 1) / kSmallThreads;
  if (sb) {                                        // per-state boundary: uncapped build only
    launch_k<T, N, 1, true>(P, grid, B, q, qd, qdd, tau, st, *sb);
  } else if (small_has_cap<T, N>() && B > small_cap_from<T, N>()) {
    launch_k<T, N, small_has_cap<T, N>() ? small_cap_mb<T, N>() : 1, false>(P, grid, B, q, qd, qdd, tau, st,
                                                                             NoStateBoundary{});
  } else {
    launch_k<T, N, 1, false>(P, grid, B, q, qd, qdd, tau, st, NoStateBoundary{});
  }
  return cudaGetLastError();
}

}  // namespace rd

// Explicit instantiations of small_launch_n<T, N> for N = A..Z.
#define RD_SMALL_INST(T, N)                                                                                   \
  template cudaError_t small_launch_n<T, N>(const LinkDHc<T>*, const Boundary<T>&, int64_t, const T*, const T*, \
                                            const T*, T*, cudaStream_t, uint32_t, const StateBoundary<T>*);
