// rnea_rev.cu -- one thread per state, serial RNEA (Eq. 1-2) with NO
// per-link stash, for long all-revolute chains (strategy REVERSE, any n).
//
// The forward sweep carries only V, Vdot (Eq. 1).  The backward sweep re-derives
// V_{i-1}, Vdot_{i-1} from V_i, Vdot_i by inverting the forward maps,
//   V_{i-1}    = Ad_{f_i} (V_i - S_i qd_i),
//   Vdot_{i-1} = Ad_{f_i} (Vdot_i - S_i qdd_i - ad_{V_i}(S_i qd_i)),
// recomputes f_i (sincos) and the bias wrench Fhat_i there, and runs Eq. (2).
// Inputs are re-read in the backward sweep (L2).  The per-state on-chip state is
// a few dozen registers whatever n is, so the kernel keeps 16 warps per SM busy
// where the stash kernel (rnea_thread.cu) cannot fit n links on chip.
// Rigid transforms are well conditioned, so the re-derivation adds O(n eps)
// relative error (GPU parity tests up to n = 200).  DH frames as in rnea_thread.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"

namespace rd {

constexpr int kRevThreads = 128;
// Input prefetch distance (links) and unroll of both sweeps: unrolling by the
// distance keeps the in-flight loads in fixed registers (no MOV rotation that
// waits on them at every loop head); tau is stored one link late, off the end
// of the backward DFMA chain (thread kernel).
constexpr int kRevPD = 4, kRevU = 4;
constexpr int kRevMinBlocks = 4;   // resident CTAs per SM (128-register cap)

template <typename T, bool PR, bool SB>
__global__ void __launch_bounds__(kRevThreads, kRevMinBlocks)
rnea_rev_kernel(int n, const LinkDHc<T>* __restrict__ Lg, const Boundary<T> bnd, int64_t B,
                const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ qdd,
                T* __restrict__ tau, const unsigned char* __restrict__ prism_g,
                const typename SBArg<T, SB>::type sb) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LinkDHc<T>* L = reinterpret_cast<LinkDHc<T>*>(smem_raw);       // model constants, broadcast reads
  unsigned char* PRs = smem_raw + (size_t)n * sizeof(LinkDHc<T>);   // prismatic flags (PR only)
  for (int i = threadIdx.x; i < n * (int)(sizeof(LinkDHc<T>) / sizeof(T)); i += blockDim.x)
    reinterpret_cast<T*>(L)[i] = reinterpret_cast<const T*>(Lg)[i];
  if (PR)
    for (int i = threadIdx.x; i < n; i += blockDim.x) PRs[i] = prism_g[i];
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
    constexpr int PD = kRevPD;
    T aq[PD], aqd[PD], aqa[PD];
#pragma unroll
    for (int j = 0; j < PD; ++j) {
      const int64_t o = (int64_t)min(j, n - 1) * B;
      aq[j] = __ldg(pq + o); aqd[j] = __ldg(pqd + o); aqa[j] = __ldg(pqa + o);
    }
#pragma unroll (kRevU)
    for (int i = 0; i < n; ++i) {
      const T qi = aq[0], qdi = aqd[0], qai = aqa[0];
#pragma unroll
      for (int j = 0; j + 1 < PD; ++j) { aq[j] = aq[j + 1]; aqd[j] = aqd[j + 1]; aqa[j] = aqa[j + 1]; }
      {
        const int64_t o = (int64_t)min(i + PD, n - 1) * B;
        aq[PD - 1] = __ldg(pq + o); aqd[PD - 1] = __ldg(pqd + o); aqa[PD - 1] = __ldg(pqa + o);
      }
      const LinkDHc<T> C = L[i];
      const bool pz = PR && PRs[i];
      T s, c, dl;
      dh_link<PR, kSc32Pair>(C, pz, qi, &s, &c, &dl);   // fp32: paired sin/cos (n = 100, 1e6: 1.144 -> 1.083 ms)
      T Vn[6], Vdn[6];
      dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, V, Vn);
      dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, Vd, Vdn);
      // S qd = (sp e_z, sr e_z); ad_V(S qd) = (sp w x e_z + sr v x e_z, sr w x e_z)
      const T sr = pz ? T(0) : qdi, sp = pz ? qdi : T(0), ar = pz ? T(0) : qai, ap = pz ? qai : T(0);
      Vn[5] += sr;
      Vdn[5] += ar;
      if (PR) { Vn[2] += sp; Vdn[2] += ap; }
      Vdn[0] = fma(sr, Vn[1], PR ? fma(sp, Vn[4], Vdn[0]) : Vdn[0]);
      Vdn[1] = fma(-sr, Vn[0], PR ? fma(-sp, Vn[3], Vdn[1]) : Vdn[1]);
      Vdn[3] = fma(sr, Vn[4], Vdn[3]);
      Vdn[4] = fma(-sr, Vn[3], Vdn[4]);
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
    T ca = 1, sa = 0, ac = 0, dc = 0, sn = 0, cn = 1;   // child transform (identity at the tip)
#pragma unroll
    for (int j = 0; j < PD; ++j) {
      const int64_t o = (int64_t)max(n - 1 - j, 0) * B;
      aq[j] = __ldg(pq + o); aqd[j] = __ldg(pqd + o); aqa[j] = __ldg(pqa + o);
    }
    T tp = 0;                                   // tau of link i+1, stored during link i
#pragma unroll (kRevU)
    for (int i = n - 1; i >= 0; --i) {
      const T qi = aq[0], qdi = aqd[0], qai = aqa[0];
#pragma unroll
      for (int j = 0; j + 1 < PD; ++j) { aq[j] = aq[j + 1]; aqd[j] = aqd[j + 1]; aqa[j] = aqa[j + 1]; }
      {
        const int64_t o = (int64_t)max(i - PD, 0) * B;
        aq[PD - 1] = __ldg(pq + o); aqd[PD - 1] = __ldg(pqd + o); aqa[PD - 1] = __ldg(pqa + o);
      }
      if (i < n - 1) tau[(int64_t)(i + 1) * B + b] = tp;
      const LinkDHc<T> C = L[i];
      const bool pz = PR && PRs[i];
      T Fh[6], Fo[6];
      bias_force_com(C, V, Vd, Fh);
      dh_bwd(ca, sa, ac, dc, sn, cn, F, Fh, Fo);
#pragma unroll
      for (int k = 0; k < 6; ++k) F[k] = Fo[k];
      tp = pz ? F[2] : F[5];                        // tau_i = S_i^T F_i
      T s, c, dl;
      dh_link<PR, kSc32Pair>(C, pz, qi, &s, &c, &dl);   // fp32: paired sin/cos (n = 100, 1e6: 1.144 -> 1.083 ms)
      // V_{i-1}, Vdot_{i-1}
      const T sr = pz ? T(0) : qdi, sp = pz ? qdi : T(0), ar = pz ? T(0) : qai, ap = pz ? qai : T(0);
      T x[6], y[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) { x[k] = V[k]; y[k] = Vd[k]; }
      x[5] -= sr;
      y[5] -= ar;
      if (PR) { x[2] -= sp; y[2] -= ap; }
      y[0] = fma(-sr, V[1], PR ? fma(-sp, V[4], y[0]) : y[0]);
      y[1] = fma(sr, V[0], PR ? fma(sp, V[3], y[1]) : y[1]);
      y[3] = fma(-sr, V[4], y[3]);
      y[4] = fma(sr, V[3], y[4]);
      dh_ad_f(C.ca, C.sa, C.a, dl, s, c, x, V);
      dh_ad_f(C.ca, C.sa, C.a, dl, s, c, y, Vd);
      ca = C.ca; sa = C.sa; ac = C.a; dc = dl; sn = s; cn = c;
    }
    tau[b] = tp;
  }
}

template <typename T, bool PR, bool SB>
static cudaError_t launch_rev(int n, const LinkDHc<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                              const T* qd, const T* qdd, T* tau, cudaStream_t st, const unsigned char* prism,
                              const typename SBArg<T, SB>::type& sb) {
  const size_t smem = (size_t)n * sizeof(LinkDHc<T>) + (PR ? (size_t)n : 0);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(rnea_rev_kernel<T, PR, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  int64_t grid = (B + kRevThreads - 1) / kRevThreads;
  const int64_t cap = (int64_t)num_sms() * kRevMinBlocks;
  if (grid > cap) grid = cap;
  rnea_rev_kernel<T, PR, SB><<<(unsigned)grid, kRevThreads, smem, st>>>(n, L_dev, bnd, B, q, qd, qdd, tau, prism,
                                                                         sb);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_rnea_rev(int n, const LinkDHc<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                            const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                            const unsigned char* prism, const StateBoundary<T>* sb) {
  ++*launches;
  if (sb)
    return prism ? launch_rev<T, true, true>(n, L_dev, bnd, B, q, qd, qdd, tau, st, prism, *sb)
                 : launch_rev<T, false, true>(n, L_dev, bnd, B, q, qd, qdd, tau, st, nullptr, *sb);
  return prism ? launch_rev<T, true, false>(n, L_dev, bnd, B, q, qd, qdd, tau, st, prism, NoStateBoundary{})
               : launch_rev<T, false, false>(n, L_dev, bnd, B, q, qd, qdd, tau, st, nullptr, NoStateBoundary{});
}

template cudaError_t launch_rnea_rev<double>(int, const LinkDHc<double>*, const Boundary<double>&, int64_t,
                                             const double*, const double*, const double*, double*, cudaStream_t,
                                             int*, const unsigned char*, const StateBoundary<double>*);
template cudaError_t launch_rnea_rev<float>(int, const LinkDHc<float>*, const Boundary<float>&, int64_t,
                                            const float*, const float*, const float*, float*, cudaStream_t, int*,
                                            const unsigned char*, const StateBoundary<float>*);

}  // namespace rd
