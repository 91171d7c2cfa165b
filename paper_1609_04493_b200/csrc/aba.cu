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
#include <cstdlib>
#include "rd_internal.h"
#include "rd_math.cuh"
#include "rd_aba.cuh"
#include "rd_async.cuh"

namespace rd {

constexpr int kAbaPerLink = 7;   // joint-frame kernel: Ubar = U/D (6), ubar = u/D, SoA [link][7][slot]
constexpr int kAbaThreads = 128;
// The DH kernel's minimum resident CTAs of kAbaThreads per SM (register cap) and the
// depth of its shared-memory ring (stages; sweeps 1 and 3 read kRing - 1 links ahead).
// Measured on B200 (A/B, profiles/r02/ab_aba_ring.txt): fp64 C4 0.442 ms (register
// prefetch, 3 CTAs) -> 0.426 ms (ring 4, 4 CTAs; ring 6 at 3 CTAs 0.437); fp32 C4
// 0.311 -> 0.294 ms with ring 6-7 (ring 4: 0.325) -- fp32 wants depth, fp64 warps.
template <typename T>
struct AbaCfg {
  static constexpr int kMinBlocks = 4;
  static constexpr int kRing = sizeof(T) == 8 ? 4 : 7;
};
int aba_ws_per_link() { return 8; }   // max(kAbaPerLink, AbaWs<double, true>::kV)

// DH kernel workspace: per (link, slot) one contiguous record of kV scalars,
// [link][slot][kV], written by sweep 2 as kChunks 16-byte stores and read back by
// sweep 3 as kChunks 16-byte cp.async copies.  Revolute fp64: (Ubar_0..4, ubar)
// = 48 B (Ubar_5 = 1 is not stored); prismatic fp64: (Ubar_0..5, ubar, pad);
// fp32: 8 scalars (padded to 32 B).
template <typename T, bool PR>
struct AbaWs {
  static constexpr int kV = (sizeof(T) == 8) ? (PR ? 8 : 6) : 8;
  static constexpr int kChunks = kV * (int)sizeof(T) / 16;
  // one ring stage: kChunks x [thread] 16-byte vectors, then q [thread], qd [thread]
  static constexpr int kStageBytes = kAbaThreads * (kChunks * 16 + 2 * (int)sizeof(T));
};

template <typename T, bool SB>
__global__ void __launch_bounds__(kAbaThreads)
aba_kernel(int n, const LinkConst<T>* __restrict__ L, const Boundary<T> bnd, int64_t B,
           const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ tau_in,
           T* __restrict__ qdd_out, T* __restrict__ ws, int64_t slots, int32_t* __restrict__ status,
           const typename SBArg<T, SB>::type sb) {
  const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= slots) return;
  const T zero6[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t b = slot; b < B; b += slots) {
    // ---- sweep 1: link velocities V_i (Eq. 1), registers only; only V_n survives
    T V[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) V[k] = bnd.V0[k];
    if constexpr (SB) {                              // per-state V_0 (NEXT-4)
      if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, V);
    }
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
    int fail = 0;                                         // tip-most link with Omega <= 0 (1-based)
#pragma unroll
    for (int k = 0; k < 6; ++k) pc[k] = bnd.Ftip[k];   // F_{n+1} enters link n like a bias wrench
    if constexpr (SB) {
      if (sb.Ft) sb_vec(sb.Ft, sb.At, B, b, pc);
    }
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
      if (!(D > (T)0) && fail == 0) fail = i + 1;
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
    if (status) status[b] = fail;
    // ---- sweep 3 (forward, the role of Eq. 19): V_i and c_i again, a'_i = X_i a_{i-1} + c_i,
    //      qdd_i = ubar_i - Ubar_i . a'_i, a_i = a'_i + S_i qdd_i
    T a[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) { a[k] = bnd.Vd0[k]; V[k] = bnd.V0[k]; }
    if constexpr (SB) {
      if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, V);
      if (sb.Vd0) sb_vec(sb.Vd0, sb.A0, B, b, a);
    }
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

// ---------------------------------------------------------------- DH-frame variant
// Revolute / prismatic chains in DH frames (the THREAD ID kernel's frames): same
// three sweeps, with the plane-rotation congruence (dh_congruence) and the
// 22-flop Ad maps.  Revolute S = (0, e_z): U = Jhat[:, 5], D = U[5],
// u = tau - phat[5]; prismatic (PR instantiation, per-link flag) S = (e_z, 0):
// U = Jhat[:, 2], D = U[2], u = tau - phat[2], d = d0 + q.
// Shared memory of the DH kernel: constants, prismatic flags, then the ring (16-byte aligned).
template <typename T>
__host__ __device__ constexpr size_t aba_ring_offset(int n, bool PR) {
  return ((size_t)n * sizeof(LinkDH<T>) + (PR ? (size_t)n : 0) + 15) / 16 * 16;
}

template <typename T, int MB, bool PR, bool SB>
__global__ void __launch_bounds__(kAbaThreads, MB)
aba_dh_kernel(int n, const LinkDH<T>* __restrict__ Lg, const Boundary<T> bnd, int64_t B,
              const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ tau_in,
              T* __restrict__ qdd_out, T* __restrict__ ws, int64_t slots, int32_t* __restrict__ status,
              const unsigned char* __restrict__ prism_g, const typename SBArg<T, SB>::type sb) {
  // model constants staged in shared memory (broadcast reads, no long-scoreboard waits)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LinkDH<T>* L = reinterpret_cast<LinkDH<T>*>(smem_raw);
  unsigned char* PRs = smem_raw + (size_t)n * sizeof(LinkDH<T>);   // prismatic flags (PR only)
  // the ring of sweeps 1 and 3 (aba_ring_offset): AbaCfg<T>::kRing stages of AbaWs::kStageBytes
  unsigned char* ring = smem_raw + aba_ring_offset<T>(n, PR);
  for (int i = threadIdx.x; i < n * (int)(sizeof(LinkDH<T>) / sizeof(T)); i += blockDim.x)
    reinterpret_cast<T*>(L)[i] = reinterpret_cast<const T*>(Lg)[i];
  if (PR)
    for (int i = threadIdx.x; i < n; i += blockDim.x) PRs[i] = prism_g[i];
  __syncthreads();
  const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= slots) return;
  const T zero6[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t b = slot; b < B; b += slots) {
    const T* pq = q + b;
    const T* pqd = qd + b;
    const T* pt = tau_in + b;
    T V[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) V[k] = bnd.V0[k];
    if constexpr (SB) {                              // per-state V_0 (NEXT-4)
      if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, V);
    }
    // sweep 1: V_n only.  q, qd stream through the shared-memory ring AbaCfg<T>::kRing - 1
    // links ahead (cp.async; a sweep-1 step is ~45 FP64 instructions, far shorter
    // than a DRAM round trip, and the ring holds no registers)
    const int tid = threadIdx.x;
    using WS = AbaWs<T, PR>;
    auto ring_q = [&](int st) { return reinterpret_cast<T*>(ring + st * WS::kStageBytes + WS::kChunks * 16 * kAbaThreads) + tid; };
    auto ring_ws = [&](int st, int j) {
      return reinterpret_cast<T*>(ring + st * WS::kStageBytes + (j * kAbaThreads + tid) * 16);
    };
    auto issue_in = [&](int j, int st) {          // q, qd of link j into stage st (one group per link)
      if (j < n) {
        cp_async_elem(ring_q(st), pq + (int64_t)j * B);
        cp_async_elem(ring_q(st) + kAbaThreads, pqd + (int64_t)j * B);
      }
    };
    {
#pragma unroll
      for (int j = 0; j < AbaCfg<T>::kRing - 1; ++j) { issue_in(j, j); cp_async_commit(); }
      int st = 0;
      for (int i = 0; i < n; ++i) {
        cp_async_wait<AbaCfg<T>::kRing - 2>();            // link i's group has landed
        const T cq = *ring_q(st), cqd = ring_q(st)[kAbaThreads];
        const int sp = (st == 0) ? AbaCfg<T>::kRing - 1 : st - 1;   // consumed one step ago
        issue_in(i + AbaCfg<T>::kRing - 1, sp);
        cp_async_commit();
        st = (st == AbaCfg<T>::kRing - 1) ? 0 : st + 1;
        const LinkDH<T>& C = L[i];
        T Vn[6];
        if constexpr (PR) {
          const bool pz = PRs[i];
          T s, c, dl;
          dh_link<PR>(C, pz, cq, &s, &c, &dl);
          dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, V, Vn);
          Vn[5] += pz ? T(0) : cqd;
          Vn[2] += pz ? cqd : T(0);
        } else {
          T s, c;
          dh_sincos(C, cq, &s, &c);
          dh_ad_finv(C, s, c, V, Vn);
          Vn[5] += cqd;
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) V[k] = Vn[k];
      }
    }
    Sym6<T> K;                                            // carried X^T Jhat^a X (0 at the tip)
    T pc[6];
    int fail = 0;                                         // tip-most link with Omega <= 0 (1-based)
#pragma unroll
    for (int k = 0; k < 6; ++k) { pc[k] = bnd.Ftip[k]; K.a[k] = 0; K.c[k] = 0; }
    if constexpr (SB) {
      if (sb.Ft) sb_vec(sb.Ft, sb.At, B, b, pc);
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) K.b[k] = 0;
    // sweep 2 (backward); inputs one link ahead (each iteration is long)
    T cq = __ldg(pq + (int64_t)(n - 1) * B), cqd = __ldg(pqd + (int64_t)(n - 1) * B),
      ct = __ldg(pt + (int64_t)(n - 1) * B);
    for (int i = n - 1; i >= 0; --i) {
      const int64_t o = (int64_t)max(i - 1, 0) * B;
      const T nq = __ldg(pq + o), nqd = __ldg(pqd + o), nt = __ldg(pt + o);
      const LinkDH<T>& C = L[i];
      const bool pz = PR && PRs[i];
      T s, c, dl;
      const T qdi = cqd;
      T cc[6];
      if constexpr (PR) {
        dh_link<PR>(C, pz, cq, &s, &c, &dl);
        // c_i = ad_V(S qd), S qd = (sp e_z, sr e_z)
        const T sr = pz ? T(0) : qdi, sp = pz ? qdi : T(0);
        cc[0] = fma(sp, V[4], sr * V[1]); cc[1] = -fma(sp, V[3], sr * V[0]); cc[2] = 0;
        cc[3] = sr * V[4]; cc[4] = -sr * V[3]; cc[5] = 0;
      } else {
        dh_sincos(C, cq, &s, &c);
        dl = C.d;
        cc[0] = qdi * V[1]; cc[1] = -qdi * V[0]; cc[2] = 0; cc[3] = qdi * V[4]; cc[4] = -qdi * V[3]; cc[5] = 0;
      }
      T ph[6];
      bias_force_v(C, V, pc, ph);                         // phat_i = p_i + X^T p^a_{i+1}
      sym6_add_inertia(C, K);                             // Jhat_i = J_i + X^T Jhat^a_{i+1} X
      // revolute: U = K e_5 = (B[:, 2], C[:, 2]); prismatic: U = K e_2 = (A[:, 2], B[2, :])
      T U[6] = {K.b[2], K.b[5], K.b[8], K.c[4], K.c[5], K.c[2]};
      if (PR && pz) {
        U[0] = K.a[4]; U[1] = K.a[5]; U[2] = K.a[2];
        U[3] = K.b[6]; U[4] = K.b[7]; U[5] = K.b[8];
      }
      const T D = (PR && pz) ? U[2] : U[5];
      const T invD = (D > (T)0) ? (T)1 / D : (T)NAN;
      if (!(D > (T)0) && fail == 0) fail = i + 1;
      const T ub = (ct - ((PR && pz) ? ph[2] : ph[5])) * invD;
      {                                                   // one record [link][slot][kV], 16-byte stores
        T rec[WS::kV];
#pragma unroll
        for (int k = 0; k < 5; ++k) rec[k] = U[k] * invD;
        if constexpr (WS::kV == 6) {
          rec[5] = ub;                                    // revolute fp64: Ubar_5 = U_5 / D = 1, not stored
        } else {
          rec[5] = U[5] * invD;
          rec[6] = ub;
          rec[7] = T(0);
        }
        T* w = ws + ((int64_t)i * slots + slot) * WS::kV;
#pragma unroll
        for (int j = 0; j < WS::kChunks; ++j)
          *reinterpret_cast<uint4*>(w + j * (16 / sizeof(T))) = *reinterpret_cast<const uint4*>(rec + j * (16 / sizeof(T)));
      }
      if (i > 0) {
        if constexpr (PR) sym6_rank1_sub(K, U, invD);     // Jhat^a
        else sym6_rank1_sub_rev(K, U, invD);
        T y0[6], pa[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) y0[k] = fma(U[k], ub, ph[k]);
        sym6_mv_xy<T, !PR>(K, cc, y0, pa);                // p^a = phat + Jhat^a c + U u / D
        if constexpr (PR) {
          dh_congruence(C.ca, C.sa, C.a, dl, s, c, K);
          dh_bwd(C.ca, C.sa, C.a, dl, s, c, pa, zero6, pc);
        } else {
          dh_congruence_rev(C.ca, C.sa, C.a, C.d, s, c, K);
          dh_bwd(C.ca, C.sa, C.a, C.d, s, c, pa, zero6, pc);
        }
        T x[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) x[k] = V[k];
        if constexpr (PR) {
          x[5] -= pz ? T(0) : qdi;
          x[2] -= pz ? qdi : T(0);
          dh_ad_f(C.ca, C.sa, C.a, dl, s, c, x, V);   // V_{i-1} = Ad_{f_i}(V_i - S qd)
        } else {
          x[5] -= qdi;
          dh_ad_f(C, s, c, x, V);
        }
      }
      cq = nq; cqd = nqd; ct = nt;
    }
    if (status) status[b] = fail;
    // sweep 3 (forward): a'_i = X_i a_{i-1} + c_i, qdd_i = ubar_i - Ubar_i . a'_i
    T a[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) { a[k] = bnd.Vd0[k]; V[k] = bnd.V0[k]; }
    if constexpr (SB) {
      if (sb.V0) sb_vec(sb.V0, sb.A0, B, b, V);
      if (sb.Vd0) sb_vec(sb.Vd0, sb.A0, B, b, a);
    }
    {
      // (Ubar, ubar) records, q and qd of link i + AbaCfg<T>::kRing - 1 are copied into the
      // ring while link i computes: the workspace comes back from DRAM (560 MB at
      // C4 does not fit in L2) and a sweep-3 step is short
      auto issue_all = [&](int j, int st) {
        if (j < n) {
          const T* w = ws + ((int64_t)j * slots + slot) * WS::kV;
#pragma unroll
          for (int c = 0; c < WS::kChunks; ++c) cp_async_16(ring_ws(st, c), w + c * (16 / sizeof(T)));
          issue_in(j, st);
        }
      };
#pragma unroll
      for (int j = 0; j < AbaCfg<T>::kRing - 1; ++j) { issue_all(j, j); cp_async_commit(); }
      int st = 0;
      for (int i = 0; i < n; ++i) {
        cp_async_wait<AbaCfg<T>::kRing - 2>();
        T rec[WS::kV];
#pragma unroll
        for (int c = 0; c < WS::kChunks; ++c)
          *reinterpret_cast<uint4*>(rec + c * (16 / sizeof(T))) = *reinterpret_cast<const uint4*>(ring_ws(st, c));
        const T cq3 = *ring_q(st), cqd3 = ring_q(st)[kAbaThreads];
        const int sp = (st == 0) ? AbaCfg<T>::kRing - 1 : st - 1;
        issue_all(i + AbaCfg<T>::kRing - 1, sp);
        cp_async_commit();
        st = (st == AbaCfg<T>::kRing - 1) ? 0 : st + 1;
        T Ub[6];
#pragma unroll
        for (int k = 0; k < 5; ++k) Ub[k] = rec[k];
        Ub[5] = (WS::kV == 6) ? T(1) : rec[5];
        const T ub = (WS::kV == 6) ? rec[5] : rec[6];
        const LinkDH<T>& C = L[i];
        const bool pz = PR && PRs[i];
        const T qdi = cqd3;
        T Vn[6], an[6];
        if constexpr (PR) {
          T s, c, dl;
          dh_link<PR>(C, pz, cq3, &s, &c, &dl);
          const T sr = pz ? T(0) : qdi, sp2 = pz ? qdi : T(0);
          dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, V, Vn);
          Vn[5] += sr;
          Vn[2] += sp2;
          dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, a, an);
          an[0] = fma(sr, Vn[1], fma(sp2, Vn[4], an[0]));
          an[1] = fma(-sr, Vn[0], fma(-sp2, Vn[3], an[1]));
          an[3] = fma(sr, Vn[4], an[3]);
          an[4] = fma(-sr, Vn[3], an[4]);
        } else {
          T s, c;
          dh_sincos(C, cq3, &s, &c);
          dh_ad_finv(C, s, c, V, Vn);
          Vn[5] += qdi;
          dh_ad_finv(C, s, c, a, an);
          an[0] = fma(qdi, Vn[1], an[0]);
          an[1] = fma(-qdi, Vn[0], an[1]);
          an[3] = fma(qdi, Vn[4], an[3]);
          an[4] = fma(-qdi, Vn[3], an[4]);
        }
        T Ua = 0;
#pragma unroll
        for (int k = 0; k < 6; ++k) Ua = fma(Ub[k], an[k], Ua);
        const T qddi = ub - Ua;
        qdd_out[(int64_t)i * B + b] = qddi;
        if (PR && pz) an[2] += qddi;
        else an[5] += qddi;
#pragma unroll
        for (int k = 0; k < 6; ++k) { a[k] = an[k]; V[k] = Vn[k]; }
      }
    }
  }
}

template <typename T, bool PR, bool SB>
static cudaError_t launch_aba_dh_pr(int n, const LinkDH<T>* L_dev, const Boundary<T>& bnd, int64_t B,
                                    const T* q, const T* qd, const T* tau, T* qdd, T* ws, int64_t ws_slots,
                                    cudaStream_t st, int32_t* status, const unsigned char* prism,
                                    const typename SBArg<T, SB>::type& sb) {
  const int64_t grid = (ws_slots + kAbaThreads - 1) / kAbaThreads;
  const size_t smem = aba_ring_offset<T>(n, PR) + (size_t)AbaCfg<T>::kRing * AbaWs<T, PR>::kStageBytes;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(aba_dh_kernel<T, AbaCfg<T>::kMinBlocks, PR, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  aba_dh_kernel<T, AbaCfg<T>::kMinBlocks, PR, SB><<<(unsigned)grid, kAbaThreads, smem, st>>>(n, L_dev, bnd, B, q, qd, tau, qdd, ws,
                                                                          ws_slots, status, prism, sb);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_aba_dh(int n, const LinkDH<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                          const T* qd, const T* tau, T* qdd, T* ws, int64_t ws_slots, cudaStream_t st,
                          int* launches, int32_t* status, const unsigned char* prism,
                          const StateBoundary<T>* sb) {
  ++*launches;
  const NoStateBoundary nsb{};
  if (sb)
    return prism ? launch_aba_dh_pr<T, true, true>(n, L_dev, bnd, B, q, qd, tau, qdd, ws, ws_slots, st, status,
                                                   prism, *sb)
                 : launch_aba_dh_pr<T, false, true>(n, L_dev, bnd, B, q, qd, tau, qdd, ws, ws_slots, st, status,
                                                    nullptr, *sb);
  return prism ? launch_aba_dh_pr<T, true, false>(n, L_dev, bnd, B, q, qd, tau, qdd, ws, ws_slots, st, status,
                                                  prism, nsb)
               : launch_aba_dh_pr<T, false, false>(n, L_dev, bnd, B, q, qd, tau, qdd, ws, ws_slots, st, status,
                                                   nullptr, nsb);
}
template cudaError_t launch_aba_dh<double>(int, const LinkDH<double>*, const Boundary<double>&, int64_t,
                                           const double*, const double*, const double*, double*, double*, int64_t,
                                           cudaStream_t, int*, int32_t*, const unsigned char*,
                                           const StateBoundary<double>*);
template cudaError_t launch_aba_dh<float>(int, const LinkDH<float>*, const Boundary<float>&, int64_t,
                                          const float*, const float*, const float*, float*, float*, int64_t,
                                          cudaStream_t, int*, int32_t*, const unsigned char*,
                                          const StateBoundary<float>*);

template <typename T>
cudaError_t launch_aba(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                       const T* qd, const T* tau, T* qdd, T* ws, int64_t ws_slots, cudaStream_t st,
                       int* launches, int32_t* status, const StateBoundary<T>* sb) {
  const int64_t grid = (ws_slots + kAbaThreads - 1) / kAbaThreads;
  if (sb)
    aba_kernel<T, true><<<(unsigned)grid, kAbaThreads, 0, st>>>(n, L_dev, bnd, B, q, qd, tau, qdd, ws, ws_slots,
                                                                 status, *sb);
  else
    aba_kernel<T, false><<<(unsigned)grid, kAbaThreads, 0, st>>>(n, L_dev, bnd, B, q, qd, tau, qdd, ws, ws_slots,
                                                                  status, NoStateBoundary{});
  ++*launches;
  return cudaGetLastError();
}

template cudaError_t launch_aba<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                        const double*, const double*, const double*, double*, double*, int64_t,
                                        cudaStream_t, int*, int32_t*, const StateBoundary<double>*);
template cudaError_t launch_aba<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                       const float*, const float*, const float*, float*, float*, int64_t,
                                       cudaStream_t, int*, int32_t*, const StateBoundary<float>*);

}  // namespace rd
