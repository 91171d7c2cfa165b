// fd_scan.cu -- forward dynamics as the paper's hybrid ABIA, Alg. 3,
// with every step on the GPU (FD strategy SCAN, n <= 32):
//   line 1    tau_bias = CalcInvDyn(q, qd, 0)       -> rnea_warp kernel (qdd = 0), Eq. (5)
//   line 2    tau_hat  = tau - tau_bias             -> fused into the scan kernel
//   line 3    CalcABI (Eq. 7, the unscannable Riccati step; on the CPU in the
//             paper) -> abi_kernel: one thread per state, serial over links
//   line 4    CalcInterIntVar Omega_i, Pi_{i-1,i} (Y is rebuilt from Pi, below)
//   line 5    InclusiveZhatScan  (Eq. 18)          -> fd_scan_kernel, one warp per state,
//   line 6    CalcChat                                lane = link: Kogge-Stone suffix scan of
//   line 7    InclusiveLambdaScan (Eq. 19)            the affine maps z -> Y z + Pi tau_hat,
//   line 8    CalcAcc                                 then prefix scan of lam -> Y^T lam + S chat
// Scan operands are the structured affine maps (6x6 linear part + offset); the
// 8x8 lifts of Eq. (18)/(19) carry an extra chat row, which here is the map of
// line 6 (A7: Omega^{-1}).  In 0-based link j with X_j = Ad_{f_j^{-1}}:
//   Pi_j = X_j^T U_j / D_j, U_j = Jhat_j S_j, D_j = Omega_j = S_j^T U_j,
//   Y_j  = X_j^T (I - U_j S_j^T / D_j) = X_j^T - Pi_j S_j^T,
//   zhat_{j-1} = Y_j zhat_j + Pi_j tau_hat_j (zhat_{n-1} = 0),
//   chat_j = (tau_hat_j - S_j^T zhat_j) / Omega_j,
//   lam_j = Y_j^T lam_{j-1} + S_j chat_j (lam_{-1} = 0),  qdd_j = chat_j - Pi_j^T lam_{j-1}.
// Expected slower than the fused thread-per-state ABA (aba.cu): each scan level
// composes 6x6 operators.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"
#include "rd_aba.cuh"
#include "rd_scan.cuh"

namespace rd {

constexpr int kAbiThreads = 128;
constexpr int kScanWarps = 4;
constexpr int kPiPerLink = 7;          // Pi (6), Omega (1)

// ---------------------------------------------------------------- Alg. 3 lines 3-4
template <typename T>
__global__ void __launch_bounds__(kAbiThreads)
abi_kernel(int n, const LinkConst<T>* __restrict__ L, int64_t B, const T* __restrict__ q, T* __restrict__ pi_ws,
           int32_t* __restrict__ status) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
    Sym6<T> K, Kc;
#pragma unroll
    for (int k = 0; k < 6; ++k) { Kc.a[k] = 0; Kc.c[k] = 0; }
#pragma unroll
    for (int k = 0; k < 9; ++k) Kc.b[k] = 0;
    int fail = 0;                                   // tip-most link with Omega <= 0 (1-based)
    for (int j = n - 1; j >= 0; --j) {
      const LinkConst<T> C = L[j];
      Rot<T> R;
      T p0, p1, p2, s, c, d;
      link_transform(C, __ldg(q + (int64_t)j * B + b), R, p0, p1, p2, s, c, d);
      // Jhat_j = J_j + X_{j+1}^T Jhat^a_{j+1} X_{j+1}  (Eq. 7)
      link_inertia(C, K);
#pragma unroll
      for (int k = 0; k < 6; ++k) { K.a[k] += Kc.a[k]; K.c[k] += Kc.c[k]; }
#pragma unroll
      for (int k = 0; k < 9; ++k) K.b[k] += Kc.b[k];
      T U[6];
      {
        const T e[6] = {0, 0, C.beta, 0, 0, C.alpha};
        sym6_mv(K, e, U);
      }
      const T D = fma(C.beta, U[2], C.alpha * U[5]);
      const T invD = (D > (T)0) ? (T)1 / D : (T)NAN;
      if (!(D > (T)0) && fail == 0) fail = j + 1;
      // Pi_j = X_j^T U / D = (R u_f, p x R u_f + R u_m) / D
      T Ud[6], Pi[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) Ud[k] = U[k] * invD;
      const T zero6[6] = {0, 0, 0, 0, 0, 0};
      bwd_step(R, p0, p1, p2, Ud, zero6, Pi);
      T* w = pi_ws + (int64_t)j * kPiPerLink * B + b;
#pragma unroll
      for (int k = 0; k < 6; ++k) w[(int64_t)k * B] = Pi[k];
      w[(int64_t)6 * B] = D;
      if (j > 0) {
        sym6_rank1_sub(K, U, invD);
        congruence(R, p0, p1, p2, K, Kc);
      }
    }
    if (status) status[b] = fail;
  }
}

// Per-lane (lane = link j) quantities of lines 4-8: (R, p) of f_j, Pi_j, Omega_j
// and Y_j = X_j^T - Pi_j S_j^T; identity Y / zero Pi on lanes >= n.
template <typename T>
__device__ __forceinline__ void scan_link_setup(bool act, const LinkConst<T>& C, int n, int64_t B, int64_t b,
                                                int lane, const T* __restrict__ q, const T* __restrict__ pi_ws,
                                                T (&Y)[36], T (&Pi)[6], T& D, Rot<T>& R, T& p0, T& p1, T& p2) {
  if (act) {
    T s, c, d;
    link_transform(C, __ldg(q + (int64_t)lane * B + b), R, p0, p1, p2, s, c, d);
    const T* w = pi_ws + (int64_t)lane * kPiPerLink * B + b;
#pragma unroll
    for (int k = 0; k < 6; ++k) Pi[k] = __ldg(w + (int64_t)k * B);
    D = __ldg(w + (int64_t)6 * B);
    // X^T = Ad^T_{f^-1} = [[R, 0], [[p]R, R]];  Y = X^T - Pi S^T, S = (beta e_z, alpha e_z)
    const T r[9] = {R.r00, R.r01, R.r02, R.r10, R.r11, R.r12, R.r20, R.r21, R.r22};
#pragma unroll
    for (int i = 0; i < 36; ++i) Y[i] = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        Y[6 * i + j] = r[3 * i + j];
        Y[6 * (3 + i) + 3 + j] = r[3 * i + j];
      }
    // [p]R rows: (p x R[:, j])
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const T x0 = r[j], x1 = r[3 + j], x2 = r[6 + j];
      Y[6 * 3 + j] = p1 * x2 - p2 * x1;
      Y[6 * 4 + j] = p2 * x0 - p0 * x2;
      Y[6 * 5 + j] = p0 * x1 - p1 * x0;
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      Y[6 * i + 2] = fma(-Pi[i], C.beta, Y[6 * i + 2]);
      Y[6 * i + 5] = fma(-Pi[i], C.alpha, Y[6 * i + 5]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 36; ++i) Y[i] = (i % 7 == 0) ? T(1) : T(0);   // identity map
#pragma unroll
    for (int i = 0; i < 6; ++i) Pi[i] = 0;
    D = 1;
    R.r00 = R.r11 = R.r22 = 1;
    R.r01 = R.r02 = R.r10 = R.r12 = R.r20 = R.r21 = 0;
    p0 = p1 = p2 = 0;
  }
}

// ---------------------------------------------------------------- Alg. 3 lines 2, 5-8
template <typename T>
__global__ void __launch_bounds__(kScanWarps * 32)
fd_scan_kernel(int n, const LinkConst<T>* __restrict__ Lg, int64_t B, const T* __restrict__ q,
               const T* __restrict__ tau_in, const T* __restrict__ tau_bias, const T* __restrict__ pi_ws,
               T* __restrict__ qdd_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool act = lane < n;
  LinkConst<T> C;
  if (act) C = Lg[lane];
  for (int64_t b = (int64_t)blockIdx.x * kScanWarps + warp; b < B; b += (int64_t)gridDim.x * kScanWarps) {
    T Y[36], zb[6], Pi[6], D = 1, th = 0, al = 0, be = 0;
    Rot<T> R;
    T p0, p1, p2;
    scan_link_setup(act, C, n, B, b, lane, q, pi_ws, Y, Pi, D, R, p0, p1, p2);
    if (act) {
      th = __ldg(tau_in + (int64_t)lane * B + b) - __ldg(tau_bias + (int64_t)lane * B + b);   // line 2
      al = C.alpha;
      be = C.beta;
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) zb[i] = Pi[i] * th;
    // line 5: suffix scan of z -> Y z + Pi tau_hat (own operand on the left)
    T Lm[36];
#pragma unroll
    for (int i = 0; i < 36; ++i) Lm[i] = Y[i];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) compose_shfl<T, true>(Lm, zb, d, lane + d < 32);
    // zhat_j = offset of the composite starting at j+1
    T z[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const T o = __shfl_down_sync(0xffffffffu, zb[k], 1);
      z[k] = (lane + 1 < n) ? o : T(0);
    }
    // line 6: chat_j = (tau_hat_j - S_j^T zhat_j) / Omega_j
    const T ch = (th - fma(be, z[2], al * z[5])) / D;
    // line 7: prefix scan of lam -> Y^T lam + S chat (own operand on the left)
    T lb[6];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = 0; j < 6; ++j) Lm[6 * i + j] = Y[6 * j + i];
#pragma unroll
    for (int k = 0; k < 6; ++k) lb[k] = 0;
    lb[2] = be * ch;
    lb[5] = al * ch;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) compose_shfl<T, false>(Lm, lb, d, lane >= d);
    // line 8: qdd_j = chat_j - Pi_j^T lam_{j-1}
    T acc = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const T lp = __shfl_up_sync(0xffffffffu, lb[k], 1);
      acc = fma(Pi[k], lane > 0 ? lp : T(0), acc);
    }
    if (act) qdd_out[(int64_t)lane * B + b] = ch - acc;
  }
}

// ---------------------------------------------------------------- Eq. (20) merged backward scan
// NEXT-2 variant (FD algorithm ABA_MERGED, n <= 31): lines 1-2 and 5-6 of Alg. 3
// replaced by ONE backward scan of the Eq. (20) operators (A7
// Omega^{-1}, A8 seeding), acting on x_i = (F_{i-1}, tau_hat_i, zhat_i, chat_{i+1}, 1)
// (paper index i = n..0, 1-based links):
//   F_{i-1}    = Ad^T_{f_{i-1,i}^{-1}} F_i + Fhat_{i-1}        (bias-force recursion, qdd = 0)
//   tau_hat_i  = tau_i - S_i^T F_i
//   zhat_i     = Pi_{i,i+1} tau_hat_{i+1} + Y_{i,i+1} zhat_{i+1}
//   chat_{i+1} = Omega_{i+1}^{-1} (tau_hat_{i+1} - S_{i+1}^T zhat_{i+1})
// seeded with (F_n, 0, 0, 0, 1), F_n = Fhat_n + F_{n+1}.  One warp per state,
// lane l = n - i holds A_i; the inclusive scan composes own-on-the-left
// (x_i = A_i(...A_n(seed))).  The operators keep the block pattern
//   F <- F;  t <- F;  z <- F, t, z;  c <- F, t, z  (+ offsets), 147 scalars,
// stored [field][lane] in shared memory (double-buffered: the composition reads
// the partner lane's operator).  Fhat comes from the warp-scan ID (qdd = 0)
// and Pi, Omega from abi_kernel, as in fd_scan_kernel; the Eq. (19) forward
// scan is the same as there.
namespace mop {   // field offsets of one operator
constexpr int FF = 0, Fo = 36, tF = 42, to = 48, zF = 49, zt = 85, zz = 91, zo = 127, cF = 133, ct = 139,
              cz = 140, co = 146, NF = 147;
}
constexpr int kMergedWarps = 3;   // 3 x 2 x 147 x 32 x 8 B = 221 KB of shared memory (fp64)

// C = Bop o Aop (Aop applied first); Bop = lane's own operator, Aop = the partner's.
template <typename T>
__device__ __noinline__ void mop_compose(const T* __restrict__ sb, int own, int src, T* __restrict__ sn) {
  using namespace mop;
  auto Bv = [&](int f) { return sb[f * 32 + own]; };
  auto Av = [&](int f) { return sb[f * 32 + src]; };
  auto Cw = [&](int f, T v) { sn[f * 32 + own] = v; };
#pragma unroll 1
  for (int i = 0; i < 6; ++i) {
    T bff[6], bzf[6], bzz[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) { bff[k] = Bv(FF + 6 * i + k); bzf[k] = Bv(zF + 6 * i + k); bzz[k] = Bv(zz + 6 * i + k); }
    const T bzt = Bv(zt + i);
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      T f = 0, zf = bzt * Av(tF + j), zzv = 0;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const T aff = Av(FF + 6 * k + j);
        f = fma(bff[k], aff, f);
        zf = fma(bzf[k], aff, zf);
        zf = fma(bzz[k], Av(zF + 6 * k + j), zf);
        zzv = fma(bzz[k], Av(zz + 6 * k + j), zzv);
      }
      Cw(FF + 6 * i + j, f);
      Cw(zF + 6 * i + j, zf);
      Cw(zz + 6 * i + j, zzv);
    }
    T fo = Bv(Fo + i), zo_ = fma(bzt, Av(to), Bv(zo + i)), ztv = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      fo = fma(bff[k], Av(Fo + k), fo);
      zo_ = fma(bzf[k], Av(Fo + k), zo_);
      zo_ = fma(bzz[k], Av(zo + k), zo_);
      ztv = fma(bzz[k], Av(zt + k), ztv);
    }
    Cw(Fo + i, fo);
    Cw(zo + i, zo_);
    Cw(zt + i, ztv);
  }
  // scalar rows t and c
  T btf[6], bcf[6], bcz[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) { btf[k] = Bv(tF + k); bcf[k] = Bv(cF + k); bcz[k] = Bv(cz + k); }
  const T bct = Bv(ct);
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    T tf = 0, cf = bct * Av(tF + j), czv = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const T aff = Av(FF + 6 * k + j);
      tf = fma(btf[k], aff, tf);
      cf = fma(bcf[k], aff, cf);
      cf = fma(bcz[k], Av(zF + 6 * k + j), cf);
      czv = fma(bcz[k], Av(zz + 6 * k + j), czv);
    }
    Cw(tF + j, tf);
    Cw(cF + j, cf);
    Cw(cz + j, czv);
  }
  T tov = Bv(to), cov = fma(bct, Av(to), Bv(co)), ctv = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    tov = fma(btf[k], Av(Fo + k), tov);
    cov = fma(bcf[k], Av(Fo + k), cov);
    cov = fma(bcz[k], Av(zo + k), cov);
    ctv = fma(bcz[k], Av(zt + k), ctv);
  }
  Cw(to, tov);
  Cw(co, cov);
  Cw(ct, ctv);
}

template <typename T>
__global__ void __launch_bounds__(kMergedWarps * 32)
fd_merged_kernel(int n, const LinkConst<T>* __restrict__ Lg, const Boundary<T> bnd, int64_t B,
                 const T* __restrict__ q, const T* __restrict__ tau_in, const T* __restrict__ fhat_ws,
                 const T* __restrict__ pi_ws, T* __restrict__ qdd_out) {
  using namespace mop;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T* buf0 = reinterpret_cast<T*>(smem_raw) + (size_t)warp * 2 * NF * 32;
  T* buf1 = buf0 + NF * 32;
  const bool act = lane < n;
  LinkConst<T> C;
  if (act) C = Lg[lane];
  const unsigned FULL = 0xffffffffu;
  for (int64_t b = (int64_t)blockIdx.x * kMergedWarps + warp; b < B; b += (int64_t)gridDim.x * kMergedWarps) {
    // lane = link j: (R, p), Pi, Omega, Y (lines 3-4), Fhat_j, tau_j
    T Y[36], Pi[6], D;
    Rot<T> R;
    T p0, p1, p2;
    scan_link_setup(act, C, n, B, b, lane, q, pi_ws, Y, Pi, D, R, p0, p1, p2);
    T Fh[6], tj = 0;
    const T al = act ? C.alpha : T(0), be = act ? C.beta : T(0);
#pragma unroll
    for (int k = 0; k < 6; ++k) Fh[k] = act ? __ldg(fhat_ws + ((int64_t)lane * 6 + k) * B + b) : T(0);
    if (act) tj = __ldg(tau_in + (int64_t)lane * B + b);
    // operator A_i on lane l = n - i: link li = n-1-l (F, t rows), li-1 (Fhat), ln = n-l (z, c rows)
    const int li = n - 1 - lane, ln = n - lane, lf = n - 2 - lane;
    const bool vli = li >= 0, vln = ln >= 0 && ln < n, vlf = lf >= 0;
    const int sli = vli ? li : 0, sln = vln ? ln : 0, slf = vlf ? lf : 0;
    __syncwarp();
    auto W0 = [&](int f, T v) { buf0[f * 32 + lane] = v; };
    {
      // FF = X_li^T = [[R, 0], [[p]R, R]] (identity on lane n, f_{-1,0} := I)
      const T r[9] = {__shfl_sync(FULL, R.r00, sli), __shfl_sync(FULL, R.r01, sli), __shfl_sync(FULL, R.r02, sli),
                      __shfl_sync(FULL, R.r10, sli), __shfl_sync(FULL, R.r11, sli), __shfl_sync(FULL, R.r12, sli),
                      __shfl_sync(FULL, R.r20, sli), __shfl_sync(FULL, R.r21, sli), __shfl_sync(FULL, R.r22, sli)};
      const T q0 = __shfl_sync(FULL, p0, sli), q1 = __shfl_sync(FULL, p1, sli), q2 = __shfl_sync(FULL, p2, sli);
      T X[36];
#pragma unroll
      for (int i = 0; i < 36; ++i) X[i] = 0;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          X[6 * i + j] = r[3 * i + j];
          X[6 * (3 + i) + 3 + j] = r[3 * i + j];
        }
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const T x0 = r[j], x1 = r[3 + j], x2 = r[6 + j];
        X[6 * 3 + j] = q1 * x2 - q2 * x1;
        X[6 * 4 + j] = q2 * x0 - q0 * x2;
        X[6 * 5 + j] = q0 * x1 - q1 * x0;
      }
#pragma unroll
      for (int i = 0; i < 36; ++i) W0(FF + i, vli ? X[i] : T(i % 7 == 0));
      const T a_li = __shfl_sync(FULL, al, sli), b_li = __shfl_sync(FULL, be, sli);
      const T t_li = __shfl_sync(FULL, tj, sli);
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const T fo = __shfl_sync(FULL, Fh[k], slf);
        W0(Fo + k, vlf ? fo : T(0));
        W0(tF + k, T(0));
        W0(cF + k, T(0));
        W0(zo + k, T(0));
      }
      W0(tF + 2, vli ? -b_li : T(0));
      W0(tF + 5, vli ? -a_li : T(0));
      W0(to, vli ? t_li : T(0));
      W0(co, T(0));
#pragma unroll
      for (int i = 0; i < 36; ++i) {
        const T y = __shfl_sync(FULL, Y[i], sln);
        W0(zz + i, vln ? y : T(0));
        W0(zF + i, T(0));
      }
      const T d_ln = __shfl_sync(FULL, D, sln), a_ln = __shfl_sync(FULL, al, sln), b_ln = __shfl_sync(FULL, be, sln);
      const T inv = vln ? T(1) / d_ln : T(0);
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const T pk = __shfl_sync(FULL, Pi[k], sln);
        W0(zt + k, vln ? pk : T(0));
        W0(cz + k, T(0));
      }
      W0(ct, inv);
      W0(cz + 2, -b_ln * inv);
      W0(cz + 5, -a_ln * inv);
    }
    // inclusive Kogge-Stone scan over lanes 0..n, own operator on the left
    T* cur = buf0;
    T* nxt = buf1;
    for (int d = 1; d <= n; d <<= 1) {
      __syncwarp();
      if (lane >= d) {
        mop_compose(cur, lane, lane - d, nxt);
      } else {
        for (int f = 0; f < NF; ++f) nxt[f * 32 + lane] = cur[f * 32 + lane];
      }
      T* t = cur; cur = nxt; nxt = t;
    }
    __syncwarp();
    // x_i = C_l(seed), seed = (F_n, 0, 0, 0, 1): chat_{i+1} = cF . F_n + co
    T cval = cur[co * 32 + lane];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const T Fn = __shfl_sync(FULL, Fh[k], n - 1) + bnd.Ftip[k];
      cval = fma(cur[(cF + k) * 32 + lane], Fn, cval);
    }
    // chat_j (link j) sits on lane n - j
    const T ch = __shfl_sync(FULL, cval, act ? n - lane : 0);
    // line 7: prefix scan of lam -> Y^T lam + S chat (own operand on the left); line 8.
    // Y, Pi are rebuilt here (L2 reloads) rather than kept live across the scan.
    scan_link_setup(act, C, n, B, b, lane, q, pi_ws, Y, Pi, D, R, p0, p1, p2);
    T Lm[36], lb[6];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = 0; j < 6; ++j) Lm[6 * i + j] = Y[6 * j + i];
#pragma unroll
    for (int k = 0; k < 6; ++k) lb[k] = 0;
    lb[2] = be * ch;
    lb[5] = al * ch;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) compose_shfl<T, false>(Lm, lb, d, lane >= d);
    T acc = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const T lp = __shfl_up_sync(FULL, lb[k], 1);
      acc = fma(Pi[k], lane > 0 ? lp : T(0), acc);
    }
    if (act) qdd_out[(int64_t)lane * B + b] = ch - acc;
  }
}

// ---------------------------------------------------------------- CTA-wide variant (32 < n <= 256)
// Alg. 3 lines 2, 5-8 for long chains (the paper's fd_200 experiment):
// one CTA per state, thread = link, the same affine-map scans as fd_scan_kernel
// done CTA-wide: Kogge-Stone inside each warp (shuffles), the warp totals scanned
// by warp 0 (shuffles again), then every lane composes with the combined total
// of the warps after it (suffix scan, Eq. 18) or before it (prefix scan, Eq. 19).
// Composition is not commutative: the own operator always stays on the left.
constexpr int kFdBlockMaxN = 256;

// (L, b) := (L, b) o (L2, b2) with (L2, b2) in shared memory
template <typename T>
__device__ __forceinline__ void compose_mem(T (&Lm)[36], T (&bv)[6], const T* __restrict__ L2,
                                            const T* __restrict__ b2) {
  T nL[36], nb[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    nb[i] = bv[i];
#pragma unroll
    for (int j = 0; j < 6; ++j) nL[6 * i + j] = 0;
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const T bk = b2[k];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const T lik = Lm[6 * i + k];
#pragma unroll
      for (int j = 0; j < 6; ++j) nL[6 * i + j] = fma(lik, L2[6 * k + j], nL[6 * i + j]);
      nb[i] = fma(lik, bk, nb[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < 36; ++i) Lm[i] = nL[i];
#pragma unroll
  for (int i = 0; i < 6; ++i) bv[i] = nb[i];
}

// CTA-wide inclusive scan of affine maps; SUFFIX: M_l = A_l o A_{l+1} o ... ,
// else prefix M_l = A_l o A_{l-1} o ...  (sh: >= 2 * nwarps * 42 scalars)
template <typename T, bool SUFFIX>
__device__ __forceinline__ void block_affine_scan(T (&Lm)[36], T (&bv)[6], T* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll 1
  for (int d = 1; d < 32; d <<= 1)
    compose_shfl<T, SUFFIX>(Lm, bv, d, SUFFIX ? (lane + d < 32) : (lane >= d));
  // warp totals: the composite of the whole warp sits on lane 0 (suffix) / lane 31 (prefix)
  T* tot = sh;                     // [nw][42]
  if (lane == (SUFFIX ? 0 : 31)) {
    for (int i = 0; i < 36; ++i) tot[warp * 42 + i] = Lm[i];
    for (int i = 0; i < 6; ++i) tot[warp * 42 + 36 + i] = bv[i];
  }
  __syncthreads();
  if (warp == 0) {
    T TL[36], Tb[6];
    if (lane < nw) {
      for (int i = 0; i < 36; ++i) TL[i] = tot[lane * 42 + i];
      for (int i = 0; i < 6; ++i) Tb[i] = tot[lane * 42 + 36 + i];
    } else {
      for (int i = 0; i < 36; ++i) TL[i] = (i % 7 == 0) ? T(1) : T(0);
      for (int i = 0; i < 6; ++i) Tb[i] = 0;
    }
#pragma unroll 1
    for (int d = 1; d < 32; d <<= 1)
      compose_shfl<T, SUFFIX>(TL, Tb, d, SUFFIX ? (lane + d < 32) : (lane >= d));
    T* acc = sh + nw * 42;         // [nw][42]: combined totals
    if (lane < nw) {
      for (int i = 0; i < 36; ++i) acc[lane * 42 + i] = TL[i];
      for (int i = 0; i < 6; ++i) acc[lane * 42 + 36 + i] = Tb[i];
    }
  }
  __syncthreads();
  const int src = SUFFIX ? warp + 1 : warp - 1;
  if (src >= 0 && src < nw) {
    const T* acc = sh + nw * 42 + src * 42;
    compose_mem(Lm, bv, acc, acc + 36);
  }
  __syncthreads();                 // sh is reused by the caller
}

template <typename T>
__global__ void __launch_bounds__(kFdBlockMaxN)
fd_scan_block_kernel(int n, const LinkConst<T>* __restrict__ Lg, int64_t B, const T* __restrict__ q,
                     const T* __restrict__ tau_in, const T* __restrict__ tau_bias, const T* __restrict__ pi_ws,
                     T* __restrict__ qdd_out) {
  __shared__ T sh[2 * (kFdBlockMaxN / 32) * 42];
  __shared__ T edge[(kFdBlockMaxN / 32) * 6];
  const int l = threadIdx.x, lane = l & 31, warp = l >> 5, nw = blockDim.x >> 5;
  const bool act = l < n;
  LinkConst<T> C;
  if (act) C = Lg[l];
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    T Y[36], zb[6], Pi[6], D = 1, th = 0, al = 0, be = 0;
    Rot<T> R;
    T p0, p1, p2;
    scan_link_setup(act, C, n, B, b, l, q, pi_ws, Y, Pi, D, R, p0, p1, p2);
    if (act) {
      th = __ldg(tau_in + (int64_t)l * B + b) - __ldg(tau_bias + (int64_t)l * B + b);   // line 2
      al = C.alpha;
      be = C.beta;
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) zb[i] = Pi[i] * th;
    // line 5: suffix scan of z -> Y z + Pi tau_hat
    T Lm[36];
#pragma unroll
    for (int i = 0; i < 36; ++i) Lm[i] = Y[i];
    block_affine_scan<T, true>(Lm, zb, sh);
    // zhat_l = offset of the composite starting at l + 1 (lane 31: the next warp's lane 0)
    if (lane == 0)
      for (int k = 0; k < 6; ++k) edge[warp * 6 + k] = zb[k];
    __syncthreads();
    T z[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const T o = __shfl_down_sync(0xffffffffu, zb[k], 1);
      const T e = (lane == 31 && warp + 1 < nw) ? edge[(warp + 1) * 6 + k] : o;
      z[k] = (l + 1 < n) ? e : T(0);
    }
    __syncthreads();
    // line 6
    const T ch = (th - fma(be, z[2], al * z[5])) / D;
    // line 7: prefix scan of lam -> Y^T lam + S chat
    T lb[6];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = 0; j < 6; ++j) Lm[6 * i + j] = Y[6 * j + i];
#pragma unroll
    for (int k = 0; k < 6; ++k) lb[k] = 0;
    lb[2] = be * ch;
    lb[5] = al * ch;
    block_affine_scan<T, false>(Lm, lb, sh);
    // line 8: qdd_l = chat_l - Pi_l^T lam_{l-1} (lane 0: the previous warp's lane 31)
    if (lane == 31)
      for (int k = 0; k < 6; ++k) edge[warp * 6 + k] = lb[k];
    __syncthreads();
    T acc = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const T o = __shfl_up_sync(0xffffffffu, lb[k], 1);
      const T e = (lane == 0 && warp > 0) ? edge[(warp - 1) * 6 + k] : o;
      acc = fma(Pi[k], l > 0 ? e : T(0), acc);
    }
    __syncthreads();
    if (act) qdd_out[(int64_t)l * B + b] = ch - acc;
  }
}

template <typename T>
cudaError_t launch_fd_scan(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                           const T* qd, const T* tau, T* qdd, T* ws, cudaStream_t st, int* launches,
                           bool* supported, int32_t* status) {
  *supported = n >= 1 && n <= kFdBlockMaxN;
  if (!*supported) return cudaSuccess;
  T* tau_bias = ws;                                  // [n][B]
  T* pi_ws = ws + (size_t)n * B;                     // [n][7][B]
  bool ok = false;
  const bool block = n > 32;                         // CTA-wide scans for long chains
  cudaError_t e = block
      ? launch_rnea_block<T>(n, L_dev, bnd, B, q, qd, nullptr, tau_bias, st, launches, &ok)     // line 1
      : launch_rnea_warp<T>(n, L_dev, bnd, B, q, qd, nullptr, tau_bias, st, launches, &ok);
  if (e != cudaSuccess) return e;
  int64_t g1 = (B + kAbiThreads - 1) / kAbiThreads;
  if (g1 > (int64_t)num_sms() * 8) g1 = (int64_t)num_sms() * 8;
  abi_kernel<T><<<(unsigned)g1, kAbiThreads, 0, st>>>(n, L_dev, B, q, pi_ws, status);                          // lines 3-4
  ++*launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (block) {
    int64_t g2 = B < (int64_t)num_sms() * 8 ? B : (int64_t)num_sms() * 8;
    fd_scan_block_kernel<T><<<(unsigned)g2, ((n + 31) / 32) * 32, 0, st>>>(n, L_dev, B, q, tau, tau_bias, pi_ws,
                                                                            qdd);
  } else {
    int64_t g2 = (B + kScanWarps - 1) / kScanWarps;
    if (g2 > (int64_t)num_sms() * 16) g2 = (int64_t)num_sms() * 16;
    fd_scan_kernel<T><<<(unsigned)g2, kScanWarps * 32, 0, st>>>(n, L_dev, B, q, tau, tau_bias, pi_ws, qdd);  // 2, 5-8
  }
  ++*launches;
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_fd_merged(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                             const T* qd, const T* tau, T* qdd, T* ws, cudaStream_t st, int* launches,
                             bool* supported, int32_t* status) {
  *supported = n >= 1 && n <= 31;                   // n + 1 operators on the lanes of one warp
  if (!*supported) return cudaSuccess;
  T* fhat_ws = ws;                                   // [n][6][B]
  T* pi_ws = ws + (size_t)n * 6 * B;                 // [n][7][B]
  bool ok = false;
  cudaError_t e = launch_rnea_warp<T>(n, L_dev, bnd, B, q, qd, nullptr, nullptr, st, launches, &ok, fhat_ws);
  if (e != cudaSuccess) return e;
  int64_t g1 = (B + kAbiThreads - 1) / kAbiThreads;
  if (g1 > (int64_t)num_sms() * 8) g1 = (int64_t)num_sms() * 8;
  abi_kernel<T><<<(unsigned)g1, kAbiThreads, 0, st>>>(n, L_dev, B, q, pi_ws, status);
  ++*launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t smem = (size_t)kMergedWarps * 2 * mop::NF * 32 * sizeof(T);
  static thread_local int attr_dev[2] = {-1, -1};
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev[sizeof(T) == 8] != dev) {
    e = cudaFuncSetAttribute(fd_merged_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_dev[sizeof(T) == 8] = dev;
  }
  int64_t g2 = (B + kMergedWarps - 1) / kMergedWarps;
  if (g2 > (int64_t)num_sms() * 8) g2 = (int64_t)num_sms() * 8;
  fd_merged_kernel<T><<<(unsigned)g2, kMergedWarps * 32, smem, st>>>(n, L_dev, bnd, B, q, tau, fhat_ws, pi_ws, qdd);
  ++*launches;
  return cudaGetLastError();
}

size_t fd_scan_ws_elems(int n, int64_t B) { return (size_t)n * B * (6 + kPiPerLink); }

template cudaError_t launch_fd_scan<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                            const double*, const double*, const double*, double*, double*,
                                            cudaStream_t, int*, bool*, int32_t*);
template cudaError_t launch_fd_merged<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                              const double*, const double*, const double*, double*, double*,
                                              cudaStream_t, int*, bool*, int32_t*);
template cudaError_t launch_fd_merged<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                             const float*, const float*, const float*, float*, float*,
                                             cudaStream_t, int*, bool*, int32_t*);
template cudaError_t launch_fd_scan<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                           const float*, const float*, const float*, float*, float*, cudaStream_t,
                                           int*, bool*, int32_t*);

}  // namespace rd
