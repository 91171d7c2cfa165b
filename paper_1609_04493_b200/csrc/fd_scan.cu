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
abi_kernel(int n, const LinkConst<T>* __restrict__ L, int64_t B, const T* __restrict__ q, T* __restrict__ pi_ws) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
    Sym6<T> K, Kc;
#pragma unroll
    for (int k = 0; k < 6; ++k) { Kc.a[k] = 0; Kc.c[k] = 0; }
#pragma unroll
    for (int k = 0; k < 9; ++k) Kc.b[k] = 0;
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
    if (act) {
      Rot<T> R;
      T p0, p1, p2, s, c, d;
      link_transform(C, __ldg(q + (int64_t)lane * B + b), R, p0, p1, p2, s, c, d);
      const T* w = pi_ws + (int64_t)lane * kPiPerLink * B + b;
#pragma unroll
      for (int k = 0; k < 6; ++k) Pi[k] = __ldg(w + (int64_t)k * B);
      D = __ldg(w + (int64_t)6 * B);
      th = __ldg(tau_in + (int64_t)lane * B + b) - __ldg(tau_bias + (int64_t)lane * B + b);   // line 2
      al = C.alpha;
      be = C.beta;
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
        Y[6 * i + 2] = fma(-Pi[i], be, Y[6 * i + 2]);
        Y[6 * i + 5] = fma(-Pi[i], al, Y[6 * i + 5]);
        zb[i] = Pi[i] * th;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 36; ++i) Y[i] = (i % 7 == 0) ? T(1) : T(0);   // identity map
#pragma unroll
      for (int i = 0; i < 6; ++i) { zb[i] = 0; Pi[i] = 0; }
    }
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

template <typename T>
cudaError_t launch_fd_scan(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                           const T* qd, const T* tau, T* qdd, T* ws, cudaStream_t st, int* launches,
                           bool* supported) {
  *supported = n >= 1 && n <= 32;
  if (!*supported) return cudaSuccess;
  T* tau_bias = ws;                                  // [n][B]
  T* pi_ws = ws + (size_t)n * B;                     // [n][7][B]
  bool ok = false;
  cudaError_t e = launch_rnea_warp<T>(n, L_dev, bnd, B, q, qd, nullptr, tau_bias, st, launches, &ok);   // line 1
  if (e != cudaSuccess) return e;
  int64_t g1 = (B + kAbiThreads - 1) / kAbiThreads;
  if (g1 > (int64_t)num_sms() * 8) g1 = (int64_t)num_sms() * 8;
  abi_kernel<T><<<(unsigned)g1, kAbiThreads, 0, st>>>(n, L_dev, B, q, pi_ws);                          // lines 3-4
  ++*launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int64_t g2 = (B + kScanWarps - 1) / kScanWarps;
  if (g2 > (int64_t)num_sms() * 16) g2 = (int64_t)num_sms() * 16;
  fd_scan_kernel<T><<<(unsigned)g2, kScanWarps * 32, 0, st>>>(n, L_dev, B, q, tau, tau_bias, pi_ws, qdd);  // 2, 5-8
  ++*launches;
  return cudaGetLastError();
}

size_t fd_scan_ws_elems(int n, int64_t B) { return (size_t)n * B * (1 + kPiPerLink); }

template cudaError_t launch_fd_scan<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                            const double*, const double*, const double*, double*, double*,
                                            cudaStream_t, int*, bool*);
template cudaError_t launch_fd_scan<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                           const float*, const float*, const float*, float*, float*, cudaStream_t,
                                           int*, bool*);

}  // namespace rd
