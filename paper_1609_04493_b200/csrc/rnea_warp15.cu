// rnea_warp15.cu -- the paper's SYNCHRONOUS forward scan, Eq. (15),
// taken literally (strategy WARP_SCAN_EQ15, n <= 32, any joints; SURVEY §8(f)
// NEXT-2): one warp per state, lane = link.
//   forward:  ONE Kogge-Stone scan of the 28x28 operators A_l acting on
//             x = (Vdot, Q, V, Fhat, 1), Q = (w x v, w1^2, w1w2, w1w3, w2^2, w2w3, w3^2)
//             (P:218), prefixes P_l = A_l P_{l-1} (A4 order), applied to the seed
//             x_0 = (Vdot_0, Q(V_0), V_0, 0, 1): the bias wrench Fhat_l comes out of
//             the scan itself ("synchronously computed") instead of a
//             separate per-lane step;
//   backward: the Eq. (16) affine suffix scan and tau_l = S_l^T F_l
//             (eq16_backward_torque, shared with rnea_warp13).
// The starred blocks of A_l (unspecified in the paper, reading A6) are the
// closed forms derived in DESIGN.md (reading A6):
//   V' = X V + s,   Vdot' = X Vdot - ad_s X V + a,       X = Ad_{f^-1}, s = S qd, a = S qdd
//   Q' = QQ Q + QV V + Qo   (w' x v' and w'w'^T in terms of w x v, ww^T, V),
//   Fhat' = J Vdot' + H Q',  H Q = (m w x v + w x (w x h), h x (w x v) + w x (I_o w)).
// Operator storage: the Vdot<-Vdot and V<-V blocks are both X for every
// composite, so one 6x6 is kept; the rest is dense: 360 scalars per lane in
// shared memory [field][lane], double-buffered (Kogge-Stone reads the partner's
// old operator): 184 KB per warp in fp64, so ONE warp per CTA.  This kernel
// exists to measure the paper's operator; the base-frame WARP_SCAN is the
// production scan.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"
#include "rd_scan.cuh"

namespace rd {

namespace e15 {   // field offsets of one operator (row-major blocks)
constexpr int X = 0, VdV = 36, Vdo = 72, QQ = 78, QV = 159, Qo = 213, Vo = 222, FVd = 228, FQ = 264, FV = 318,
              Fo = 354, NF = 360;
constexpr int kJH = 90;   // per-lane constants J (36) and H (54)
__device__ __forceinline__ int widx(int j, int k) {   // (11, 12, 13, 22, 23, 33)
  const int a = j < k ? j : k, b = j < k ? k : j;
  return a == 0 ? b : (a == 1 ? 2 + b : 5);
}
}  // namespace e15

template <typename T>
__device__ __forceinline__ int e15_warps() { return sizeof(T) == 8 ? 1 : 2; }

// C[R x Cc] (+)= B[R x K] A[K x Cc]; B on lane `own` of buf, A on lane `src` of buf, C on lane `own` of out.
template <int R, int K, int Cc, bool ACC, typename T>
__device__ __forceinline__ void e15_mm(const T* __restrict__ buf, int offB, int offA, T* __restrict__ out, int offC,
                                       int own, int src) {
#pragma unroll 1
  for (int i = 0; i < R; ++i) {
    T b[K];
#pragma unroll
    for (int m = 0; m < K; ++m) b[m] = buf[(offB + i * K + m) * 32 + own];
#pragma unroll
    for (int j = 0; j < Cc; ++j) {
      T s = ACC ? out[(offC + i * Cc + j) * 32 + own] : T(0);
#pragma unroll
      for (int m = 0; m < K; ++m) s = fma(b[m], buf[(offA + m * Cc + j) * 32 + src], s);
      out[(offC + i * Cc + j) * 32 + own] = s;
    }
  }
}
template <typename T>
__device__ __forceinline__ void e15_addown(const T* __restrict__ buf, int off, T* __restrict__ out, int len, int own) {
  for (int i = 0; i < len; ++i) out[(off + i) * 32 + own] += buf[(off + i) * 32 + own];
}

// out = B o A (A = the earlier prefix on lane src, B = own operator on lane own)
template <typename T>
__device__ __noinline__ void e15_compose(const T* __restrict__ cur, T* __restrict__ nxt, int own, int src) {
  using namespace e15;
  e15_mm<6, 6, 6, false>(cur, X, X, nxt, X, own, src);
  e15_mm<6, 6, 6, false>(cur, X, VdV, nxt, VdV, own, src);
  e15_mm<6, 6, 6, true>(cur, VdV, X, nxt, VdV, own, src);
  e15_mm<6, 6, 1, false>(cur, X, Vdo, nxt, Vdo, own, src);
  e15_mm<6, 6, 1, true>(cur, VdV, Vo, nxt, Vdo, own, src);
  e15_addown(cur, Vdo, nxt, 6, own);
  e15_mm<9, 9, 9, false>(cur, QQ, QQ, nxt, QQ, own, src);
  e15_mm<9, 9, 6, false>(cur, QQ, QV, nxt, QV, own, src);
  e15_mm<9, 6, 6, true>(cur, QV, X, nxt, QV, own, src);
  e15_mm<9, 9, 1, false>(cur, QQ, Qo, nxt, Qo, own, src);
  e15_mm<9, 6, 1, true>(cur, QV, Vo, nxt, Qo, own, src);
  e15_addown(cur, Qo, nxt, 9, own);
  e15_mm<6, 6, 1, false>(cur, X, Vo, nxt, Vo, own, src);
  e15_addown(cur, Vo, nxt, 6, own);
  e15_mm<6, 6, 6, false>(cur, FVd, X, nxt, FVd, own, src);
  e15_mm<6, 9, 9, false>(cur, FQ, QQ, nxt, FQ, own, src);
  e15_mm<6, 6, 6, false>(cur, FVd, VdV, nxt, FV, own, src);
  e15_mm<6, 9, 6, true>(cur, FQ, QV, nxt, FV, own, src);
  e15_mm<6, 6, 6, true>(cur, FV, X, nxt, FV, own, src);
  e15_mm<6, 6, 1, false>(cur, FVd, Vdo, nxt, Fo, own, src);
  e15_mm<6, 9, 1, true>(cur, FQ, Qo, nxt, Fo, own, src);
  e15_mm<6, 6, 1, true>(cur, FV, Vo, nxt, Fo, own, src);
  e15_addown(cur, Fo, nxt, 6, own);
}

template <typename T>
__global__ void __launch_bounds__(64)
rnea_warp15_kernel(int n, const LinkConst<T>* __restrict__ Lg, const Boundary<T> bnd, int64_t B,
                   const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ qdd,
                   T* __restrict__ tau) {
  using namespace e15;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = e15_warps<T>();
  T* buf0 = reinterpret_cast<T*>(smem_raw) + (size_t)warp * (2 * NF + kJH) * 32;
  T* buf1 = buf0 + NF * 32;
  T* jh = buf1 + NF * 32;                                          // J (36) and H (54) of this lane's link
  const bool act = lane < n;
  LinkConst<T> C;
  if (act) {
    C = Lg[lane];
  } else {
#pragma unroll
    for (int k = 0; k < 9; ++k) C.Rm[k] = (k % 4 == 0) ? T(1) : T(0);
#pragma unroll
    for (int k = 0; k < 3; ++k) { C.pm[k] = 0; C.h[k] = 0; }
#pragma unroll
    for (int k = 0; k < 6; ++k) C.I[k] = 0;
    C.m = 0; C.alpha = 0; C.beta = 0;
  }
  // J = [[m I, -[h]], [[h], I_o]] and H (6x9) of this lane's link (state independent), to shared memory
  auto Jv = [&](int i) -> T& { return jh[i * 32 + lane]; };
  auto Hv = [&](int i) -> T& { return jh[(36 + i) * 32 + lane]; };
  {
    const T h0 = C.h[0], h1 = C.h[1], h2 = C.h[2];
    const T Io[9] = {C.I[0], C.I[3], C.I[4], C.I[3], C.I[1], C.I[5], C.I[4], C.I[5], C.I[2]};
    const T Sh[9] = {0, -h2, h1, h2, 0, -h0, -h1, h0, 0};
    for (int i = 0; i < 36; ++i) Jv(i) = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      Jv(6 * i + i) = C.m;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        Jv(6 * i + 3 + j) = -Sh[3 * i + j];
        Jv(6 * (3 + i) + j) = Sh[3 * i + j];
        Jv(6 * (3 + i) + 3 + j) = Io[3 * i + j];
      }
    }
    for (int i = 0; i < 54; ++i) Hv(i) = 0;
    const T hv[3] = {h0, h1, h2};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      Hv(9 * k + k) = C.m;                                         // m (w x v)
#pragma unroll
      for (int j = 0; j < 3; ++j) {                                // w x (w x h) = w (w.h) - h |w|^2
        Hv(9 * k + 3 + widx(k, j)) += hv[j];
        Hv(9 * k + 3 + widx(j, j)) -= hv[k];
        Hv(9 * (3 + k) + j) = Sh[3 * k + j];                       // h x (w x v)
      }
    }
    // w x (I_o w): component k = sum eps_{kab} w_a (I_o w)_b
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int a1 = (k + 1) % 3, b1 = (k + 2) % 3;                // eps_{k a1 b1} = +1, eps_{k b1 a1} = -1
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        Hv(9 * (3 + k) + 3 + widx(a1, c)) += Io[3 * b1 + c];
        Hv(9 * (3 + k) + 3 + widx(b1, c)) -= Io[3 * a1 + c];
      }
    }
  }
  for (int64_t b = (int64_t)blockIdx.x * nw + warp; b < B; b += (int64_t)gridDim.x * nw) {
    T qi = 0, qdi = 0, qddi = 0;
    if (act) {
      qi = __ldg(q + (int64_t)lane * B + b);
      qdi = __ldg(qd + (int64_t)lane * B + b);
      qddi = __ldg(qdd + (int64_t)lane * B + b);
    }
    T sn, cs;
    rd_sincos(C.alpha * qi, &sn, &cs);
    const Rot<T> R = make_rot(C, sn, cs);
    const T d = C.beta * qi;
    const T p0 = fma(d, C.Rm[2], C.pm[0]), p1 = fma(d, C.Rm[5], C.pm[1]), p2 = fma(d, C.Rm[8], C.pm[2]);
    // ---- elementary operator A_l into buf0
    __syncwarp();
    auto W = [&](int f, T v) { buf0[f * 32 + lane] = v; };
    const T Rt[9] = {R.r00, R.r10, R.r20, R.r01, R.r11, R.r21, R.r02, R.r12, R.r22};   // R^T row-major
    const T pv[3] = {p0, p1, p2};
    const T sv2 = C.beta * qdi, sw2 = C.alpha * qdi;              // s = (0, 0, sv2, 0, 0, sw2)
    {
      // X = Ad_{f^-1} = [[R^T, -R^T [p]], [0, R^T]];  -R^T[p] column j = -R^T (e_j x ... ) = R^T (p x e_j)... :
      // (-R^T [p])_{ij} = -sum_k Rt_ik [p]_kj
      const T Pm[9] = {0, -p2, p1, p2, 0, -p0, -p1, p0, 0};
      T Xm[36];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          Xm[6 * i + j] = Rt[3 * i + j];
          Xm[6 * (3 + i) + 3 + j] = Rt[3 * i + j];
          Xm[6 * (3 + i) + j] = 0;
          Xm[6 * i + 3 + j] = -(Rt[3 * i] * Pm[j] + Rt[3 * i + 1] * Pm[3 + j] + Rt[3 * i + 2] * Pm[6 + j]);
        }
#pragma unroll
      for (int i = 0; i < 36; ++i) W(X + i, Xm[i]);
      // VdV = -ad_s X, ad_s = [[S_w, S_v], [0, S_w]], S_w = [sw2 e_z], S_v = [sv2 e_z]:
      // ([c e_z] y) = c (-y1, y0, 0)
      T VdVm[36];
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const T x0 = Xm[j], x1 = Xm[6 + j], x3 = Xm[18 + j], x4 = Xm[24 + j];
        VdVm[j] = -(-sw2 * x1 - sv2 * x4);
        VdVm[6 + j] = -(sw2 * x0 + sv2 * x3);
        VdVm[12 + j] = 0;
        VdVm[18 + j] = -(-sw2 * x4);
        VdVm[24 + j] = -(sw2 * x3);
        VdVm[30 + j] = 0;
      }
#pragma unroll
      for (int i = 0; i < 36; ++i) W(VdV + i, VdVm[i]);
      const T av[6] = {0, 0, C.beta * qddi, 0, 0, C.alpha * qddi};
      const T sv[6] = {0, 0, sv2, 0, 0, sw2};
#pragma unroll
      for (int k = 0; k < 6; ++k) { W(Vdo + k, av[k]); W(Vo + k, sv[k]); }
      // QQ = [[R^T, R^T G(p)], [0, Cq]],  G(p) ww = w x (w x p)
      T QQm[81];
#pragma unroll
      for (int i = 0; i < 81; ++i) QQm[i] = 0;
      T Gp[18];
#pragma unroll
      for (int i = 0; i < 18; ++i) Gp[i] = 0;
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          Gp[6 * k + widx(k, j)] += pv[j];
          Gp[6 * k + widx(j, j)] -= pv[k];
        }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
#pragma unroll
        for (int c = 0; c < 3; ++c) QQm[9 * r + c] = Rt[3 * r + c];
#pragma unroll
        for (int e = 0; e < 6; ++e)
          QQm[9 * r + 3 + e] = Rt[3 * r] * Gp[e] + Rt[3 * r + 1] * Gp[6 + e] + Rt[3 * r + 2] * Gp[12 + e];
      }
#pragma unroll
      for (int a_ = 0; a_ < 3; ++a_)
#pragma unroll
        for (int b_ = a_; b_ < 3; ++b_)
#pragma unroll
          for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k) QQm[9 * (3 + widx(a_, b_)) + 3 + widx(j, k)] += Rt[3 * a_ + j] * Rt[3 * b_ + k];
      // QV, Qo: s_v = sv2 e_z, s_w = sw2 e_z
      T QVm[54], Qom[9];
#pragma unroll
      for (int i = 0; i < 54; ++i) QVm[i] = 0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        // [s_w] R^T v : rows (-sw2 Rt[1][c], sw2 Rt[0][c], 0)
        QVm[6 * 0 + c] = -sw2 * Rt[3 + c];
        QVm[6 * 1 + c] = sw2 * Rt[c];
        // w coefficient: -[s_v] R^T - [s_w] R^T [p]
        const T RtP0 = -(Rt[0] * Pm[c] + Rt[1] * Pm[3 + c] + Rt[2] * Pm[6 + c]);   // (-R^T[p])_{0c}
        const T RtP1 = -(Rt[3] * Pm[c] + Rt[4] * Pm[3 + c] + Rt[5] * Pm[6 + c]);   // (-R^T[p])_{1c}
        QVm[6 * 0 + 3 + c] = sv2 * Rt[3 + c] + (-sw2) * RtP1;
        QVm[6 * 1 + 3 + c] = -sv2 * Rt[c] + sw2 * RtP0;
      }
      const T swv[3] = {0, 0, sw2};
#pragma unroll
      for (int a_ = 0; a_ < 3; ++a_)
#pragma unroll
        for (int b_ = a_; b_ < 3; ++b_) {
          const int row = 3 + widx(a_, b_);
#pragma unroll
          for (int j = 0; j < 3; ++j) QVm[6 * row + 3 + j] = Rt[3 * a_ + j] * swv[b_] + swv[a_] * Rt[3 * b_ + j];
          Qom[row] = swv[a_] * swv[b_];
        }
      Qom[0] = 0; Qom[1] = 0; Qom[2] = 0;                          // s_w x s_v = 0 (both along e_z)
#pragma unroll
      for (int i = 0; i < 81; ++i) W(QQ + i, QQm[i]);
#pragma unroll
      for (int i = 0; i < 54; ++i) W(QV + i, QVm[i]);
#pragma unroll
      for (int i = 0; i < 9; ++i) W(Qo + i, Qom[i]);
      // F rows: FVd = J X; FQ = H QQ; FV = J VdV + H QV; Fo = J a + H Qo (operands re-read from smem)
      __syncwarp();
      auto Rd = [&](int f) { return buf0[f * 32 + lane]; };
#pragma unroll 1
      for (int r = 0; r < 6; ++r) {
#pragma unroll 1
        for (int c = 0; c < 6; ++c) {
          T x = 0, y = 0;
#pragma unroll
          for (int k = 0; k < 6; ++k) { x = fma(Jv(6 * r + k), Rd(X + 6 * k + c), x); y = fma(Jv(6 * r + k), Rd(VdV + 6 * k + c), y); }
#pragma unroll
          for (int k = 0; k < 9; ++k) y = fma(Hv(9 * r + k), Rd(QV + 6 * k + c), y);
          W(FVd + 6 * r + c, x);
          W(FV + 6 * r + c, y);
        }
#pragma unroll 1
        for (int c = 0; c < 9; ++c) {
          T x = 0;
#pragma unroll
          for (int k = 0; k < 9; ++k) x = fma(Hv(9 * r + k), Rd(QQ + 9 * k + c), x);
          W(FQ + 9 * r + c, x);
        }
        T o = 0;
#pragma unroll
        for (int k = 0; k < 6; ++k) o = fma(Jv(6 * r + k), Rd(Vdo + k), o);
#pragma unroll
        for (int k = 0; k < 9; ++k) o = fma(Hv(9 * r + k), Rd(Qo + k), o);
        W(Fo + r, o);
      }
    }
    // ---- inclusive Kogge-Stone scan, own operator on the left
    T* cur = buf0;
    T* nxt = buf1;
    for (int dd = 1; dd < n; dd <<= 1) {
      __syncwarp();
      if (lane >= dd) e15_compose(cur, nxt, lane, lane - dd);
      else
        for (int f = 0; f < NF; ++f) nxt[f * 32 + lane] = cur[f * 32 + lane];
      T* t = cur; cur = nxt; nxt = t;
    }
    __syncwarp();
    // ---- Fhat_l = F rows of P_l applied to x_0 = (Vdot_0, Q(V_0), V_0, 0, 1)
    T x0q[9];
    {
      const T v0 = bnd.V0[0], v1 = bnd.V0[1], v2 = bnd.V0[2], w0 = bnd.V0[3], w1 = bnd.V0[4], w2 = bnd.V0[5];
      x0q[0] = w1 * v2 - w2 * v1; x0q[1] = w2 * v0 - w0 * v2; x0q[2] = w0 * v1 - w1 * v0;
      x0q[3] = w0 * w0; x0q[4] = w0 * w1; x0q[5] = w0 * w2; x0q[6] = w1 * w1; x0q[7] = w1 * w2; x0q[8] = w2 * w2;
    }
    T Fh[6];
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      T acc = cur[(Fo + r) * 32 + lane];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        acc = fma(cur[(FVd + 6 * r + k) * 32 + lane], bnd.Vd0[k], acc);
        acc = fma(cur[(FV + 6 * r + k) * 32 + lane], bnd.V0[k], acc);
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) acc = fma(cur[(FQ + 9 * r + k) * 32 + lane], x0q[k], acc);
      Fh[r] = acc;
    }
    const T t = eq16_backward_torque(lane, n, act, R, p0, p1, p2, Fh, bnd.Ftip, C.alpha, C.beta);
    if (act) tau[(int64_t)lane * B + b] = t;
  }
}

template <typename T>
cudaError_t launch_rnea_warp15(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                               const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                               bool* supported) {
  *supported = n >= 1 && n <= 32;
  if (!*supported) return cudaSuccess;
  const int nw = sizeof(T) == 8 ? 1 : 2;
  const size_t smem = (size_t)nw * (2 * e15::NF + e15::kJH) * 32 * sizeof(T);
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(rnea_warp15_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  int64_t grid = (B + nw - 1) / nw;
  if (grid > (int64_t)num_sms() * 4) grid = (int64_t)num_sms() * 4;
  rnea_warp15_kernel<T><<<(unsigned)grid, nw * 32, smem, st>>>(n, L_dev, bnd, B, q, qd, qdd, tau);
  ++*launches;
  return cudaGetLastError();
}

template cudaError_t launch_rnea_warp15<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                                const double*, const double*, const double*, double*, cudaStream_t,
                                                int*, bool*);
template cudaError_t launch_rnea_warp15<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                               const float*, const float*, const float*, float*, cudaStream_t, int*,
                                               bool*);

}  // namespace rd
