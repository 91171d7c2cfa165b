// jsiia.cu -- forward dynamics by joint-space inertia inversion, Alg. 2
// (Eq. 5, 6, 17): one WARP per state, the n+1 data-independent
// inverse dynamics of Alg. 2 line 1 run one per LANE ("All n+1 inverse
// dynamics are data independent, and thus may be solved simultaneously"):
//   lane j < n : M_{.,j} = ID(q, 0, delta_{.,j}, 0, 0, 0)          (Eq. 17)
//   lane n     : tau_bias = ID(q, qd, 0, V_0, Vdot_0, F_{n+1})      (Eq. 5)
// then tau_diff = tau - tau_bias (line 2) and a warp-cooperative Cholesky
// factorisation and two triangular solves in shared memory instead of the
// explicit inverse of lines 3-4 (the paper points to parallel Cholesky).
//
// Each lane's RNEA keeps no per-link stash: the backward sweep re-derives V_i,
// Vdot_i by inverting the (rigid, well-conditioned) forward maps,
// V_{i-1} = Ad_{f_i}(V_i - S_i qd_i),
// Vdot_{i-1} = Ad_{f_i}(Vdot_i - S_i qdd_i - ad_{V_i}(S_i qd_i)),
// so the whole ID runs in registers; the link transforms (sin, cos, d) are
// computed once per state by lane i and shared through shared memory.
// n <= 31.  A non-SPD M (pivot <= 0) makes that state's qdd NaN (A11).
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"

namespace rd {

constexpr int kJsWarps = 4;

// out = Ad_f in = (R v + p x (R w), R w)
template <typename T>
__device__ __forceinline__ void ad_f(const Rot<T>& R, T p0, T p1, T p2, const T* in, T* out) {
  T w0, w1, w2;
  rot_n(R, in[3], in[4], in[5], w0, w1, w2);
  T v0, v1, v2;
  rot_n(R, in[0], in[1], in[2], v0, v1, v2);
  out[0] = fma(p1, w2, fma(-p2, w1, v0));
  out[1] = fma(p2, w0, fma(-p0, w2, v1));
  out[2] = fma(p0, w1, fma(-p1, w0, v2));
  out[3] = w0; out[4] = w1; out[5] = w2;
}

template <typename T>
__global__ void __launch_bounds__(kJsWarps * 32)
jsiia_kernel(int n, const LinkConst<T>* __restrict__ Lg, const Boundary<T> bnd, int64_t B,
             const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ tau_in,
             T* __restrict__ qdd_out, int32_t* __restrict__ status) {
  constexpr int NF = sizeof(LinkConst<T>) / sizeof(T);
  __shared__ T sc[NF][32];                  // link constants [field][link]
  __shared__ T strf[kJsWarps][3][32];       // per-state link transforms (sin, cos, d)
  __shared__ T sM[kJsWarps][32][33];        // M(q), then its Cholesky factor (lower)
  for (int idx = threadIdx.x; idx < NF * 32; idx += blockDim.x) {
    const int f = idx / 32, l = idx % 32;
    sc[f][l] = l < n ? reinterpret_cast<const T*>(Lg + l)[f] : T(0);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned full = 0xffffffffu;
  auto cst = [&](int i) {
    LinkConst<T> C;
#pragma unroll
    for (int f = 0; f < 9; ++f) C.Rm[f] = sc[f][i];
#pragma unroll
    for (int f = 0; f < 3; ++f) { C.pm[f] = sc[9 + f][i]; C.h[f] = sc[13 + f][i]; }
    C.m = sc[12][i];
#pragma unroll
    for (int f = 0; f < 6; ++f) C.I[f] = sc[16 + f][i];
    C.alpha = sc[22][i];
    C.beta = sc[23][i];
    return C;
  };
  T (*M)[33] = sM[warp];
  for (int64_t b = (int64_t)blockIdx.x * kJsWarps + warp; b < B; b += (int64_t)gridDim.x * kJsWarps) {
    // CalcTransform: lane l owns link l
    T qdl = 0, taul = 0;
    if (lane < n) {
      const T ql = __ldg(q + (int64_t)lane * B + b);
      qdl = __ldg(qd + (int64_t)lane * B + b);
      taul = __ldg(tau_in + (int64_t)lane * B + b);
      T s, c;
      rd_sincos(sc[22][lane] * ql, &s, &c);
      strf[warp][0][lane] = s;
      strf[warp][1][lane] = c;
      strf[warp][2][lane] = sc[23][lane] * ql;
    }
    __syncwarp();
    const bool bias = lane == n;
    // ---- forward sweep of this lane's ID
    T V[6], Vd[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) { V[k] = bias ? bnd.V0[k] : T(0); Vd[k] = bias ? bnd.Vd0[k] : T(0); }
    for (int i = 0; i < n; ++i) {
      const LinkConst<T> C = cst(i);
      const T s = strf[warp][0][i], c = strf[warp][1][i], d = strf[warp][2][i];
      const Rot<T> R = make_rot(C, s, c);
      const T p0 = fma(d, C.Rm[2], C.pm[0]), p1 = fma(d, C.Rm[5], C.pm[1]), p2 = fma(d, C.Rm[8], C.pm[2]);
      const T qds = __shfl_sync(full, qdl, i);        // every lane joins the shuffle
      const T qdi = bias ? qds : T(0);
      const T qddi = (lane == i) ? T(1) : T(0);
      T Vn[6], Vdn[6];
      fwd_step<T, false>(C, R, p0, p1, p2, qdi, qddi, V, Vd, Vn, Vdn);
#pragma unroll
      for (int k = 0; k < 6; ++k) { V[k] = Vn[k]; Vd[k] = Vdn[k]; }
    }
    // ---- backward sweep: F_i = Fhat_i + Ad^T F_{i+1}; tau_i = S_i^T F_i; then invert the forward map
    T F[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) F[k] = bias ? bnd.Ftip[k] : T(0);
    Rot<T> Rn{1, 0, 0, 0, 1, 0, 0, 0, 1};
    T pn0 = 0, pn1 = 0, pn2 = 0;
    for (int i = n - 1; i >= 0; --i) {
      const LinkConst<T> C = cst(i);
      T Fh[6], Fo[6];
      bias_force(C, V, Vd, Fh);
      bwd_step(Rn, pn0, pn1, pn2, F, Fh, Fo);
#pragma unroll
      for (int k = 0; k < 6; ++k) F[k] = Fo[k];
      const T ti = fma(C.beta, F[2], C.alpha * F[5]);
      if (lane < n) M[i][lane] = ti;            // column j = lane of M(q), Eq. (17)
      if (bias) M[i][31] = ti;                  // tau_bias (n <= 31 keeps column 31 free)
      // rebuild V_{i-1}, Vdot_{i-1}
      const T s = strf[warp][0][i], c = strf[warp][1][i], d = strf[warp][2][i];
      Rn = make_rot(C, s, c);
      pn0 = fma(d, C.Rm[2], C.pm[0]); pn1 = fma(d, C.Rm[5], C.pm[1]); pn2 = fma(d, C.Rm[8], C.pm[2]);
      const T qds = __shfl_sync(full, qdl, i);        // every lane joins the shuffle
      const T qdi = bias ? qds : T(0);
      const T qddi = (lane == i) ? T(1) : T(0);
      const T a = C.alpha, be = C.beta, aq = a * qdi, bq = be * qdi;
      T x[6], y[6];
      // Vdot_i - S qdd - ad_{V_i}(S qd); ad_V(S qd) = qd (beta w x e_z + alpha v x e_z, alpha w x e_z)
      y[0] = Vd[0] - fma(bq, V[4], aq * V[1]);
      y[1] = Vd[1] + fma(bq, V[3], aq * V[0]);
      y[2] = Vd[2] - be * qddi;
      y[3] = Vd[3] - aq * V[4];
      y[4] = Vd[4] + aq * V[3];
      y[5] = Vd[5] - a * qddi;
#pragma unroll
      for (int k = 0; k < 6; ++k) x[k] = V[k];
      x[2] -= bq;
      x[5] -= aq;
      ad_f(Rn, pn0, pn1, pn2, x, V);
      ad_f(Rn, pn0, pn1, pn2, y, Vd);
    }
    __syncwarp();
    // ---- tau_diff = tau - tau_bias; Cholesky M = L L^T; solve (Alg. 2 lines 2-4)
    T rhs = (lane < n) ? taul - M[lane][31] : T(0);
    bool spd = true;
    int fail = 0;                                   // first non-positive Cholesky pivot (1-based)
    for (int k = 0; k < n; ++k) {
      const T piv = M[k][k];
      if (spd && !(piv > T(0))) fail = k + 1;
      spd = spd && (piv > T(0));
      const T lkk = sqrt(piv > T(0) ? piv : T(1));
      __syncwarp();
      if (lane > k && lane < n) M[lane][k] /= lkk;
      __syncwarp();
      if (lane > k && lane < n) {
        const T lik = M[lane][k];
        for (int j = k + 1; j <= lane; ++j) M[lane][j] = fma(-lik, M[j][k], M[lane][j]);
      }
      if (lane == k) M[k][k] = lkk;
      __syncwarp();
    }
    // L y = rhs (column sweep), then L^T x = y
    for (int i = 0; i < n; ++i) {
      const T yi = __shfl_sync(full, rhs, i) / M[i][i];
      if (lane == i) rhs = yi;
      if (lane > i && lane < n) rhs = fma(-M[lane][i], yi, rhs);
    }
    for (int i = n - 1; i >= 0; --i) {
      const T xi = __shfl_sync(full, rhs, i) / M[i][i];
      if (lane == i) rhs = xi;
      if (lane < i) rhs = fma(-M[i][lane], xi, rhs);
    }
    if (lane < n) qdd_out[(int64_t)lane * B + b] = spd ? rhs : T(NAN);
    if (status && lane == 0) status[b] = fail;
    __syncwarp();
  }
}

// ---------------------------------------------------------------- CTA-wide variant (31 < n <= 256)
// The paper's fd_200 comparison: one CTA per state, thread j < n
// computes column j of M(q) (Eq. 17), thread n tau_bias (Eq. 5), each with the
// same stash-free register RNEA as the warp kernel; M (n x n, plus tau_bias in
// column n) lives in a per-CTA global workspace (L1/L2-resident), factorised by
// a right-looking Cholesky with one barrier per column (rows of the trailing
// update spread over the threads), then the two triangular solves with one
// barrier per step.  O(n^3) per state: the cost the paper attributes to JSIIA
// at large n.
constexpr int kJsBlockMaxN = 256;
constexpr int kJsBlockThreads = 288;      // >= n + 1, whole warps

template <typename T, bool SMEM>
__global__ void __launch_bounds__(kJsBlockThreads)
jsiia_block_kernel(int n, const LinkConst<T>* __restrict__ Lg, const Boundary<T> bnd, int64_t B,
                   const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ tau_in,
                   T* __restrict__ qdd_out, int32_t* __restrict__ status, T* __restrict__ ws) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ T strf[3][kJsBlockMaxN];
  __shared__ T rhs[kJsBlockMaxN];
  __shared__ T s_piv;
  __shared__ int s_fail;
  const int t = threadIdx.x, nt = blockDim.x;
  const int ld = n + 1;                                    // row stride of M (column n = tau_bias)
  // M in shared memory when it fits (n <= 160 fp64), else a per-CTA global workspace
  T* M = SMEM ? reinterpret_cast<T*>(smem_raw) : ws + (size_t)blockIdx.x * (size_t)n * ld;
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    for (int l = t; l < n; l += nt) {                      // CalcTransform, link l
      const T ql = __ldg(q + (int64_t)l * B + b);
      T s, c;
      rd_sincos(Lg[l].alpha * ql, &s, &c);
      strf[0][l] = s;
      strf[1][l] = c;
      strf[2][l] = Lg[l].beta * ql;
    }
    __syncthreads();
    if (t <= n) {
      const bool bias = t == n;
      T V[6], Vd[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) { V[k] = bias ? bnd.V0[k] : T(0); Vd[k] = bias ? bnd.Vd0[k] : T(0); }
      for (int i = 0; i < n; ++i) {
        const LinkConst<T> C = Lg[i];
        const T s = strf[0][i], c = strf[1][i], d = strf[2][i];
        const Rot<T> R = make_rot(C, s, c);
        const T p0 = fma(d, C.Rm[2], C.pm[0]), p1 = fma(d, C.Rm[5], C.pm[1]), p2 = fma(d, C.Rm[8], C.pm[2]);
        const T qdi = bias ? __ldg(qd + (int64_t)i * B + b) : T(0);
        const T qddi = (t == i) ? T(1) : T(0);
        T Vn[6], Vdn[6];
        fwd_step<T, false>(C, R, p0, p1, p2, qdi, qddi, V, Vd, Vn, Vdn);
#pragma unroll
        for (int k = 0; k < 6; ++k) { V[k] = Vn[k]; Vd[k] = Vdn[k]; }
      }
      T F[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) F[k] = bias ? bnd.Ftip[k] : T(0);
      Rot<T> Rn{1, 0, 0, 0, 1, 0, 0, 0, 1};
      T pn0 = 0, pn1 = 0, pn2 = 0;
      for (int i = n - 1; i >= 0; --i) {
        const LinkConst<T> C = Lg[i];
        T Fh[6], Fo[6];
        bias_force(C, V, Vd, Fh);
        bwd_step(Rn, pn0, pn1, pn2, F, Fh, Fo);
#pragma unroll
        for (int k = 0; k < 6; ++k) F[k] = Fo[k];
        M[(size_t)i * ld + t] = fma(C.beta, F[2], C.alpha * F[5]);   // column t (t = n: tau_bias)
        const T s = strf[0][i], c = strf[1][i], d = strf[2][i];
        Rn = make_rot(C, s, c);
        pn0 = fma(d, C.Rm[2], C.pm[0]); pn1 = fma(d, C.Rm[5], C.pm[1]); pn2 = fma(d, C.Rm[8], C.pm[2]);
        const T qdi = bias ? __ldg(qd + (int64_t)i * B + b) : T(0);
        const T qddi = (t == i) ? T(1) : T(0);
        const T a = C.alpha, be = C.beta, aq = a * qdi, bq = be * qdi;
        T x[6], y[6];
        y[0] = Vd[0] - fma(bq, V[4], aq * V[1]);
        y[1] = Vd[1] + fma(bq, V[3], aq * V[0]);
        y[2] = Vd[2] - be * qddi;
        y[3] = Vd[3] - aq * V[4];
        y[4] = Vd[4] + aq * V[3];
        y[5] = Vd[5] - a * qddi;
#pragma unroll
        for (int k = 0; k < 6; ++k) x[k] = V[k];
        x[2] -= bq;
        x[5] -= aq;
        ad_f(Rn, pn0, pn1, pn2, x, V);
        ad_f(Rn, pn0, pn1, pn2, y, Vd);
      }
    }
    if (t == 0) s_fail = 0;
    __syncthreads();
    for (int i = t; i < n; i += nt) rhs[i] = __ldg(tau_in + (int64_t)i * B + b) - M[(size_t)i * ld + n];   // line 2
    // Cholesky M = L L^T, lower triangle in place
    for (int k = 0; k < n; ++k) {
      if (t == 0) {
        const T piv = M[(size_t)k * ld + k];
        if (s_fail == 0 && !(piv > T(0))) s_fail = k + 1;
        const T lkk = sqrt(piv > T(0) ? piv : T(1));
        M[(size_t)k * ld + k] = lkk;
        s_piv = lkk;
      }
      __syncthreads();
      const T inv = T(1) / s_piv;
      for (int i = k + 1 + t; i < n; i += nt) M[(size_t)i * ld + k] *= inv;
      __syncthreads();
      // trailing update, one column j per thread: at each row i the threads of a
      // warp touch consecutive M[i][j] (coalesced / conflict-free) and share M[i][k]
      for (int j = k + 1 + t; j < n; j += nt) {
        const T ljk = M[(size_t)j * ld + k];
#pragma unroll 4
        for (int i = j; i < n; ++i) M[(size_t)i * ld + j] = fma(-M[(size_t)i * ld + k], ljk, M[(size_t)i * ld + j]);
      }
      __syncthreads();
    }
    // L y = rhs, then L^T x = y (column sweeps)
    for (int i = 0; i < n; ++i) {
      const T yi = rhs[i] / M[(size_t)i * ld + i];
      __syncthreads();
      for (int j = i + 1 + t; j < n; j += nt) rhs[j] = fma(-M[(size_t)j * ld + i], yi, rhs[j]);
      if (t == 0) rhs[i] = yi;
      __syncthreads();
    }
    for (int i = n - 1; i >= 0; --i) {
      const T xi = rhs[i] / M[(size_t)i * ld + i];
      __syncthreads();
      for (int j = t; j < i; j += nt) rhs[j] = fma(-M[(size_t)i * ld + j], xi, rhs[j]);
      if (t == 0) rhs[i] = xi;
      __syncthreads();
    }
    const bool spd = s_fail == 0;
    for (int i = t; i < n; i += nt) qdd_out[(int64_t)i * B + b] = spd ? rhs[i] : T(NAN);
    if (status && t == 0) status[b] = s_fail;
    __syncthreads();
  }
}

constexpr size_t kJsSmemMax = 200 * 1024;   // + ~9 KB static: one CTA per SM
int64_t jsiia_block_grid(int64_t B) { return B < (int64_t)num_sms() * 2 ? B : (int64_t)num_sms() * 2; }
size_t jsiia_ws_elems(int n, int64_t B) {
  return n > 31 ? (size_t)jsiia_block_grid(B) * (size_t)n * (size_t)(n + 1) : 0;
}

template <typename T>
cudaError_t launch_jsiia(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                         const T* qd, const T* tau, T* qdd, cudaStream_t st, int* launches, bool* supported,
                         int32_t* status, T* ws) {
  *supported = n >= 1 && n <= kJsBlockMaxN;
  if (!*supported) return cudaSuccess;
  if (n > 31) {
    const int threads = ((n + 1 + 31) / 32) * 32;
    const size_t mbytes = (size_t)n * (n + 1) * sizeof(T);
    ++*launches;
    if (mbytes <= kJsSmemMax) {
      static thread_local int attr_dev = -1;
      int dev = 0;
      cudaGetDevice(&dev);
      if (attr_dev != dev) {
        cudaError_t e = cudaFuncSetAttribute(jsiia_block_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kJsSmemMax);
        if (e != cudaSuccess) return e;
        attr_dev = dev;
      }
      const int64_t grid = B < (int64_t)num_sms() ? B : (int64_t)num_sms();
      jsiia_block_kernel<T, true><<<(unsigned)grid, threads, mbytes, st>>>(n, L_dev, bnd, B, q, qd, tau, qdd,
                                                                           status, ws);
    } else {
      jsiia_block_kernel<T, false><<<(unsigned)jsiia_block_grid(B), threads, 0, st>>>(n, L_dev, bnd, B, q, qd, tau,
                                                                                      qdd, status, ws);
    }
    return cudaGetLastError();
  }
  int64_t grid = (B + kJsWarps - 1) / kJsWarps;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (grid > cap) grid = cap;
  jsiia_kernel<T><<<(unsigned)grid, kJsWarps * 32, 0, st>>>(n, L_dev, bnd, B, q, qd, tau, qdd, status);
  ++*launches;
  return cudaGetLastError();
}

template cudaError_t launch_jsiia<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                          const double*, const double*, const double*, double*, cudaStream_t,
                                          int*, bool*, int32_t*, double*);
template cudaError_t launch_jsiia<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                         const float*, const float*, const float*, float*, cudaStream_t, int*,
                                         bool*, int32_t*, float*);

}  // namespace rd
