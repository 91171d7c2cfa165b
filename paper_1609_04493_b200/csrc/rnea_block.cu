// rnea_block.cu -- one CTA per state, thread = link, for long chains in the
// latency regime (strategy BLOCK_SCAN, n <= 512; the
// paper's single-robot experiment, "GPU time ~ log n").
//
// Same base-frame scan formulation as rnea_warp.cu (Alg. 1's two forward scans
// as one SE(3) prefix product plus vector prefix sums, the backward force scan
// as a suffix sum), with each scan done across the whole CTA: Kogge-Stone
// inside every warp, a scan of the per-warp totals by warp 0 in shared memory,
// then every warp folds in the total of the warps before (after) it.
// Depth: 2 * ceil(log2 32) + 1 combine rounds per scan for n <= 512.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"

namespace rd {

template <typename T>
struct SE3 { Rot<T> R; T p0, p1, p2; };

template <typename T>
__device__ __forceinline__ SE3<T> se3_mul(const SE3<T>& a, const SE3<T>& b) {    // a o b
  SE3<T> c;
  c.R.r00 = fma(a.R.r00, b.R.r00, fma(a.R.r01, b.R.r10, a.R.r02 * b.R.r20));
  c.R.r01 = fma(a.R.r00, b.R.r01, fma(a.R.r01, b.R.r11, a.R.r02 * b.R.r21));
  c.R.r02 = fma(a.R.r00, b.R.r02, fma(a.R.r01, b.R.r12, a.R.r02 * b.R.r22));
  c.R.r10 = fma(a.R.r10, b.R.r00, fma(a.R.r11, b.R.r10, a.R.r12 * b.R.r20));
  c.R.r11 = fma(a.R.r10, b.R.r01, fma(a.R.r11, b.R.r11, a.R.r12 * b.R.r21));
  c.R.r12 = fma(a.R.r10, b.R.r02, fma(a.R.r11, b.R.r12, a.R.r12 * b.R.r22));
  c.R.r20 = fma(a.R.r20, b.R.r00, fma(a.R.r21, b.R.r10, a.R.r22 * b.R.r20));
  c.R.r21 = fma(a.R.r20, b.R.r01, fma(a.R.r21, b.R.r11, a.R.r22 * b.R.r21));
  c.R.r22 = fma(a.R.r20, b.R.r02, fma(a.R.r21, b.R.r12, a.R.r22 * b.R.r22));
  c.p0 = fma(a.R.r00, b.p0, fma(a.R.r01, b.p1, fma(a.R.r02, b.p2, a.p0)));
  c.p1 = fma(a.R.r10, b.p0, fma(a.R.r11, b.p1, fma(a.R.r12, b.p2, a.p1)));
  c.p2 = fma(a.R.r20, b.p0, fma(a.R.r21, b.p1, fma(a.R.r22, b.p2, a.p2)));
  return c;
}

template <typename T>
__device__ __forceinline__ SE3<T> se3_shfl_up(const SE3<T>& a, int d) {
  SE3<T> o;
  const unsigned f = 0xffffffffu;
  o.R.r00 = __shfl_up_sync(f, a.R.r00, d); o.R.r01 = __shfl_up_sync(f, a.R.r01, d); o.R.r02 = __shfl_up_sync(f, a.R.r02, d);
  o.R.r10 = __shfl_up_sync(f, a.R.r10, d); o.R.r11 = __shfl_up_sync(f, a.R.r11, d); o.R.r12 = __shfl_up_sync(f, a.R.r12, d);
  o.R.r20 = __shfl_up_sync(f, a.R.r20, d); o.R.r21 = __shfl_up_sync(f, a.R.r21, d); o.R.r22 = __shfl_up_sync(f, a.R.r22, d);
  o.p0 = __shfl_up_sync(f, a.p0, d); o.p1 = __shfl_up_sync(f, a.p1, d); o.p2 = __shfl_up_sync(f, a.p2, d);
  return o;
}

template <typename T>
__device__ __forceinline__ SE3<T> se3_identity() {
  SE3<T> g;
  g.R = Rot<T>{1, 0, 0, 0, 1, 0, 0, 0, 1};
  g.p0 = g.p1 = g.p2 = 0;
  return g;
}

// CTA-wide inclusive prefix product g_l = x_0 o x_1 o ... o x_l (earlier on the left)
template <typename T>
__device__ SE3<T> block_se3_scan(SE3<T> x, SE3<T>* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const SE3<T> e = se3_shfl_up(x, d);
    if (lane >= d) x = se3_mul(e, x);
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    SE3<T> t = lane < nw ? sh[lane] : se3_identity<T>();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const SE3<T> e = se3_shfl_up(t, d);
      if (lane >= d) t = se3_mul(e, t);
    }
    if (lane < nw) sh[lane] = t;
  }
  __syncthreads();
  if (warp > 0) x = se3_mul(sh[warp - 1], x);
  __syncthreads();
  return x;
}

// CTA-wide inclusive prefix (UP) or suffix (!UP) sum of a 6-vector
template <typename T, bool UP>
__device__ void block_vec_scan(T (&v)[6], T* sh /* [32][6] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const T o = UP ? __shfl_up_sync(0xffffffffu, v[k], d) : __shfl_down_sync(0xffffffffu, v[k], d);
      if (UP ? lane >= d : lane + d < 32) v[k] += o;
    }
  }
  if (lane == (UP ? 31 : 0)) {
#pragma unroll
    for (int k = 0; k < 6; ++k) sh[6 * warp + k] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
    T t[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) t[k] = lane < nw ? sh[6 * lane + k] : T(0);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const T o = UP ? __shfl_up_sync(0xffffffffu, t[k], d) : __shfl_down_sync(0xffffffffu, t[k], d);
        if (UP ? lane >= d : lane + d < 32) t[k] += o;
      }
    }
    if (lane < nw) {
#pragma unroll
      for (int k = 0; k < 6; ++k) sh[6 * lane + k] = t[k];
    }
  }
  __syncthreads();
  if (UP ? warp > 0 : warp + 1 < nw) {
    const int w = UP ? warp - 1 : warp + 1;
#pragma unroll
    for (int k = 0; k < 6; ++k) v[k] += sh[6 * w + k];
  }
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(512)
rnea_block_kernel(int n, const LinkConst<T>* __restrict__ Lg, const Boundary<T> bnd, int64_t B,
                  const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ qdd,
                  T* __restrict__ tau) {
  __shared__ SE3<T> shg[32];
  __shared__ T shv[32 * 6];
  const int l = threadIdx.x;
  const bool act = l < n;
  LinkConst<T> C;
  if (act) {
    C = Lg[l];
  } else {                                   // padding link: identity transform, no mass, no joint
    for (int k = 0; k < 9; ++k) C.Rm[k] = (k % 4 == 0) ? T(1) : T(0);
    for (int k = 0; k < 3; ++k) { C.pm[k] = 0; C.h[k] = 0; }
    for (int k = 0; k < 6; ++k) C.I[k] = 0;
    C.m = 0;
    C.alpha = 0;
    C.beta = 0;
  }
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    T qi = 0, qdi = 0, qddi = 0;
    if (act) {
      qi = __ldg(q + (int64_t)l * B + b);
      qdi = __ldg(qd + (int64_t)l * B + b);
      qddi = qdd ? __ldg(qdd + (int64_t)l * B + b) : T(0);   // qdd == nullptr: tau_bias (Eq. 5)
    }
    // CalcTransform, then the SE(3) scan g_{0,l}
    T s, cc;
    rd_sincos(C.alpha * qi, &s, &cc);
    SE3<T> g;
    g.R = make_rot(C, s, cc);
    const T d = C.beta * qi;
    g.p0 = fma(d, C.Rm[2], C.pm[0]); g.p1 = fma(d, C.Rm[5], C.pm[1]); g.p2 = fma(d, C.Rm[8], C.pm[2]);
    g = block_se3_scan(g, shg);
    const Rot<T>& R = g.R;
    const T p0 = g.p0, p1 = g.p1, p2 = g.p2;
    // S0 = Ad_g S, V0 = V_0 + prefix sum of S0 qd
    const T z0 = R.r02, z1 = R.r12, z2 = R.r22;
    T S0[6];
    S0[0] = fma(C.beta, z0, C.alpha * (p1 * z2 - p2 * z1));
    S0[1] = fma(C.beta, z1, C.alpha * (p2 * z0 - p0 * z2));
    S0[2] = fma(C.beta, z2, C.alpha * (p0 * z1 - p1 * z0));
    S0[3] = C.alpha * z0;
    S0[4] = C.alpha * z1;
    S0[5] = C.alpha * z2;
    T V[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) V[k] = S0[k] * qdi;
    block_vec_scan<T, true>(V, shv);
#pragma unroll
    for (int k = 0; k < 6; ++k) V[k] += bnd.V0[k];
    // Vd0 = Vd_0 + prefix sum of (S0 qdd + ad_{V0}(S0 qd))
    T A[6];
    {
      const T x0 = S0[0] * qdi, x1 = S0[1] * qdi, x2 = S0[2] * qdi;
      const T y0 = S0[3] * qdi, y1 = S0[4] * qdi, y2 = S0[5] * qdi;
      A[0] = fma(S0[0], qddi, (V[4] * x2 - V[5] * x1) + (V[1] * y2 - V[2] * y1));
      A[1] = fma(S0[1], qddi, (V[5] * x0 - V[3] * x2) + (V[2] * y0 - V[0] * y2));
      A[2] = fma(S0[2], qddi, (V[3] * x1 - V[4] * x0) + (V[0] * y1 - V[1] * y0));
      A[3] = fma(S0[3], qddi, V[4] * y2 - V[5] * y1);
      A[4] = fma(S0[4], qddi, V[5] * y0 - V[3] * y2);
      A[5] = fma(S0[5], qddi, V[3] * y1 - V[4] * y0);
    }
    block_vec_scan<T, true>(A, shv);
#pragma unroll
    for (int k = 0; k < 6; ++k) A[k] += bnd.Vd0[k];
    // bias wrench per link (body frame), moved to the base frame
    T Vb[6], Ab[6], Fh[6], F[6];
    ad_finv(R, p0, p1, p2, V, Vb);
    ad_finv(R, p0, p1, p2, A, Ab);
    bias_force(C, Vb, Ab, Fh);
    const T zero6[6] = {0, 0, 0, 0, 0, 0};
    bwd_step(R, p0, p1, p2, Fh, zero6, F);
    if (!act) {
#pragma unroll
      for (int k = 0; k < 6; ++k) F[k] = 0;
    }
    if (l == n - 1) {
      T Ft[6];
      bwd_step(R, p0, p1, p2, bnd.Ftip, zero6, Ft);
#pragma unroll
      for (int k = 0; k < 6; ++k) F[k] += Ft[k];
    }
    block_vec_scan<T, false>(F, shv);          // backward force scan (Eq. 16) = suffix sum
    T t = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) t = fma(S0[k], F[k], t);
    if (act) tau[(int64_t)l * B + b] = t;
  }
}

template <typename T>
cudaError_t launch_rnea_block(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                              const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                              bool* supported) {
  *supported = n >= 1 && n <= 512;
  if (!*supported) return cudaSuccess;
  const int threads = ((n + 31) / 32) * 32;
  int64_t grid = B;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (grid > cap) grid = cap;
  rnea_block_kernel<T><<<(unsigned)grid, threads, 0, st>>>(n, L_dev, bnd, B, q, qd, qdd, tau);
  ++*launches;
  return cudaGetLastError();
}

template cudaError_t launch_rnea_block<double>(int, const LinkConst<double>*, const Boundary<double>&, int64_t,
                                               const double*, const double*, const double*, double*, cudaStream_t,
                                               int*, bool*);
template cudaError_t launch_rnea_block<float>(int, const LinkConst<float>*, const Boundary<float>&, int64_t,
                                              const float*, const float*, const float*, float*, cudaStream_t, int*,
                                              bool*);

}  // namespace rd
