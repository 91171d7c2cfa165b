// rnea_chunk.cu -- L lanes per state, each lane one CHUNK of c = ceil(n/L)
// consecutive links (strategy CHUNK, L in {2, 4, 8, 16, 32}, any n, revolute and
// prismatic joints in DH frames).
//
// The two scans of Alg. 1 at chunk granularity: every lane runs the
// serial recursions of Eq. (1)-(2) over its own links, and the L chunk results of
// one state are combined with log2(L)-round shuffle scans -- the paper's scan
// decomposition (Eq. 12-16) with the chunk, not the link, as the scan
// element, so that per-state storage is spread over L lanes (SURVEY §8(a) a8,
// "(or L-chunks)"; the paper's "scan data fitted into shared memory and local
// registers").
//
//  pass 1 (forward, local): lane j composes its chunk's element of the Eq. (13)
//    semigroup, acting on (Vdot, V):  V' = X V + xi2,  Vdot' = X Vdot + xi1 -
//    ad_{xi2}(X V), X = Ad_{g^-1}, g = f_s ... f_e (the chunk's SE(3) product,
//    frame e -> frame s-1); (xi2, xi1) are (V_e, Vdot_e) of the chunk run from
//    V_{s-1} = Vdot_{s-1} = 0, i.e. the serial recursion itself.  (sin, cos) of
//    every link go to the stash.
//  forward scan: inclusive Kogge-Stone over the L lanes with the semigroup
//    product (earlier element applied first, reading A4):
//      g = g_a g_b,  xi2 = X_b xi2_a + xi2_b,
//      xi1 = X_b xi1_a + xi1_b - ad_{xi2_b}(X_b xi2_a);
//    the exclusive prefix applied to (V_0, Vdot_0) is the chunk's (V_{s-1}, Vdot_{s-1}).
//  pass 2 (forward, true): Eq. (1) from (V_{s-1}, Vdot_{s-1}); the bias wrench
//    Fhat_i (at the centre of mass) goes to the stash.
//  pass A (backward, local): Eq. (2) over the chunk with zero wrench from the tip
//    side, then G_j = Ad^T_{f_s^-1} F_s: the chunk's wrench pushed into frame s-1.
//  backward scan: suffix Kogge-Stone of the affine maps x -> G_j + Ad^T_{g_j^-1} x
//    (the Eq. (16) operator at chunk granularity): (g_j g_k, G_j + Ad^T_{g_j^-1} G_k);
//    applied to F_{n+1} (f_{n,n+1} = I, A5) it gives the wrench entering chunk j
//    from the tip side.
//  pass B (backward, true): Eq. (2) from that wrench; tau_i = S_i^T F_i.
//
// The per-link stash (sin, cos, Fhat) = 8 scalars is a slot-contiguous global
// workspace (L2-resident): ws[(t * 8 + k) * NL + lane_global], t = link within the
// chunk, so a warp's access is 32 consecutive scalars.  Work per link is about
// 1.7x the THREAD kernel's (pass 1 and pass A repeat the recursions to build the
// scan elements); what it buys is log-depth latency per state at L lanes, for
// batches too small to fill the GPU with one thread per state.
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"

namespace rd {

constexpr int kChunkThreads = 128;
constexpr int kChunkMinBlocks = 3;     // 168-register cap (no spills in fp64): 12 warps per SM
constexpr int kChunkPerLink = 8;       // stash scalars per link: sin, cos, Fhat
constexpr int kPD = 4;                 // forward passes: inputs / stash read this many links ahead
constexpr int kBPD = 2;                // backward passes: stash read this many links ahead

// SE(3) element g = (R, p) as 12 scalars.
template <typename T>
struct SE3 {
  Rot<T> R;
  T p0, p1, p2;
};
template <typename T>
__device__ __forceinline__ SE3<T> se3_identity() {
  SE3<T> g;
  g.R = Rot<T>{1, 0, 0, 0, 1, 0, 0, 0, 1};
  g.p0 = g.p1 = g.p2 = 0;
  return g;
}
// a * b
template <typename T>
__device__ __forceinline__ SE3<T> se3_mul(const SE3<T>& a, const SE3<T>& b) {
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
// g <- g * f with f = Rx(alpha) Tx(a) Rz(theta) Tz(d) (modified DH):
// R f_R = (R Rx) Rz, p += R (a, -sa d, ca d) = a R e_x + d (R Rx) e_z.
template <typename T>
__device__ __forceinline__ void se3_mul_dh(SE3<T>& g, T ca, T sa, T a, T d, T s, T c) {
  // R1 = R Rx(alpha): columns (R0, ca R1 + sa R2, -sa R1 + ca R2)
  const T c1x = fma(ca, g.R.r01, sa * g.R.r02), c1y = fma(ca, g.R.r11, sa * g.R.r12),
          c1z = fma(ca, g.R.r21, sa * g.R.r22);
  const T c2x = fma(ca, g.R.r02, -(sa * g.R.r01)), c2y = fma(ca, g.R.r12, -(sa * g.R.r11)),
          c2z = fma(ca, g.R.r22, -(sa * g.R.r21));
  g.p0 = fma(a, g.R.r00, fma(d, c2x, g.p0));
  g.p1 = fma(a, g.R.r10, fma(d, c2y, g.p1));
  g.p2 = fma(a, g.R.r20, fma(d, c2z, g.p2));
  // R2 = R1 Rz(theta): columns (c R0 + s c1, -s R0 + c c1, c2)
  const T n0x = fma(c, g.R.r00, s * c1x), n0y = fma(c, g.R.r10, s * c1y), n0z = fma(c, g.R.r20, s * c1z);
  const T n1x = fma(c, c1x, -(s * g.R.r00)), n1y = fma(c, c1y, -(s * g.R.r10)), n1z = fma(c, c1z, -(s * g.R.r20));
  g.R.r00 = n0x; g.R.r10 = n0y; g.R.r20 = n0z;
  g.R.r01 = n1x; g.R.r11 = n1y; g.R.r21 = n1z;
  g.R.r02 = c2x; g.R.r12 = c2y; g.R.r22 = c2z;
}
// out = ad_xi(x) = (w x x_v + v x x_w, w x x_w), xi = (v, w)
template <typename T>
__device__ __forceinline__ void ad_twist(const T* xi, const T* x, T* out) {
  const T v0 = xi[0], v1 = xi[1], v2 = xi[2], w0 = xi[3], w1 = xi[4], w2 = xi[5];
  out[0] = fma(w1, x[2], fma(-w2, x[1], fma(v1, x[5], -(v2 * x[4]))));
  out[1] = fma(w2, x[0], fma(-w0, x[2], fma(v2, x[3], -(v0 * x[5]))));
  out[2] = fma(w0, x[1], fma(-w1, x[0], fma(v0, x[4], -(v1 * x[3]))));
  out[3] = fma(w1, x[5], -(w2 * x[4]));
  out[4] = fma(w2, x[3], -(w0 * x[5]));
  out[5] = fma(w0, x[4], -(w1 * x[3]));
}

// Forward scan element (Eq. 13 semigroup on (Vdot, V), chunk granularity).
template <typename T>
struct FwdElem {
  SE3<T> g;
  T x2[6], x1[6];      // xi2 (velocity offset), xi1 (acceleration offset)
};
// a then b (a: the earlier chunk)
template <typename T>
__device__ __forceinline__ FwdElem<T> fwd_combine(const FwdElem<T>& a, const FwdElem<T>& b) {
  FwdElem<T> r;
  r.g = se3_mul(a.g, b.g);
  T Xa2[6], Xa1[6], ad[6];
  ad_finv(b.g.R, b.g.p0, b.g.p1, b.g.p2, a.x2, Xa2);
  ad_finv(b.g.R, b.g.p0, b.g.p1, b.g.p2, a.x1, Xa1);
  ad_twist(b.x2, Xa2, ad);
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    r.x2[k] = Xa2[k] + b.x2[k];
    r.x1[k] = Xa1[k] + b.x1[k] - ad[k];
  }
  return r;
}
template <typename T>
__device__ __forceinline__ T shfl_up_w(T v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
template <typename T>
__device__ __forceinline__ T shfl_dn_w(T v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
template <typename T, bool UP>
__device__ __forceinline__ SE3<T> shfl_se3(const SE3<T>& g, int d) {
  SE3<T> r;
  const T* src = &g.R.r00;
  T* dst = &r.R.r00;
#pragma unroll
  for (int k = 0; k < 9; ++k) dst[k] = UP ? shfl_up_w(src[k], d) : shfl_dn_w(src[k], d);
  r.p0 = UP ? shfl_up_w(g.p0, d) : shfl_dn_w(g.p0, d);
  r.p1 = UP ? shfl_up_w(g.p1, d) : shfl_dn_w(g.p1, d);
  r.p2 = UP ? shfl_up_w(g.p2, d) : shfl_dn_w(g.p2, d);
  return r;
}

// Eq. (2) over one chunk (links s0 .. s0+cnt-1, tip to base) from the wrench Fin
// entering link s0+cnt-1 from its child side (already in that link's frame):
// F_i = Fhat_i + Ad^T_{f_{i+1}^-1} F_{i+1}.  Stores tau_i = S_i^T F_i if tau
// (and store); returns G = Ad^T_{f_s0^-1} F_s0, the chunk's wrench in frame s0-1.
template <typename T, bool PR>
__device__ __forceinline__ void chunk_backward(const LinkDHc<T>* Ls, const unsigned char* PRs,
                                               const T* __restrict__ q, int64_t B, int64_t b,
                                               const T* __restrict__ w, int64_t NL, int s0, int cnt, const T* Fin,
                                               T* __restrict__ tau, bool store, T* G) {
  T F[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) F[k] = Fin[k];
  T cca = 1, csa = 0, cav = 0, cd = 0, csn = 0, ccn = 1;    // child transform: identity at the chunk end
  // stash (sin, cos, Fhat) [and q] of the next kBPD links (tip to base) in flight
  T rw[kBPD][kChunkPerLink], rq[kBPD];
#pragma unroll
  for (int u = 0; u < kBPD; ++u) {
    const int tu = max(0, cnt - 1 - u);
#pragma unroll
    for (int k = 0; k < kChunkPerLink; ++k) rw[u][k] = cnt > 0 ? w[(int64_t)(tu * kChunkPerLink + k) * NL] : T(0);
    rq[u] = (PR && cnt > 0) ? __ldg(q + (int64_t)(s0 + tu) * B + b) : T(0);
  }
#pragma unroll kBPD
  for (int t = cnt - 1; t >= 0; --t) {
    const int i = s0 + t;
    const LinkDHc<T>& C = Ls[i];
    const bool pz = PR && PRs[i];
    T cur[kChunkPerLink];
#pragma unroll
    for (int k = 0; k < kChunkPerLink; ++k) cur[k] = rw[0][k];
    const T qi = rq[0];
#pragma unroll
    for (int u = 0; u + 1 < kBPD; ++u) {
#pragma unroll
      for (int k = 0; k < kChunkPerLink; ++k) rw[u][k] = rw[u + 1][k];
      rq[u] = rq[u + 1];
    }
    {
      const int tu = max(0, t - kBPD);
#pragma unroll
      for (int k = 0; k < kChunkPerLink; ++k) rw[kBPD - 1][k] = w[(int64_t)(tu * kChunkPerLink + k) * NL];
      rq[kBPD - 1] = PR ? __ldg(q + (int64_t)(s0 + tu) * B + b) : T(0);
    }
    T Fo[6];
    dh_bwd(cca, csa, cav, cd, csn, ccn, F, cur + 2, Fo);
#pragma unroll
    for (int k = 0; k < 6; ++k) F[k] = Fo[k];
    if (tau && store) tau[(int64_t)i * B + b] = pz ? F[2] : F[5];
    cca = C.ca; csa = C.sa; cav = C.a;
    cd = pz ? C.d + qi : C.d;
    csn = cur[0];
    ccn = cur[1];
  }
  const T zero[6] = {0, 0, 0, 0, 0, 0};
  dh_bwd(cca, csa, cav, cd, csn, ccn, F, zero, G);
}

template <typename T, int L, bool PR>
__global__ void __launch_bounds__(kChunkThreads, kChunkMinBlocks)
rnea_chunk_kernel(int n, int c, const LinkDHc<T>* __restrict__ Lg, const Boundary<T> bnd, int64_t B,
                  const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ qdd,
                  T* __restrict__ tau, const unsigned char* __restrict__ prism_g, T* __restrict__ ws) {
  static_assert(L >= 2 && L <= 32 && (L & (L - 1)) == 0, "L: power of two in [2, 32]");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LinkDHc<T>* Ls = reinterpret_cast<LinkDHc<T>*>(smem_raw);      // model constants, broadcast reads
  unsigned char* PRs = smem_raw + (size_t)n * sizeof(LinkDHc<T>);
  for (int i = threadIdx.x; i < n * (int)(sizeof(LinkDHc<T>) / sizeof(T)); i += blockDim.x)
    reinterpret_cast<T*>(Ls)[i] = reinterpret_cast<const T*>(Lg)[i];
  if (PR)
    for (int i = threadIdx.x; i < n; i += blockDim.x) PRs[i] = prism_g[i];
  __syncthreads();

  constexpr int SPW = 32 / L;                               // states per warp
  const int lane = threadIdx.x & 31;
  const int j = lane % L;                                   // chunk index of this lane
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t NL = (int64_t)gridDim.x * blockDim.x;      // lanes in the grid (workspace pitch)
  T* __restrict__ w = ws + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int s0 = j * c;
  const int cnt = max(0, min(n, s0 + c) - s0);              // links of this chunk (0: empty chunk)

  for (int64_t base = gwarp * SPW; base < B; base += nwarps * SPW) {
    const int64_t bs = base + lane / L;
    const bool valid = bs < B;
    const int64_t b = valid ? bs : B - 1;                   // idle lanes compute a copy of the last state
    // ---------------- pass 1: the chunk's semigroup element
    FwdElem<T> E;
    E.g = se3_identity<T>();
#pragma unroll
    for (int k = 0; k < 6; ++k) { E.x2[k] = 0; E.x1[k] = 0; }
    // inputs kPD links ahead (independent of the recursion chain; unrolled by kPD so
    // the ring stays in fixed registers)
    T rq[kPD], rqd[kPD], rqa[kPD];
#pragma unroll
    for (int u = 0; u < kPD; ++u) {
      const int64_t o = (int64_t)(s0 + max(0, min(u, cnt - 1))) * B + b;
      if (cnt > 0) { rq[u] = __ldg(q + o); rqd[u] = __ldg(qd + o); rqa[u] = __ldg(qdd + o); }
      else { rq[u] = rqd[u] = rqa[u] = T(0); }
    }
#pragma unroll kPD
    for (int t = 0; t < cnt; ++t) {
      const int i = s0 + t;
      const T qi = rq[0], qdi = rqd[0], qai = rqa[0];
#pragma unroll
      for (int u = 0; u + 1 < kPD; ++u) { rq[u] = rq[u + 1]; rqd[u] = rqd[u + 1]; rqa[u] = rqa[u + 1]; }
      {
        const int64_t o = (int64_t)(s0 + min(t + kPD, cnt - 1)) * B + b;
        rq[kPD - 1] = __ldg(q + o); rqd[kPD - 1] = __ldg(qd + o); rqa[kPD - 1] = __ldg(qdd + o);
      }
      const LinkDHc<T>& C = Ls[i];
      const bool pz = PR && PRs[i];
      T s, cs, dl;
      dh_link<PR>(C, pz, qi, &s, &cs, &dl);
      w[(int64_t)(t * kChunkPerLink + 0) * NL] = s;
      w[(int64_t)(t * kChunkPerLink + 1) * NL] = cs;
      T Vn[6], An[6];
      dh_ad_finv(C.ca, C.sa, C.a, dl, s, cs, E.x2, Vn);
      dh_ad_finv(C.ca, C.sa, C.a, dl, s, cs, E.x1, An);
      const T sr = pz ? T(0) : qdi, sp = pz ? qdi : T(0), ar = pz ? T(0) : qai, ap = pz ? qai : T(0);
      Vn[5] += sr;
      An[5] += ar;
      if (PR) { Vn[2] += sp; An[2] += ap; }
      An[0] = fma(sr, Vn[1], PR ? fma(sp, Vn[4], An[0]) : An[0]);
      An[1] = fma(-sr, Vn[0], PR ? fma(-sp, Vn[3], An[1]) : An[1]);
      An[3] = fma(sr, Vn[4], An[3]);
      An[4] = fma(-sr, Vn[3], An[4]);
#pragma unroll
      for (int k = 0; k < 6; ++k) { E.x2[k] = Vn[k]; E.x1[k] = An[k]; }
      se3_mul_dh(E.g, C.ca, C.sa, C.a, dl, s, cs);
    }
    const SE3<T> gj = E.g;                                  // the chunk's own product, for the backward scan
    // ---------------- forward scan (inclusive, then shifted by one lane)
#pragma unroll
    for (int d = 1; d < L; d <<= 1) {
      FwdElem<T> P;
      P.g = shfl_se3<T, true>(E.g, d);
#pragma unroll
      for (int k = 0; k < 6; ++k) { P.x2[k] = shfl_up_w(E.x2[k], d); P.x1[k] = shfl_up_w(E.x1[k], d); }
      if (j >= d) E = fwd_combine(P, E);
    }
    T V[6], A[6];
    {
      FwdElem<T> P;                                         // exclusive prefix: chunks 0 .. j-1
      P.g = shfl_se3<T, true>(E.g, 1);
#pragma unroll
      for (int k = 0; k < 6; ++k) { P.x2[k] = shfl_up_w(E.x2[k], 1); P.x1[k] = shfl_up_w(E.x1[k], 1); }
      if (j == 0) {
        P.g = se3_identity<T>();
#pragma unroll
        for (int k = 0; k < 6; ++k) { P.x2[k] = 0; P.x1[k] = 0; }
      }
      // (V_{s-1}, Vdot_{s-1}) = P applied to (V_0, Vdot_0)
      T XV[6], XA[6], ad[6];
      ad_finv(P.g.R, P.g.p0, P.g.p1, P.g.p2, bnd.V0, XV);
      ad_finv(P.g.R, P.g.p0, P.g.p1, P.g.p2, bnd.Vd0, XA);
      ad_twist(P.x2, XV, ad);
#pragma unroll
      for (int k = 0; k < 6; ++k) { V[k] = XV[k] + P.x2[k]; A[k] = XA[k] + P.x1[k] - ad[k]; }
    }
    // ---------------- pass 2: Eq. (1) from the true chunk input, Fhat to the stash
    {
      // (qd, qdd, q, sin, cos) of the next links in flight (L2 hits: read in pass 1)
      T rqd2[kPD], rqa2[kPD], rq2[kPD], rs[kPD], rc[kPD];
#pragma unroll
      for (int u = 0; u < kPD; ++u) {
        const int tu = max(0, min(u, cnt - 1));
        const int64_t o = (int64_t)(s0 + tu) * B + b;
        if (cnt > 0) {
          rqd2[u] = __ldg(qd + o); rqa2[u] = __ldg(qdd + o); rq2[u] = PR ? __ldg(q + o) : T(0);
          rs[u] = w[(int64_t)(tu * kChunkPerLink + 0) * NL]; rc[u] = w[(int64_t)(tu * kChunkPerLink + 1) * NL];
        } else {
          rqd2[u] = rqa2[u] = rq2[u] = rs[u] = rc[u] = T(0);
        }
      }
#pragma unroll kPD
      for (int t = 0; t < cnt; ++t) {
        const int i = s0 + t;
        const T qdi = rqd2[0], qai = rqa2[0], qi = rq2[0], s = rs[0], cs = rc[0];
#pragma unroll
        for (int u = 0; u + 1 < kPD; ++u) {
          rqd2[u] = rqd2[u + 1]; rqa2[u] = rqa2[u + 1]; rq2[u] = rq2[u + 1]; rs[u] = rs[u + 1]; rc[u] = rc[u + 1];
        }
        {
          const int tu = min(t + kPD, cnt - 1);
          const int64_t o = (int64_t)(s0 + tu) * B + b;
          rqd2[kPD - 1] = __ldg(qd + o); rqa2[kPD - 1] = __ldg(qdd + o); rq2[kPD - 1] = PR ? __ldg(q + o) : T(0);
          rs[kPD - 1] = w[(int64_t)(tu * kChunkPerLink + 0) * NL];
          rc[kPD - 1] = w[(int64_t)(tu * kChunkPerLink + 1) * NL];
        }
        const LinkDHc<T>& C = Ls[i];
        const bool pz = PR && PRs[i];
        const T dl = pz ? C.d + qi : C.d;
        T Vn[6], An[6];
        dh_ad_finv(C.ca, C.sa, C.a, dl, s, cs, V, Vn);
        dh_ad_finv(C.ca, C.sa, C.a, dl, s, cs, A, An);
        const T sr = pz ? T(0) : qdi, sp = pz ? qdi : T(0), ar = pz ? T(0) : qai, ap = pz ? qai : T(0);
        Vn[5] += sr;
        An[5] += ar;
        if (PR) { Vn[2] += sp; An[2] += ap; }
        An[0] = fma(sr, Vn[1], PR ? fma(sp, Vn[4], An[0]) : An[0]);
        An[1] = fma(-sr, Vn[0], PR ? fma(-sp, Vn[3], An[1]) : An[1]);
        An[3] = fma(sr, Vn[4], An[3]);
        An[4] = fma(-sr, Vn[3], An[4]);
        T Fh[6];
        bias_force_com(C, Vn, An, Fh);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          w[(int64_t)(t * kChunkPerLink + 2 + k) * NL] = Fh[k];
          V[k] = Vn[k];
          A[k] = An[k];
        }
      }
    }
    // ---------------- pass A: the chunk's own wrench, G_j = Ad^T_{f_s^-1} F_s with a zero tip side
    T G[6];
    {
      const T zero[6] = {0, 0, 0, 0, 0, 0};
      chunk_backward<T, PR>(Ls, PRs, q, B, b, w, NL, s0, cnt, zero, nullptr, false, G);
    }
    // ---------------- backward scan: suffix composition of x -> G_j + Ad^T_{g_j^-1} x
    SE3<T> gs = gj;
#pragma unroll
    for (int d = 1; d < L; d <<= 1) {
      const SE3<T> gn = shfl_se3<T, false>(gs, d);
      T Gn[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) Gn[k] = shfl_dn_w(G[k], d);
      if (j + d < L) {
        T AG[6];
        const T zero[6] = {0, 0, 0, 0, 0, 0};
        bwd_step(gs.R, gs.p0, gs.p1, gs.p2, Gn, zero, AG);      // Ad^T_{g^-1} Gn = (R f, p x R f + R m)
#pragma unroll
        for (int k = 0; k < 6; ++k) G[k] += AG[k];
        gs = se3_mul(gs, gn);
      }
    }
    // wrench entering chunk j from the tip side: the suffix of chunks j+1 .. L-1 applied to F_{n+1}
    T Fin[6];
    {
      const SE3<T> gn = shfl_se3<T, false>(gs, 1);
      T Gn[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) Gn[k] = shfl_dn_w(G[k], 1);
      if (j + 1 < L) {
        T AF[6];
        bwd_step(gn.R, gn.p0, gn.p1, gn.p2, bnd.Ftip, Gn, AF);
#pragma unroll
        for (int k = 0; k < 6; ++k) Fin[k] = AF[k];
      } else {
#pragma unroll
        for (int k = 0; k < 6; ++k) Fin[k] = bnd.Ftip[k];      // f_{n,n+1} = I (A5)
      }
    }
    // ---------------- pass B: Eq. (2) from the true wrench; tau_i = S_i^T F_i
    {
      T Gd[6];
      chunk_backward<T, PR>(Ls, PRs, q, B, b, w, NL, s0, cnt, Fin, tau, valid, Gd);
    }
  }
}

template <typename T, int L, bool PR>
static cudaError_t launch_chunk_l(int n, const LinkDHc<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                                  const T* qd, const T* qdd, T* tau, cudaStream_t st, const unsigned char* prism,
                                  T* ws, int64_t grid) {
  const int c = (n + L - 1) / L;
  const size_t smem = (size_t)n * sizeof(LinkDHc<T>) + (PR ? (size_t)n : 0);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(rnea_chunk_kernel<T, L, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  rnea_chunk_kernel<T, L, PR><<<(unsigned)grid, kChunkThreads, smem, st>>>(n, c, L_dev, bnd, B, q, qd, qdd, tau,
                                                                           prism, ws);
  return cudaGetLastError();
}

int chunk_default_lanes(int n) {
  // smallest L with chunks of at most 16 links (the per-lane serial depth)
  int L = 2;
  while (L < 32 && (n + L - 1) / L > 16) L <<= 1;
  return L;
}

int64_t chunk_grid(int64_t B, int lanes) {
  const int64_t spb = kChunkThreads / lanes;                 // states per CTA per round
  const int64_t want = (B + spb - 1) / spb;
  const int64_t cap = (int64_t)num_sms() * kChunkMinBlocks;
  return want < cap ? want : cap;
}

size_t chunk_ws_elems(int n, int64_t B, int lanes) {
  const int c = (n + lanes - 1) / lanes;
  return (size_t)chunk_grid(B, lanes) * kChunkThreads * c * kChunkPerLink;
}

template <typename T>
cudaError_t launch_rnea_chunk(int n, int lanes, const LinkDHc<T>* L_dev, const Boundary<T>& bnd, int64_t B,
                              const T* q, const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                              const unsigned char* prism, T* ws) {
  const int64_t grid = chunk_grid(B, lanes);
  ++*launches;
#define RD_CHUNK_CASE(LL)                                                                                  \
  case LL:                                                                                                 \
    return prism ? launch_chunk_l<T, LL, true>(n, L_dev, bnd, B, q, qd, qdd, tau, st, prism, ws, grid)    \
                 : launch_chunk_l<T, LL, false>(n, L_dev, bnd, B, q, qd, qdd, tau, st, nullptr, ws, grid);
  switch (lanes) {
    RD_CHUNK_CASE(2)
    RD_CHUNK_CASE(4)
    RD_CHUNK_CASE(8)
    RD_CHUNK_CASE(16)
    RD_CHUNK_CASE(32)
    default: return cudaErrorInvalidValue;
  }
#undef RD_CHUNK_CASE
}

template cudaError_t launch_rnea_chunk<double>(int, int, const LinkDHc<double>*, const Boundary<double>&, int64_t,
                                               const double*, const double*, const double*, double*, cudaStream_t,
                                               int*, const unsigned char*, double*);
template cudaError_t launch_rnea_chunk<float>(int, int, const LinkDHc<float>*, const Boundary<float>&, int64_t,
                                              const float*, const float*, const float*, float*, cudaStream_t, int*,
                                              const unsigned char*, float*);

}  // namespace rd
