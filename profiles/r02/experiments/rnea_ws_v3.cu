// rnea_ws.cu -- warp-specialised THREAD kernel: serial RNEA per state (Eq. 1-2,
// P:60-78; the forward and backward scans of Alg. 1, as one forward
// and one backward sweep per state), fp64, revolute DH chains, even n <= 32.
//
// Why: the ping-pong thread kernel runs both
// sweeps in one thread and needs ~250 registers, so only 8 warps fit per SM
// and the FP64 pipe idles on dependency waits (57 % busy).  Here each tile of
// 256 states is served by 8 warp PAIRS: in every step
//   * warp A (warps 8..15) runs the chain of Eq. (1) for link k of tile t --
//     sin/cos of theta_k, V_k = Ad_{f^-1} V_{k-1} + S qd_k, Vdot_k (lean DH
//     factors) -- and re-derives (sin, cos) of link n-1-k of tile t-1 for the
//     backward sweep (so the stash holds 6 scalars per link instead of 8);
//   * warp B (warps 0..7) takes (V_k, Vdot_k) from a shared-memory ring,
//     computes Fhat_k = J Vdot - ad^T_V J V (centre-of-mass form) into
//     the on-chip stash (Tensor Memory for the first `lt` links, shared memory
//     for the rest), and runs Eq. (2) for link n-1-k of tile t-1 from the stash:
//     F_i = Fhat_i + Ad^T_{f_{i,i+1}^{-1}} F_{i+1}, tau_i = S_i^T F_i.
// Each role holds one chain's registers (<= 128: 16 warps per SM, twice the
// ping-pong kernel's), the two roles are balanced (~80 / ~71 FP64 instructions
// per link) and meet only at a two-slot ring guarded by per-slot mbarriers.
// Steps run in pairs (slot 0, slot 1), so every ring / input-register slot is
// a compile-time choice (no register rotation); FP64 operands cannot come from
// the constant bank on sm_100a, so the link constants and the sin/cos
// coefficients are read as double2 pairs from shared memory (half the loads).
#include <cuda_runtime.h>
#include <cstdint>
#include "rd_internal.h"
#include "rd_math.cuh"

namespace rd {

namespace {

constexpr int kWsMaxN = 32;
constexpr int kPairs = 8;                 // warp pairs per CTA
constexpr int kTile = kPairs * 32;        // states per tile
constexpr int kCols = 12;                 // TMEM columns per stashed link (6 doubles)
constexpr int kLtCap = 20;                // links in TMEM per state (even; 2 B warps share a lane quarter: 256 cols)
constexpr int kKC = 8;                    // double2 per link in the shared constant table
constexpr int kRingV2 = 7;                // double2 per state per ring slot: V (3), Vdot (3), (sin, cos) (1)

struct WsParams {
  LinkDHc<double> L[kWsMaxN];
  Boundary<double> bnd;
  int n;
  int lt;         // stash slots in TMEM (the rest in shared memory)
};

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(b), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n WS_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WS_WAIT_%=;\n}\n" :: "r"(b), "r"(parity) : "memory");
}

// 6 doubles <-> 12 TMEM columns of this thread's lane (32x32b shape, x8 + x4).
__device__ __forceinline__ void tm_st6(uint32_t a, const double* v) {
  uint32_t r[12];
#pragma unroll
  for (int k = 0; k < 6; ++k) { r[2 * k] = __double2loint(v[k]); r[2 * k + 1] = __double2hiint(v[k]); }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n"
               :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n"
               :: "r"(a + 8u), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]));
}
__device__ __forceinline__ void tm_ld6(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(a));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]) : "r"(a + 8u));
}
__device__ __forceinline__ void tm_wait_ld(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]));
}
__device__ __forceinline__ void tm_unpack6(const uint32_t* r, double* v) {
#pragma unroll
  for (int k = 0; k < 6; ++k) v[k] = __hiloint2double(r[2 * k + 1], r[2 * k]);
}

// sin/cos of NX angles (1 or 2) with the coefficients of rd_math.cuh's rd_sincos
// (same operations in the same order: identical results) read once from the
// shared table T[8] = (shifter, 2/pi) (pi/2 hi, lo) (S6, S5) (S4, S3) (S2, S1)
// (C6, C5) (C4, C3) (C2, C1) and shared by both angles.
template <int NX>
__device__ __forceinline__ void sincos_tab(const double2* T, const double* x, double* s, double* c) {
  const double2 t0 = T[0], t1 = T[1];
  double k[NX], r[NX], z[NX], ps[NX], pc[NX];
  int quad[NX];
#pragma unroll
  for (int j = 0; j < NX; ++j) {
    const double t = fma(x[j], t0.y, t0.x);
    quad[j] = __double2loint(t);
    k[j] = t - t0.x;
    r[j] = fma(-k[j], t1.x, x[j]);
    r[j] = fma(-k[j], t1.y, r[j]);
    z[j] = r[j] * r[j];
  }
  const double2 s65 = T[2], s43 = T[3], s21 = T[4], c65 = T[5], c43 = T[6], c21 = T[7];
#pragma unroll
  for (int j = 0; j < NX; ++j) {
    ps[j] = fma(z[j], s65.x, s65.y);
    pc[j] = fma(z[j], c65.x, c65.y);
    ps[j] = fma(z[j], ps[j], s43.x);
    pc[j] = fma(z[j], pc[j], c43.x);
    ps[j] = fma(z[j], ps[j], s43.y);
    pc[j] = fma(z[j], pc[j], c43.y);
    ps[j] = fma(z[j], ps[j], s21.x);
    pc[j] = fma(z[j], pc[j], c21.x);
    ps[j] = fma(z[j], ps[j], s21.y);
    pc[j] = fma(z[j], pc[j], c21.y);
    const double sn = fma(z[j] * r[j], ps[j], r[j]);
    const double cs = fma(z[j] * z[j], pc[j], fma(-0.5, z[j], 1.0));
    const bool swap = quad[j] & 1;
    const double a = swap ? cs : sn;
    const double b = swap ? sn : cs;
    const unsigned sa = ((unsigned)quad[j] & 2u) << 30, sb = ((unsigned)(quad[j] + 1) & 2u) << 30;
    s[j] = __hiloint2double(__double2hiint(a) ^ (int)sa, __double2loint(a));
    c[j] = __hiloint2double(__double2hiint(b) ^ (int)sb, __double2loint(b));
  }
}

struct Shared {
  double2 kc[kWsMaxN][kKC];   // per link: (ca, sa) (a, d) (th0, m) (c0, c1) (c2, Ic0) (Ic1, Ic2) (Ic3, Ic4) (Ic5, 0)
  double2 sct[8];             // sin/cos table (sincos_tab)
  uint64_t full[kPairs][2], empty[kPairs][2];
  uint32_t tmem_slot;
};

// ---------------------------------------------------------------- role A
// Inputs of step k+2 are loaded at step k into the register slot step k just
// consumed (two slots, one per step parity): the forward stream reads q, qd,
// qdd of link k+2 of tile t (pointers pf*, advancing by +B), the backward
// stream q of link n-3-k of tile t-1 (pb, by -B); before the last two steps of
// a tile both move on (next tile's links 0, 1; this tile's links n-1, n-2).
struct AIn { double q, qd, qa, qb; };
struct AState {
  double V[6], Vd[6];
  double sn, cs, sb, cb;        // sin/cos of this step's forward link and backward link (computed a step ahead)
  AIn in[2];
  const double *pfq, *pfqd, *pfqa, *pbq;
};

// sin/cos of step (kn) from the inputs `nx`: forward link kn, backward link n-1-kn.
__device__ __forceinline__ void a_sincos_next(const Shared& sh, int n, int kn, const AIn& nx, double* sc, double* cc) {
  const double x[2] = {nx.q + sh.kc[kn][2].x, nx.qb + sh.kc[n - 1 - kn][2].x};
  sincos_tab<2>(sh.sct, x, sc, cc);
}

// Step k (input slot S); kn = the next step's link (k + 1, or 0 after the last link).
// The next step's sin/cos chains run in this step's basic block beside the
// Ad chains of this one (they depend only on inputs loaded a step earlier).
template <bool DoF, bool DoB, int S>
__device__ __forceinline__ void a_step(AState& s, const Shared& sh, int64_t B, int n, int k, int kn, double2* ring,
                                       uint32_t full, uint32_t empty, uint32_t phase) {
  double nsc[2], ncc[2];
  a_sincos_next(sh, n, kn, s.in[S ^ 1], nsc, ncc);
  const AIn cur = s.in[S];
  s.in[S].q = __ldg(s.pfq); s.in[S].qd = __ldg(s.pfqd); s.in[S].qa = __ldg(s.pfqa); s.in[S].qb = __ldg(s.pbq);
  s.pfq += B; s.pfqd += B; s.pfqa += B; s.pbq -= B;
  double Vn[6], Vdn[6];
  if (DoF) {
    const double2 k0 = sh.kc[k][0], k1 = sh.kc[k][1];
    dh_ad_finv(k0.x, k0.y, k1.x, k1.y, s.sn, s.cs, s.V, Vn);
    dh_ad_finv(k0.x, k0.y, k1.x, k1.y, s.sn, s.cs, s.Vd, Vdn);
    Vn[5] += cur.qd;
    Vdn[5] += cur.qa;
    Vdn[0] = fma(cur.qd, Vn[1], Vdn[0]);
    Vdn[1] = fma(-cur.qd, Vn[0], Vdn[1]);
    Vdn[3] = fma(cur.qd, Vn[4], Vdn[3]);
    Vdn[4] = fma(-cur.qd, Vn[3], Vdn[4]);
  }
  // hand (V_k, Vdot_k) and (sin, cos) of backward link n-1-k to the partner warp
  double2* slot = ring + S * kRingV2 * kTile;
  mbar_wait(empty + 8u * S, phase ^ 1u);
  if (DoF) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      slot[j * kTile] = make_double2(Vn[2 * j], Vn[2 * j + 1]);
      slot[(3 + j) * kTile] = make_double2(Vdn[2 * j], Vdn[2 * j + 1]);
    }
  }
  if (DoB) slot[6 * kTile] = make_double2(s.sb, s.cb);
  mbar_arrive(full + 8u * S);
  if (DoF) {
#pragma unroll
    for (int j = 0; j < 6; ++j) { s.V[j] = Vn[j]; s.Vd[j] = Vdn[j]; }
  }
  s.sn = nsc[0]; s.cs = ncc[0]; s.sb = nsc[1]; s.cb = ncc[1];
}

// One tile: the step pairs, then the last two steps with the input streams
// moved on (next tile's links 0, 1; this tile's links n-1, n-2).  At tile
// start the next tile's inputs are prefetched into L2 (one bulk prefetch per
// link row and array; lane j takes link j), so the two-step register loads hit L2.
template <bool DoF, bool DoB>
__device__ __forceinline__ void a_tile(AState& s, const Shared& sh, int64_t B, int n, double2* ring, uint32_t full,
                                       uint32_t empty, uint32_t& phase, const double* q, const double* qd,
                                       const double* qdd, int64_t bnc, int64_t bfc, int64_t bn2) {
  const int lane = threadIdx.x & 31;
  if (lane < n && bn2 >= 0 && (B & 1) == 0) {                  // 16-byte aligned rows only
    const int64_t off = (int64_t)lane * B + bn2;
    const uint32_t bytes = 32 * sizeof(double);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" :: "l"(q + off), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" :: "l"(qd + off), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" :: "l"(qdd + off), "r"(bytes) : "memory");
  }
  for (int k = 0; k < n - 2; k += 2) {
    a_step<DoF, DoB, 0>(s, sh, B, n, k, k + 1, ring, full, empty, phase);
    a_step<DoF, DoB, 1>(s, sh, B, n, k + 1, k + 2, ring, full, empty, phase);
    phase ^= 1u;
  }
  s.pfq = q + bnc; s.pfqd = qd + bnc; s.pfqa = qdd + bnc;     // next tile, links 0, 1
  s.pbq = q + (int64_t)(n - 1) * B + bfc;                      // this tile, links n-1, n-2
  a_step<DoF, DoB, 0>(s, sh, B, n, n - 2, n - 1, ring, full, empty, phase);
  a_step<DoF, DoB, 1>(s, sh, B, n, n - 1, 0, ring, full, empty, phase);
  phase ^= 1u;
}

// ---------------------------------------------------------------- role B
struct BState {
  double F[6];
  double ca, sa, a, d, s, c;   // DH constants and (sin, cos) of the child link i+1 (identity at the tip, A5)
  double tp;                   // tau of the previous backward link, stored one step later
  int ip;                      // its link (-1: none)
};

// One B step: ring slot S -> (V, Vdot, sin/cos); backward link i = n-1-k of
// the old tile from stash `cur`; Fhat of link k of the new tile -> `st`.
template <bool DoF, bool DoB, int S>
__device__ __forceinline__ void b_step(BState& g, const Shared& sh, int64_t B, int n, int k, const double* cur,
                                       double* st, const double2* ring, uint32_t full, uint32_t empty,
                                       uint32_t phase, double* __restrict__ tau, int64_t bb, bool vb) {
  const double2* slot = ring + S * kRingV2 * kTile;
  mbar_wait(full + 8u * S, phase);
  double V[6], Vd[6];
  double2 sc = make_double2(0.0, 1.0);
  if (DoF) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double2 x = slot[j * kTile], y = slot[(3 + j) * kTile];
      V[2 * j] = x.x; V[2 * j + 1] = x.y; Vd[2 * j] = y.x; Vd[2 * j + 1] = y.y;
    }
  }
  if (DoB) sc = slot[6 * kTile];
  mbar_arrive(empty + 8u * S);
  if (DoB) {
    if (vb && g.ip >= 0) tau[(int64_t)g.ip * B + bb] = g.tp;
    const int i = n - 1 - k;
    double Fo[6];
    dh_bwd(g.ca, g.sa, g.a, g.d, g.s, g.c, g.F, cur, Fo);
#pragma unroll
    for (int j = 0; j < 6; ++j) g.F[j] = Fo[j];
    g.tp = Fo[5];
    g.ip = i;
    const double2 c0 = sh.kc[i][0], c1 = sh.kc[i][1];
    g.ca = c0.x; g.sa = c0.y; g.a = c1.x; g.d = c1.y;
    g.s = sc.x; g.c = sc.y;
  }
  if (DoF) {
    const double2* K = sh.kc[k];
    const double2 m2 = K[2], c01 = K[3], c2I0 = K[4], I12 = K[5], I34 = K[6], I5 = K[7];
    LinkDHc<double> C;
    C.m = m2.y; C.c[0] = c01.x; C.c[1] = c01.y; C.c[2] = c2I0.x;
    C.Ic[0] = c2I0.y; C.Ic[1] = I12.x; C.Ic[2] = I12.y; C.Ic[3] = I34.x; C.Ic[4] = I34.y; C.Ic[5] = I5.x;
    bias_force_com(C, V, Vd, st);
  }
}

}  // namespace

__global__ void __launch_bounds__(2 * kTile, 1)
rnea_ws_kernel(const __grid_constant__ WsParams P, int64_t B, const double* __restrict__ q,
               const double* __restrict__ qd, const double* __restrict__ qdd, double* __restrict__ tau) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Shared sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool role_b = warp < kPairs;
  const int pair = role_b ? warp : warp - kPairs;
  const int tt = pair * 32 + lane;                         // state within the tile
  const int n = P.n, lt = P.lt;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(su32(&sh.tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x < 2 * kPairs * 2) {
    const int p = threadIdx.x >> 2, r = threadIdx.x & 1;
    mbar_init(su32((threadIdx.x & 2) ? &sh.empty[p][r] : &sh.full[p][r]), 32);
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const LinkDHc<double>& C = P.L[i];
    sh.kc[i][0] = make_double2(C.ca, C.sa);
    sh.kc[i][1] = make_double2(C.a, C.d);
    sh.kc[i][2] = make_double2(C.th0, C.m);
    sh.kc[i][3] = make_double2(C.c[0], C.c[1]);
    sh.kc[i][4] = make_double2(C.c[2], C.Ic[0]);
    sh.kc[i][5] = make_double2(C.Ic[1], C.Ic[2]);
    sh.kc[i][6] = make_double2(C.Ic[3], C.Ic[4]);
    sh.kc[i][7] = make_double2(C.Ic[5], 0.0);
  }
  if (threadIdx.x == 0) {
    sh.sct[0] = make_double2(kSinCosD[0], kSinCosD[1]);
    sh.sct[1] = make_double2(kSinCosD[2], kSinCosD[3]);
    sh.sct[2] = make_double2(kSinCosD[4], kSinCosD[5]);
    sh.sct[3] = make_double2(kSinCosD[6], kSinCosD[7]);
    sh.sct[4] = make_double2(kSinCosD[8], kSinCosD[9]);
    sh.sct[5] = make_double2(kSinCosD[10], kSinCosD[11]);
    sh.sct[6] = make_double2(kSinCosD[12], kSinCosD[13]);
    sh.sct[7] = make_double2(kSinCosD[14], kSinCosD[15]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int64_t ntiles = (B + kTile - 1) / kTile;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t stride = (int64_t)gridDim.x * kTile;
  double2* vstash = reinterpret_cast<double2*>(smem_raw);            // [slot - lt][3][kTile]
  double2* ring = vstash + (size_t)(n - lt) * 3 * kTile + tt;        // [2][7][kTile], this state's column
  const uint32_t full = su32(&sh.full[pair][0]), empty = su32(&sh.empty[pair][0]);
  uint32_t phase = 0;

  if (!role_b) {
    // ------------------------------------------------------------ A warps
    AState s;
    for (int64_t it = 0; it <= my_tiles; ++it) {
      const int64_t bf = (int64_t)blockIdx.x * kTile + it * stride + tt;      // tile it
      const int64_t bfc = min(bf, B - 1), bnc = min(bf + stride, B - 1);     // its / the next tile's column
      const int64_t w0 = bf + stride - (threadIdx.x & 31);                   // next tile: this warp's first state
      const int64_t bn2 = w0 + 32 <= B ? w0 : -1;                            // (full warps only)
#pragma unroll
      for (int j = 0; j < 6; ++j) { s.V[j] = P.bnd.V0[j]; s.Vd[j] = P.bnd.Vd0[j]; }
      if (it == 0) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          s.in[j].q = __ldg(q + (int64_t)j * B + bfc);
          s.in[j].qd = __ldg(qd + (int64_t)j * B + bfc);
          s.in[j].qa = __ldg(qdd + (int64_t)j * B + bfc);
          s.in[j].qb = 0.0;
        }
        s.pfq = q + 2 * B + bfc; s.pfqd = qd + 2 * B + bfc; s.pfqa = qdd + 2 * B + bfc;
        s.pbq = q + (int64_t)(n - 3) * B + bfc;                                // (tile -1: unused)
        double sc[2], cc[2];
        a_sincos_next(sh, n, 0, s.in[0], sc, cc);
        s.sn = sc[0]; s.cs = cc[0]; s.sb = sc[1]; s.cb = cc[1];
        a_tile<true, false>(s, sh, B, n, ring, full, empty, phase, q, qd, qdd, bnc, bfc, bn2);
      } else if (it == my_tiles) {
        a_tile<false, true>(s, sh, B, n, ring, full, empty, phase, q, qd, qdd, bnc, bfc, bn2);
      } else {
        a_tile<true, true>(s, sh, B, n, ring, full, empty, phase, q, qd, qdd, bnc, bfc, bn2);
      }
    }
  } else {
    // ------------------------------------------------------------ B warps (own the stash)
    const uint32_t tbase = sh.tmem_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 256);
    double2* vs = vstash + tt;
    auto sm_put = [&](int slot, const double* v) {
      double2* d = vs + (size_t)(slot - lt) * 3 * kTile;
#pragma unroll
      for (int j = 0; j < 3; ++j) d[j * kTile] = make_double2(v[2 * j], v[2 * j + 1]);
    };
    auto sm_get = [&](int slot, double* v) {
      const double2* d = vs + (size_t)(slot - lt) * 3 * kTile;
#pragma unroll
      for (int j = 0; j < 3; ++j) { const double2 x = d[j * kTile]; v[2 * j] = x.x; v[2 * j + 1] = x.y; }
    };
    BState g;
    g.ip = -1;
    g.tp = 0.0;
    for (int64_t it = 0; it <= my_tiles; ++it) {
      const int64_t bb = (int64_t)blockIdx.x * kTile + (it - 1) * stride + tt;   // tile it-1 (backward)
      const bool vb = it > 0 && bb < B;
      const int bpar = (int)((it - 1) & 1);                                       // it = 0: 1 (slot = link)
#pragma unroll
      for (int j = 0; j < 6; ++j) g.F[j] = P.bnd.Ftip[j];
      g.ca = 1; g.sa = 0; g.a = 0; g.d = 0; g.s = 0; g.c = 1;                   // f_{n,n+1} = I (A5)
      g.ip = -1;
      if (it == 0) {
        for (int k = 0; k < n; k += 2) {
          double st[6];
          b_step<true, false, 0>(g, sh, B, n, k, nullptr, st, ring, full, empty, phase, tau, bb, vb);
          if (k < lt) tm_st6(tbase + (uint32_t)(k * kCols), st);
          else sm_put(k, st);
          b_step<true, false, 1>(g, sh, B, n, k + 1, nullptr, st, ring, full, empty, phase, tau, bb, vb);
          if (k + 1 < lt) tm_st6(tbase + (uint32_t)((k + 1) * kCols), st);
          else sm_put(k + 1, st);
          phase ^= 1u;
        }
      } else if (it == my_tiles) {
        auto get = [&](int slot, double* cur) {
          if (slot < lt) {
            uint32_t r[12];
            tm_ld6(tbase + (uint32_t)(slot * kCols), r);
            tm_wait_ld(r);
            tm_unpack6(r, cur);
          } else {
            sm_get(slot, cur);
          }
        };
        for (int k = 0; k < n; k += 2) {
          double cur[6];
          get(bpar ? k : n - 1 - k, cur);
          b_step<false, true, 0>(g, sh, B, n, k, cur, nullptr, ring, full, empty, phase, tau, bb, vb);
          get(bpar ? k + 1 : n - 2 - k, cur);
          b_step<false, true, 1>(g, sh, B, n, k + 1, cur, nullptr, ring, full, empty, phase, tau, bb, vb);
          phase ^= 1u;
        }
      } else {
        auto smem_seg = [&](int k0, int k1) {
          for (int k = k0; k < k1; k += 2) {
            double cur[6], st[6];
            const int s0 = bpar ? k : n - 1 - k, s1 = bpar ? k + 1 : n - 2 - k;
            sm_get(s0, cur);
            b_step<true, true, 0>(g, sh, B, n, k, cur, st, ring, full, empty, phase, tau, bb, vb);
            sm_put(s0, st);
            sm_get(s1, cur);
            b_step<true, true, 1>(g, sh, B, n, k + 1, cur, st, ring, full, empty, phase, tau, bb, vb);
            sm_put(s1, st);
            phase ^= 1u;
          }
        };
        auto tmem_seg = [&](int k0, int k1) {
          if (k0 >= k1) return;
          uint32_t r[12];
          tm_ld6(tbase + (uint32_t)((bpar ? k0 : n - 1 - k0) * kCols), r);
          for (int k = k0; k < k1; k += 2) {
            double cur[6], st[6];
            const int s0 = bpar ? k : n - 1 - k, s1 = bpar ? k + 1 : n - 2 - k;
            const int k2 = min(k + 2, k1 - 1);
            const int s2 = bpar ? k2 : n - 1 - k2;
            tm_wait_ld(r);
            tm_unpack6(r, cur);
            tm_ld6(tbase + (uint32_t)(s1 * kCols), r);              // next step's slot, in flight
            b_step<true, true, 0>(g, sh, B, n, k, cur, st, ring, full, empty, phase, tau, bb, vb);
            tm_st6(tbase + (uint32_t)(s0 * kCols), st);
            tm_wait_ld(r);
            tm_unpack6(r, cur);
            tm_ld6(tbase + (uint32_t)(s2 * kCols), r);
            b_step<true, true, 1>(g, sh, B, n, k + 1, cur, st, ring, full, empty, phase, tau, bb, vb);
            tm_st6(tbase + (uint32_t)(s1 * kCols), st);
            phase ^= 1u;
          }
          tm_wait_ld(r);
        };
        if (bpar) {
          tmem_seg(0, lt);
          smem_seg(lt, n);
        } else {
          smem_seg(0, n - lt);
          tmem_seg(n - lt, n);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      if (vb && g.ip >= 0) tau[(int64_t)g.ip * B + bb] = g.tp;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(sh.tmem_slot));
}

bool ws_kernel_has_n(int n) { return n >= 4 && n <= kWsMaxN && (n % 2) == 0; }

static size_t ws_smem_bytes(int n) {
  const int lt = n < kLtCap ? n : kLtCap;
  return (size_t)(n - lt) * 3 * kTile * sizeof(double2) + (size_t)2 * kRingV2 * kTile * sizeof(double2);
}

cudaError_t launch_rnea_ws(int n, const LinkDHc<double>* L_host, const Boundary<double>& bnd, int64_t B,
                           const double* q, const double* qd, const double* qdd, double* tau, cudaStream_t st,
                           int* launches) {
  if (!ws_kernel_has_n(n)) return cudaErrorInvalidValue;
  WsParams P;
  for (int i = 0; i < n; ++i) P.L[i] = L_host[i];
  P.bnd = bnd;
  P.n = n;
  P.lt = n < kLtCap ? n : kLtCap;
  const size_t smem = ws_smem_bytes(n);
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(rnea_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)ws_smem_bytes(kWsMaxN));
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  const int64_t ntiles = (B + kTile - 1) / kTile;
  const int64_t grid = ntiles < num_sms() ? ntiles : num_sms();
  ++*launches;
  rnea_ws_kernel<<<(unsigned)grid, 2 * kTile, smem, st>>>(P, B, q, qd, qdd, tau);
  return cudaGetLastError();
}

}  // namespace rd
