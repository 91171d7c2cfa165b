// rnea_thread.cu -- one thread per state, serial RNEA (Eq. 1-2; the two
// scans of Alg. 1, run as one forward and one backward sweep per
// state), for n <= 32 links.
//
// Design:
//  * one persistent CTA per SM, W warps (W = 8 or 16), looping over tiles of
//    32*W states; one thread per state;
//  * the per-link stash the backward sweep needs, (sin q, cos q, Fhat) = 8
//    scalars, lives ON CHIP: the first `lt` links in Tensor Memory (tcgen05.st /
//    tcgen05.ld, 32x32b shape: warp w owns TMEM lanes 32(w%4).., and columns
//    [(w/4) * 2048/W, ...)), the remaining n - lt links in shared memory laid
//    out [link][8/VW][thread] of 16-byte vectors (conflict-free);
//  * ping-pong: the backward sweep of tile t-1 and the forward sweep of tile t
//    share each loop step and the stash slots (below);
//  * model constants are a __grid_constant__ kernel parameter indexed by the
//    (warp-uniform) link counter: uniform constant-bank loads;
//  * inputs q, qd, qdd are read coalesced (x[i*B + b]) kPD links ahead of use
//    (streaming across the tile boundary), the step loops unrolled by a divisor
//    of kPD (StepCfg); tau is written coalesced one backward step late;
//  * the link loops stay rolled (besides that unroll): the whole kernel stays in
//    the instruction cache (a fully unrolled n = 30 body thrashed it, profiles/r01);
//  * instantiations: precision x W x prismatic joints (PR) x per-state boundary (SB).
#include <cuda_runtime.h>
#include <type_traits>
#include <cstdint>
#include <cstdlib>
#include <atomic>
#include "rd_internal.h"
#include "rd_math.cuh"
#include "rd_f32x2.cuh"

namespace rd {

constexpr int kMaxThreadN = 32;

template <typename T>
struct ThreadParams {
  LinkDHc<T> L[kMaxThreadN];   // DH transform + inertia about the CoM
  Boundary<T> bnd;
  int n;          // links
  int lt;         // links stashed in TMEM (the rest in shared memory)
  uint32_t prism; // bit k: link k is prismatic (PR instantiation only)
};

// ------------------------------------------------------------------ TMEM helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tmem_alloc_512(uint32_t* slot_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(smem_u32(slot_smem)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
__device__ __forceinline__ void tmem_dealloc_512(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// 8 scalars of type T <-> 16 (fp64) or 8 (fp32) 32-bit TMEM columns of this thread's lane.
template <typename T> struct TmemIO;

template <> struct TmemIO<double> {
  static constexpr int kCols = 16;
  typedef uint32_t Regs[16];
  __device__ static __forceinline__ void st(uint32_t a, const double* v) {
    uint32_t r[16];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      r[2 * k] = __double2loint(v[k]);
      r[2 * k + 1] = __double2hiint(v[k]);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};\n"
        :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
           "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
  }
  __device__ static __forceinline__ void ld(uint32_t a, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(a));
  }
  // Completes outstanding tcgen05.ld; "+r" orders every use of r after the wait.
  __device__ static __forceinline__ void wait(uint32_t* r) {
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]));
  }
  __device__ static __forceinline__ void unpack(const uint32_t* r, double* v) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __hiloint2double(r[2 * k + 1], r[2 * k]);
  }
};

template <> struct TmemIO<float> {
  static constexpr int kCols = 8;
  typedef uint32_t Regs[8];
  __device__ static __forceinline__ void st(uint32_t a, const float* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n"
                 :: "r"(a), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                    "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                    "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])));
  }
  __device__ static __forceinline__ void ld(uint32_t a, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(a));
  }
  __device__ static __forceinline__ void wait(uint32_t* r) {
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]));
  }
  __device__ static __forceinline__ void unpack(const uint32_t* r, float* v) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(r[k]);
  }
};

// ------------------------------------------------------------------ ping-pong kernel
// Same arithmetic, but the backward sweep of tile t-1 and the forward sweep of
// tile t run in the SAME loop (step k: backward of link n-1-k, forward of link
// k): two independent dependency chains per thread, i.e. twice the ILP, at no
// extra stash.  Tile parity alternates the link->slot map (slot(j) = j for even
// tiles, n-1-j for odd ones) so that at step k both sweeps touch the same slot:
// the backward read of the old tile's link frees exactly the slot the forward
// write of the new tile needs.  Every steady-state
// step is ONE basic block (no branch between the two sweeps), so ptxas can
// interleave them; the slot kind (TMEM or shared) is fixed per loop segment.
// Input prefetch distance (links, in stream order over tiles) and unroll factor
// of the steady-state step loops, per precision.  Unrolling by a divisor of the
// distance lets ptxas keep the in-flight loads in fixed registers instead of
// rotating them with MOVs that wait on the loads at every loop head (ncu: those
// MOVs and the back-edge carried ~20 % long-scoreboard stalls).  Measured on
// B200: fp64 n = 30 (W = 8), 1M states 0.543 -> 0.494 ms with
// (8, 4); fp32 n = 30 (W = 16) 0.312 -> 0.309 ms with (4, 2); the 16-warp fp64
// plan (n <= 15, 128-register cap) also (4, 2): n = 15, 1M 0.227 -> 0.222 ms.
// kFwdFirst: issue the forward link before the backward one in a step (fp32 -3 %,
// fp64 +5 %, measured).
template <typename T, int W> struct StepCfg {       // fp64, W = 16 (n <= 15, 128 registers)
  static constexpr int kPD = 4, kUnroll = 2;
  static constexpr bool kFwdFirst = false;
};
template <> struct StepCfg<double, 8> {
  static constexpr int kPD = 8, kUnroll = 4;
  static constexpr bool kFwdFirst = false;
};
template <> struct StepCfg<float, 8> {
  static constexpr int kPD = 4, kUnroll = 2;
  static constexpr bool kFwdFirst = true;
};
template <> struct StepCfg<float, 16> {
  static constexpr int kPD = 4, kUnroll = 2;
  static constexpr bool kFwdFirst = true;
};

template <typename T, int PD>
struct FwdState {
  T V[6], Vd[6];                        // fp64
  float2 VV[6];                         // fp32: (V_k, Vdot_k) packed for FFMA2 (f32x2)
  static constexpr int kPD = PD;
  T a_q[kPD], a_qd[kPD], a_qa[kPD];    // inputs of the next kPD links in stream order ([0] = current)
  const T *pq, *pqd, *pqa;              // this tile's column
  const T *xq, *xqd, *xqa;              // the next tile's column (prefetch across the tile boundary)
};
template <typename T>
struct BwdState {
  T F[6];                       // fp64
  float2 FF[3];                 // fp32: (f_k, m_k) packed for FFMA2
  T ca, sa, a, d, s, c;         // DH constants and stashed (sin, cos) of the child link i+1
  int64_t b;
  bool valid;
  T tp;                         // tau of the previous backward link, stored one step later
  int ip;                       // its link index (-1: none pending)
};

// fp32 runs the per-link algebra on packed pairs (FFMA2 / FMUL2, sm_100a f32x2):
// the forward Ad, the bias-wrench pieces and the sin/cos polynomials act on
// (V, Vdot) component pairs, the backward Ad^T on (f, m) pairs.  Same FP32 pipe
// rate as FFMA (measured, tools/ffma2_peak.cu) at half the issue slots; the fp32
// kernel is issue-bound.
template <typename T> constexpr bool kPacked = std::is_same<T, float>::value;
template <typename T, int PD>
__device__ __forceinline__ void fwd_unpack(FwdState<T, PD>& f) {
  if constexpr (kPacked<T>) {
#pragma unroll
    for (int k = 0; k < 6; ++k) { f.V[k] = f.VV[k].x; f.Vd[k] = f.VV[k].y; }
  }
}
template <typename T, int PD>
__device__ __forceinline__ void fwd_pack(FwdState<T, PD>& f) {
  if constexpr (kPacked<T>) {
#pragma unroll
    for (int k = 0; k < 6; ++k) f.VV[k] = make_float2(f.V[k], f.Vd[k]);
  }
}
template <typename T>
__device__ __forceinline__ void bwd_pack(BwdState<T>& g) {
  if constexpr (kPacked<T>) {
#pragma unroll
    for (int k = 0; k < 3; ++k) g.FF[k] = make_float2(g.F[k], g.F[k + 3]);
  }
}
// Inputs are consumed as ONE stream over (tile, link): the loads issued at link
// k fetch link k+2 of this tile, or link k+2-n of the NEXT tile, so the first
// links of a tile are already in registers when its forward sweep starts.
template <typename T, int PD>
__device__ __forceinline__ void fwd_init(FwdState<T, PD>& f, const ThreadParams<T>& P, int64_t B, int64_t bl,
                                         int64_t bl_next, const T* q, const T* qd, const T* qdd, bool first) {
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    if constexpr (kPacked<T>) f.VV[k] = make_float2(P.bnd.V0[k], P.bnd.Vd0[k]);
    else { f.V[k] = P.bnd.V0[k]; f.Vd[k] = P.bnd.Vd0[k]; }
  }
  f.pq = q + bl; f.pqd = qd + bl; f.pqa = qdd + bl;
  f.xq = q + bl_next; f.xqd = qd + bl_next; f.xqa = qdd + bl_next;
  if (first) {
#pragma unroll
    for (int j = 0; j < PD; ++j) {
      const bool here = j < P.n;
      const int64_t off = (int64_t)(here ? j : min(j - P.n, P.n - 1)) * B;   // n < kPD: reloaded per tile
      f.a_q[j] = __ldg((here ? f.pq : f.xq) + off);
      f.a_qd[j] = __ldg((here ? f.pqd : f.xqd) + off);
      f.a_qa[j] = __ldg((here ? f.pqa : f.xqa) + off);
    }
  }
}
template <typename T>
__device__ __forceinline__ void bwd_flush(BwdState<T>& g, int64_t B, T* __restrict__ tau) {
  if (g.valid && g.ip >= 0) tau[(int64_t)g.ip * B + g.b] = g.tp;
  g.ip = -1;
}
template <typename T>
__device__ __forceinline__ void bwd_init(BwdState<T>& g, const ThreadParams<T>& P) {
  g.ip = -1;
#pragma unroll
  for (int k = 0; k < 6; ++k) g.F[k] = P.bnd.Ftip[k];
  if constexpr (kPacked<T>) {
#pragma unroll
    for (int k = 0; k < 3; ++k) g.FF[k] = make_float2(P.bnd.Ftip[k], P.bnd.Ftip[k + 3]);
  }
  g.ca = 1; g.sa = 0; g.a = g.d = 0; g.s = 0; g.c = 1;   // f_{n,n+1} = I (A5)
}
// forward link k: V_k, Vdot_k, Fhat_k -> st[8]
template <bool PR, typename T, int PD>
__device__ __forceinline__ void fwd_link(FwdState<T, PD>& f, const ThreadParams<T>& P, int64_t B, int k, T* st) {
  const int n = P.n;
  // this link's inputs (loaded two links earlier) and the loads for link k+2
  // (stream order over tiles).  (A variant that prefetched into L1 and loaded in
  // place was 20 % slower.)
  const T cq = f.a_q[0], cqd = f.a_qd[0], cqa = f.a_qa[0];
  constexpr int kPD = PD;
  const int k2 = k + kPD;
  const bool here = k2 < n;
  const int64_t off2 = (int64_t)(here ? k2 : min(k2 - n, n - 1)) * B;   // n < kPD: reloaded per tile
  const T f_q = __ldg((here ? f.pq : f.xq) + off2);
  const T f_qd = __ldg((here ? f.pqd : f.xqd) + off2);
  const T f_qa = __ldg((here ? f.pqa : f.xqa) + off2);
  const LinkDHc<T>& C = P.L[k];
  // PR (the model has prismatic joints): link type from C.pr (warp-uniform), selects only.
  const bool prism = PR && ((P.prism >> k) & 1u);
  const T qang = prism ? T(0) : cq;               // revolute: theta = th0 + q; prismatic: th0
  T s, c;
  if constexpr (sizeof(T) == 8) {
    rd_sincos(qang + C.th0, &s, &c);          // fp64: rounding of q + th0 is ~ulp(q)
  } else {
    T s0, c0;                                     // fp32: sin/cos(q) then add th0 exactly
    sincos_mufu(qang, &s0, &c0);                 // SFU (n = 25 / 26, 1e6: -2.6 % vs the polynomial pair)
    s = fma(s0, C.cth0, c0 * C.sth0);
    c = fma(c0, C.cth0, -(s0 * C.sth0));
  }
  // Eq. (1): V = Ad_{f^-1} V + S qd, Vd = Ad_{f^-1} Vd + S qdd + ad_V(S qd),
  // S = (0, e_z) (revolute) or (e_z, 0) (prismatic, d = d0 + q)
  if constexpr (kPacked<T>) {
    float2 VVn[6];
    const float dl = PR && prism ? C.d + cq : C.d;
    dh_ad_finv_x2(C.ca, C.sa, C.a, dl, s, c, f.VV, VVn);
    const float sr = prism ? 0.f : cqd, sp = prism ? cqd : 0.f;
    const float ar = prism ? 0.f : cqa, ap = prism ? cqa : 0.f;
    VVn[5].x += sr; VVn[5].y += ar;                 // lane adds: no pair to assemble
    if (PR) { VVn[2].x += sp; VVn[2].y += ap; }
    // ad_V (sp e_z, sr e_z) into the Vdot lanes
    VVn[0].y = fmaf(sr, VVn[1].x, PR ? fmaf(sp, VVn[4].x, VVn[0].y) : VVn[0].y);
    VVn[1].y = fmaf(-sr, VVn[0].x, PR ? fmaf(-sp, VVn[3].x, VVn[1].y) : VVn[1].y);
    VVn[3].y = fmaf(sr, VVn[4].x, VVn[3].y);
    VVn[4].y = fmaf(-sr, VVn[3].x, VVn[4].y);
    st[0] = (PR && prism) ? cq : s;
    st[1] = c;
    bias_force_com_x2(C, VVn, st + 2);
#pragma unroll
    for (int j = 0; j < 6; ++j) f.VV[j] = VVn[j];
  } else {
  T Vn[6], Vdn[6];
  if (PR) {
    const T dq = prism ? cq : T(0);
    const T dl = C.d + dq;
    dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, f.V, Vn);
    dh_ad_finv(C.ca, C.sa, C.a, dl, s, c, f.Vd, Vdn);
    const T sr = prism ? T(0) : cqd, sp = prism ? cqd : T(0);
    const T ar = prism ? T(0) : cqa, ap = prism ? cqa : T(0);
    Vn[5] += sr;
    Vn[2] += sp;
    Vdn[5] += ar;
    Vdn[2] += ap;
    // ad_V (sp e_z, sr e_z) = (sp w x e_z + sr v x e_z, sr w x e_z)
    Vdn[0] = fma(sr, Vn[1], fma(sp, Vn[4], Vdn[0]));
    Vdn[1] = fma(-sr, Vn[0], fma(-sp, Vn[3], Vdn[1]));
    Vdn[3] = fma(sr, Vn[4], Vdn[3]);
    Vdn[4] = fma(-sr, Vn[3], Vdn[4]);
    st[0] = prism ? cq : s;                         // prismatic: (s, c) are constants, keep q
  } else {
    dh_ad_finv(C, s, c, f.V, Vn);
    dh_ad_finv(C, s, c, f.Vd, Vdn);
    Vn[5] += cqd;
    Vdn[5] += cqa;
    Vdn[0] = fma(cqd, Vn[1], Vdn[0]);
    Vdn[1] = fma(-cqd, Vn[0], Vdn[1]);
    Vdn[3] = fma(cqd, Vn[4], Vdn[3]);
    Vdn[4] = fma(-cqd, Vn[3], Vdn[4]);
    st[0] = s;
  }
  st[1] = c;
  bias_force_com(C, Vn, Vdn, st + 2);
#pragma unroll
  for (int j = 0; j < 6; ++j) { f.V[j] = Vn[j]; f.Vd[j] = Vdn[j]; }
  }
#pragma unroll
  for (int j = 0; j + 1 < kPD; ++j) { f.a_q[j] = f.a_q[j + 1]; f.a_qd[j] = f.a_qd[j + 1]; f.a_qa[j] = f.a_qa[j + 1]; }
  f.a_q[kPD - 1] = f_q; f.a_qd[kPD - 1] = f_qd; f.a_qa[kPD - 1] = f_qa;
}
// backward link i from its stash cur[8]: F_i, tau_i, then (R, p) of link i for link i-1
template <bool PR, typename T>
__device__ __forceinline__ void bwd_link(BwdState<T>& g, const ThreadParams<T>& P, int64_t B, int i,
                                         const T* cur, T* __restrict__ tau) {
  T Fo[6];
  // the previous link's tau, whose DFMA chain finished a whole step ago (storing
  // it right after the chain stalled the warp on the fixed-latency dependency)
  if (g.valid && g.ip >= 0) tau[(int64_t)g.ip * B + g.b] = g.tp;
  const LinkDHc<T>& C = P.L[i];
  const bool prism = PR && ((P.prism >> i) & 1u);
  T ti;                                            // tau_i = S_i^T F_i
  if constexpr (kPacked<T>) {
    dh_bwd_x2(g.ca, g.sa, g.a, g.d, g.s, g.c, g.FF, cur + 2);
    ti = prism ? g.FF[2].x : g.FF[2].y;
  } else {
    dh_bwd(g.ca, g.sa, g.a, g.d, g.s, g.c, g.F, cur + 2, Fo);
#pragma unroll
    for (int j = 0; j < 6; ++j) g.F[j] = Fo[j];
    ti = prism ? g.F[2] : g.F[5];
  }
  g.tp = ti;
  g.ip = i;
  g.ca = C.ca; g.sa = C.sa; g.a = C.a;
  if (PR) {
    g.d = prism ? C.d + cur[0] : C.d;               // prismatic: d = d0 + q
    g.s = prism ? C.sth0 : cur[0];
  } else {
    g.d = C.d;
    g.s = cur[0];
  }
  g.c = cur[1];
}

template <typename T, int W, bool PR, bool SB>
__global__ void __launch_bounds__(W * 32, 1)
rnea_thread_pp_kernel(const __grid_constant__ ThreadParams<T> P, int64_t B,
                      const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ qdd,
                      T* __restrict__ tau, const __grid_constant__ typename SBArg<T, SB>::type sb) {
  constexpr int NT = W * 32;
  constexpr int kColsPerWarp = 2048 / W;
  constexpr int KC = TmemIO<T>::kCols;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5;
  const int tid = threadIdx.x;
  if (warp == 0) tmem_alloc_512(&tmem_slot);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tbase = tmem_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * kColsPerWarp);
  const int n = P.n, lt = P.lt;
  const int64_t ntiles = (B + NT - 1) / NT;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // 16-byte vectors: [slot - lt][8 / VW][NT] of (double2 | float4) -- conflict-free
  // (consecutive threads 16 B apart), 2 (fp32) / 4 (fp64) shared-memory
  // instructions per slot instead of 8 (the fp32 kernel is issue-bound)
  using V16 = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
  constexpr int VW = 16 / sizeof(T), NV = 8 / VW;
  V16* vstash = reinterpret_cast<V16*>(smem_raw);
  auto vptr = [&](int slot) { return vstash + (size_t)(slot - lt) * NV * NT + tid; };
  auto put_smem = [&](int slot, const T* st) {
    V16* d = vptr(slot);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      V16 v;
      T* e = reinterpret_cast<T*>(&v);
#pragma unroll
      for (int j = 0; j < VW; ++j) e[j] = st[k * VW + j];
      d[k * NT] = v;
    }
  };
  auto get_smem = [&](int slot, T* cur) {
    const V16* d = vptr(slot);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const V16 v = d[k * NT];
      const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (int j = 0; j < VW; ++j) cur[k * VW + j] = e[j];
    }
  };
  auto put_any = [&](int slot, const T* st) {
    if (slot < lt) TmemIO<T>::st(tbase + (uint32_t)(slot * KC), st);
    else put_smem(slot, st);
  };
  auto get_any = [&](int slot, T* cur) {
    if (slot < lt) {
      typename TmemIO<T>::Regs r;
      TmemIO<T>::ld(tbase + (uint32_t)(slot * KC), r);
      TmemIO<T>::wait(r);
      TmemIO<T>::unpack(r, cur);
    } else {
      get_smem(slot, cur);
    }
  };

  using Cfg = StepCfg<T, W>;
  FwdState<T, Cfg::kPD> f;
  BwdState<T> g;
  g.b = 0;
  g.valid = false;
  g.ip = -1;
  for (int64_t it = 0; it <= my_tiles; ++it) {
    const int64_t b = (blockIdx.x + it * gridDim.x) * NT + tid;
    const bool fvalid = b < B;
    if (it == my_tiles) {
      if (it == 0) break;
      // epilogue: backward of the last tile alone (slot parity of tile it-1)
      const int bpar = (int)((it - 1) & 1);
      bwd_init(g, P);
      if constexpr (SB) {                            // per-state F_{n+1} of tile it-1 (NEXT-4)
        if (sb.Ft) { sb_vec(sb.Ft, sb.At, B, min(g.b, B - 1), g.F); bwd_pack(g); }
      }
      for (int i = n - 1; i >= 0; --i) {
        T cur[8];
        get_any(bpar ? n - 1 - i : i, cur);
        bwd_link<PR>(g, P, B, i, cur, tau);
      }
      bwd_flush(g, B, tau);
      break;
    }
    const int64_t bn = b + (int64_t)gridDim.x * NT;
    fwd_init(f, P, B, fvalid ? b : (B - 1), bn < B ? bn : (B - 1), q, qd, qdd, it == 0 || P.n < Cfg::kPD);
    if constexpr (SB) {                              // per-state V_0, Vdot_0 (NEXT-4)
      if (sb.V0 || sb.Vd0) {
        fwd_unpack(f);
        if (sb.V0) sb_vec(sb.V0, sb.A0, B, fvalid ? b : (B - 1), f.V);
        if (sb.Vd0) sb_vec(sb.Vd0, sb.A0, B, fvalid ? b : (B - 1), f.Vd);
        fwd_pack(f);
      }
    }
    if (it == 0) {
      // prologue: forward of the first tile alone (parity 0: slot = link)
      for (int k = 0; k < n; ++k) {
        T st[8];
        fwd_link<PR>(f, P, B, k, st);
        put_any(k, st);
      }
    } else {
      // steady state: backward of tile it-1 (parity bpar) + forward of tile it (parity !bpar);
      // at step k both use slot s_k = bpar ? k : n-1-k.
      bwd_init(g, P);
      if constexpr (SB) {                            // per-state F_{n+1} of tile it-1 (NEXT-4)
        if (sb.Ft) { sb_vec(sb.Ft, sb.At, B, min(g.b, B - 1), g.F); bwd_pack(g); }
      }
      const int bpar = (int)((it - 1) & 1);
      auto smem_step = [&](int k) {
        const int slot = bpar ? k : n - 1 - k;
        T cur[8], st[8];
        get_smem(slot, cur);
        if constexpr (Cfg::kFwdFirst) {                 // order of the two chains in the step
          fwd_link<PR>(f, P, B, k, st);
          bwd_link<PR>(g, P, B, n - 1 - k, cur, tau);
        } else {
          bwd_link<PR>(g, P, B, n - 1 - k, cur, tau);
          fwd_link<PR>(f, P, B, k, st);
        }
        put_smem(slot, st);
      };
      auto tmem_seg = [&](int k0, int k1) {
        if (k0 >= k1) return;
        typename TmemIO<T>::Regs r;
        TmemIO<T>::ld(tbase + (uint32_t)((bpar ? k0 : n - 1 - k0) * KC), r);
#pragma unroll (Cfg::kUnroll)
        for (int k = k0; k < k1; ++k) {
          const int slot = bpar ? k : n - 1 - k;
          const int knx = min(k + 1, k1 - 1);
          const int slot_nx = bpar ? knx : n - 1 - knx;
          TmemIO<T>::wait(r);
          T cur[8], st[8];
          TmemIO<T>::unpack(r, cur);
          TmemIO<T>::ld(tbase + (uint32_t)(slot_nx * KC), r);       // next step's slot, in flight
          if constexpr (Cfg::kFwdFirst) {                 // order of the two chains in the step
            fwd_link<PR>(f, P, B, k, st);
            bwd_link<PR>(g, P, B, n - 1 - k, cur, tau);
          } else {
            bwd_link<PR>(g, P, B, n - 1 - k, cur, tau);
            fwd_link<PR>(f, P, B, k, st);
          }
          TmemIO<T>::st(tbase + (uint32_t)(slot * KC), st);
        }
        TmemIO<T>::wait(r);
      };
      if (bpar) {
        tmem_seg(0, lt);
#pragma unroll (Cfg::kUnroll)
        for (int k = lt; k < n; ++k) smem_step(k);
      } else {
#pragma unroll (Cfg::kUnroll)
        for (int k = 0; k < n - lt; ++k) smem_step(k);
        tmem_seg(n - lt, n);
      }
    }
    tmem_wait_st();
    bwd_flush(g, B, tau);
    g.b = b;
    g.valid = fvalid;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0) tmem_dealloc_512(tmem_slot);
}

// SM count of the current device, cached per device ordinal (thread-safe).
int num_sms() {
  constexpr int kMaxDev = 64;
  static std::atomic<int> cache[kMaxDev];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>* slot = (dev >= 0 && dev < kMaxDev) ? &cache[dev] : nullptr;
  int sms = slot ? slot->load(std::memory_order_relaxed) : 0;
  if (sms <= 0) {
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    if (slot) slot->store(sms, std::memory_order_relaxed);
  }
  return sms;
}

// Stash plan: the largest W in {16, 8} whose TMEM + shared-memory capacity
// holds n links.
struct StashPlan { int W, lt, ls; size_t smem; };
static constexpr size_t kSmemCap = 227 * 1024;
static constexpr size_t kSmemFloor = 120 * 1024;   // forces one CTA per SM (it owns all TMEM)

template <typename T>
static bool plan_for(int n, StashPlan* out) {
  for (int W : {16, 8}) {
    const int cols_per_warp = 2048 / W;
    const int lt_cap = cols_per_warp / TmemIO<T>::kCols;
    const int lt = n < lt_cap ? n : lt_cap;
    const int ls = n - lt;
    const size_t smem = (size_t)ls * 8 * sizeof(T) * W * 32;
    if (smem <= kSmemCap - 1024) {
      out->W = W; out->lt = lt; out->ls = ls;
      out->smem = smem < kSmemFloor ? kSmemFloor : smem;
      return true;
    }
  }
  return false;
}

bool thread_kernel_has_n(int n, bool fp64) {
  if (n < 1 || n > kMaxThreadN) return false;
  StashPlan p;
  return fp64 ? plan_for<double>(n, &p) : plan_for<float>(n, &p);
}

template <typename T, int W, bool PR, bool SB>
static cudaError_t launch_w(const ThreadParams<T>& P, size_t smem, int64_t B, const T* q, const T* qd,
                            const T* qdd, T* tau, cudaStream_t st, const typename SBArg<T, SB>::type& sb) {
  static thread_local int attr_dev = -1;          // the opt-in is per device; set it once
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(rnea_thread_pp_kernel<T, W, PR, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kSmemCap - 1024));
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  const int64_t ntiles = (B + W * 32 - 1) / (W * 32);
  const int64_t grid = ntiles < num_sms() ? ntiles : num_sms();
  rnea_thread_pp_kernel<T, W, PR, SB><<<(unsigned)grid, W * 32, smem, st>>>(P, B, q, qd, qdd, tau, sb);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_rnea_thread(int n, const LinkDHc<T>* L_host, const Boundary<T>& bnd, int64_t B,
                               const T* q, const T* qd, const T* qdd, T* tau, cudaStream_t st,
                               int* launches, bool* supported, uint32_t prism_mask, const StateBoundary<T>* sb) {
  if (small_kernel_has_n(n, sizeof(T) == 8, B)) {     // short chain: everything in registers
    *supported = true;
    return launch_rnea_small<T>(n, L_host, bnd, B, q, qd, qdd, tau, st, launches, prism_mask, sb);
  }
  StashPlan plan;
  *supported = n >= 1 && n <= kMaxThreadN && plan_for<T>(n, &plan);
  if (!*supported) return cudaSuccess;
  ThreadParams<T> P;
  for (int i = 0; i < n; ++i) P.L[i] = L_host[i];
  P.bnd = bnd;
  P.n = n;
  P.lt = plan.lt;
  ++*launches;
  P.prism = prism_mask;
  const NoStateBoundary nsb{};
  if (sb) {                                        // per-state boundary: the SB instantiations
    if (prism_mask != 0) {
      if (plan.W == 16) return launch_w<T, 16, true, true>(P, plan.smem, B, q, qd, qdd, tau, st, *sb);
      return launch_w<T, 8, true, true>(P, plan.smem, B, q, qd, qdd, tau, st, *sb);
    }
    if (plan.W == 16) return launch_w<T, 16, false, true>(P, plan.smem, B, q, qd, qdd, tau, st, *sb);
    return launch_w<T, 8, false, true>(P, plan.smem, B, q, qd, qdd, tau, st, *sb);
  }
  if (prism_mask != 0) {                           // any prismatic joint: the PR instantiation
    if (plan.W == 16) return launch_w<T, 16, true, false>(P, plan.smem, B, q, qd, qdd, tau, st, nsb);
    return launch_w<T, 8, true, false>(P, plan.smem, B, q, qd, qdd, tau, st, nsb);
  }
  if (plan.W == 16) return launch_w<T, 16, false, false>(P, plan.smem, B, q, qd, qdd, tau, st, nsb);
  return launch_w<T, 8, false, false>(P, plan.smem, B, q, qd, qdd, tau, st, nsb);
}

template cudaError_t launch_rnea_thread<double>(int, const LinkDHc<double>*, const Boundary<double>&, int64_t,
                                                const double*, const double*, const double*, double*,
                                                cudaStream_t, int*, bool*, uint32_t, const StateBoundary<double>*);
template cudaError_t launch_rnea_thread<float>(int, const LinkDHc<float>*, const Boundary<float>&, int64_t,
                                               const float*, const float*, const float*, float*,
                                               cudaStream_t, int*, bool*, uint32_t, const StateBoundary<float>*);

}  // namespace rd
