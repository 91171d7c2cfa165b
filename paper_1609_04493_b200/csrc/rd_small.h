// rd_small.h -- configuration and entry of the register-resident THREAD kernel
// (rnea_small.cuh; instantiated per link count in rnea_small_f64.cu,
// rnea_small_f32a.cu, rnea_small_f32b.cu so the build compiles them in parallel).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "rd_internal.h"

namespace rd {

#ifndef SMALL_MAX_F32
#define SMALL_MAX_F32 32
#endif
// Longest chain per precision (the stash kernel takes longer ones).  fp64 chains of
// 9..12 links re-derive (sin, cos) in the backward sweep (small_recompute) and then
// beat the stash kernel at every batch (n = 12, 1e6 states: 141.8 vs 148.7 us,
// profiles/r02/ab_small_recompute_f64.csv); fp32 every n <= 32 but the spill cliff.
#ifndef SMALL_MAX_F64
#define SMALL_MAX_F64 12
#endif
template <typename T>
constexpr int small_max_n() { return sizeof(T) == 8 ? SMALL_MAX_F64 : SMALL_MAX_F32; }
constexpr int kSmallMaxN64Any = SMALL_MAX_F64;   // fp64: every batch size up to this n
// fp32 lengths where ptxas' allocation of the 255-register kernel falls off a
// spill cliff (n = 25 / 26, 1e6 states: 317 / 367 us vs 191 us at n = 27;
// profiles/r02/ab_small_f32_pack.csv): the stash kernel runs them.
constexpr bool small_f32_cliff(int n) { return n == 25 || n == 26; }
constexpr int kSmallThreads = 128;
// fp64, N >= 6: left alone ptxas hoists every load and sincos and takes ~220
// registers at N = 7-8 (2 CTAs of 128 per SM, no spills); capped at 168 (3 CTAs)
// it spills ~150 B.  Measured (graph replay, n = 7): B = 1e5 8.8 us uncapped vs
// 9.5 us capped; B = 1e6 96 vs 85 us -- the cap pays once there are many waves,
// so both are built and the launch picks by batch (kSmallCapBatch).
#ifndef SMALL_CAP_BATCH
#define SMALL_CAP_BATCH 300000
#endif
#ifndef SMALL_CAP_MB
#define SMALL_CAP_MB 3
#endif
constexpr int64_t kSmallCapBatch = SMALL_CAP_BATCH;
constexpr int kSmallCapMB = SMALL_CAP_MB;      // resident CTAs per SM of the capped build
template <typename T, int N>
constexpr bool small_has_cap() { return sizeof(T) == 8 && N >= 6; }

// One launch of the N-link kernel (explicitly instantiated in the per-precision TUs).
template <typename T, int N>
cudaError_t small_launch_n(const LinkDHc<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q, const T* qd,
                           const T* qdd, T* tau, cudaStream_t st, uint32_t prism, const StateBoundary<T>* sb);

}  // namespace rd
