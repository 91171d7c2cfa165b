// rd_small.h -- configuration and entry of the register-resident THREAD kernel
// (rnea_small.cuh; instantiated per link count in rnea_small_f64.cu,
// rnea_small_f32a.cu, rnea_small_f32b.cu so the build compiles them in parallel).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "rd_internal.h"

namespace rd {

// Longest chain per precision (the stash kernel takes longer ones).  fp64 chains of
// 9..12 links re-derive (sin, cos) in the backward sweep (small_recompute) and then
// beat the stash kernel at every batch (n = 12, 1e6 states: 141.8 vs 148.7 us,
// profiles/r02/ab_small_recompute_f64.csv); fp32 every n <= 32 but the spill cliff.
template <typename T>
constexpr int small_max_n() { return sizeof(T) == 8 ? 16 : 32; }
// fp64: every batch size up to this n; 13..16 only up to kSmallCapBatch states (n = 13:
// 7.1 vs 14.2 us at 2e4 states, 16.9 vs 26.2 at 1e5, but 174 vs 163 us at 1e6 for
// the stash kernel; profiles/r02/ab_small_f64_13_16.csv)
constexpr int kSmallMaxN64Any = 12;
// fp32 lengths where ptxas' allocation of the 255-register kernel falls off a
// spill cliff (n = 25 / 26, 1e6 states: 317 / 367 us vs 191 us at n = 27;
// profiles/r02/ab_small_f32_pack.csv): the stash kernel runs them.
constexpr bool small_f32_cliff(int n) { return n == 25 || n == 26; }
constexpr int kSmallThreads = 128;
// fp64, 6 <= N <= 12: left alone ptxas hoists every load and sincos and takes
// ~190-255 registers (2 CTAs of 128 per SM); a register cap buys warps for ~100-400 B
// of spills.  Measured (graph replay; bench.py's cold-L2 timing for C2):
//   N = 6:      uncapped to 300k states, then 3 CTAs/SM (1e6: 62.0 vs 71.5 us at 4);
//   N = 7..12:  4 CTAs/SM at every batch (1e6: n = 7 75.8 -> 69.3 us, n = 9 111.3 ->
//               89.0; C2 cold 17.7 -> 16.2 us; 1e5 warm within 2 %).
// profiles/r02/ab_small_cap.csv, ab_small_cap_c2_cold.txt.
constexpr int64_t kSmallCapBatch = 300000;
template <typename T, int N>
constexpr bool small_has_cap() { return sizeof(T) == 8 && N >= 6 && N <= 12; }
template <typename T, int N>
constexpr int small_cap_mb() { return N == 6 ? 3 : 4; }
template <typename T, int N>
constexpr int64_t small_cap_from() { return N == 6 ? kSmallCapBatch : 0; }   // capped build above this batch

// One launch of the N-link kernel (explicitly instantiated in the per-precision TUs).
template <typename T, int N>
cudaError_t small_launch_n(const LinkDHc<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q, const T* qd,
                           const T* qdd, T* tau, cudaStream_t st, uint32_t prism, const StateBoundary<T>* sb);

}  // namespace rd
