// rd_internal.h -- host/device shared declarations of librd (product path).
// No oracle code is included or linked here.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rd {

// Per-link constants in the JOINT frame of each link:
// the link frame is re-chosen so that S'_i = (beta e_z, alpha e_z), i.e. the
// joint axis is the local z axis through the origin.  f'_{i-1,i}(q) =
// (Rm, pm) * (Rz(alpha q), (0, 0, beta q)).  alpha = 1, beta = pitch for a
// revolute/screw joint; alpha = 0, beta = 1 for a prismatic joint.
// Spatial inertia J' = [[m I, -[h]], [[h], I]] with h = m c and I the
// rotational inertia about the (joint-frame) origin, I = {xx, yy, zz, xy, xz, yz}.
template <typename T>
struct LinkConst {
  T Rm[9];      // row-major
  T pm[3];
  T m;
  T h[3];
  T I[6];
  T alpha, beta;
};

// Per-link constants of the DH-frame kernels (thread, reverse, ABA-DH) in
// Denavit-Hartenberg (modified, Craig) frames:
// f_{i-1,i}(q) = Rx(alpha) Tx(a) Rz(theta) Tz(d), R = Rx(alpha) Rz(theta),
// p = (a, -sin(alpha) d, cos(alpha) d) = (p0, p1, p2).  Revolute joint:
// theta = th0 + q, d constant, S_i = (0, e_z).  Prismatic joint (flagged in a
// separate per-link mask so this struct keeps its 17 scalars -- one more costs
// the thread kernel 1.5 %): theta = th0, d = d0 + q, i.e.
// p = (p0, p1 - sa q, p2 + ca q), S_i = (e_z, 0).  Inertia as in LinkConst.
template <typename T>
struct LinkDH {
  T ca, sa;       // cos/sin alpha
  T a, d;         // DH translations: f = Rx(alpha) Tx(a) Rz(theta) Tz(d), p = (a, -sa d, ca d)
  T th0;          // joint angle offset
  T cth0, sth0;   // cos/sin th0 (fp32 uses the angle-addition form for accuracy at large |q|)
  T m;
  T h[3];
  T I[6];
};

// The thread and REVERSE kernels' per-link constants: the DH transform of LinkDH and the
// inertia about the centre of mass (for the Newton-Euler form of Fhat,
// rd_math.cuh bias_force_com): c = h / m, I_c = I - m (|c|^2 1 - c c^T).
template <typename T>
struct LinkDHc {
  T ca, sa;
  T a, d;
  T th0;
  T cth0, sth0;
  T m;
  T c[3];         // centre of mass in the DH frame
  T Ic[6];        // rotational inertia about the centre of mass (xx yy zz xy xz yz)
};

// Boundary data of Eq. (3) in the joint frames: V_0, Vdot_0 (base frame,
// unchanged) and F_{n+1} (expressed in link n's joint frame).
template <typename T>
struct Boundary {
  T V0[6], Vd0[6], Ftip[6];
};

// Per-state boundary data (NEXT-4, rd_*_dynamics_bnd_*): device arrays [6][B]
// (component-major, x[k*B + b]) in the USER's frames, or nullptr for the
// model's value; A0 maps a base-frame twist into the kernel's base frame
// (identity for joint frames, Ad_{D_0^-1} for DH frames), At a wrench in user
// frame n into the kernel's frame n (Ad_{T_n}^T).
template <typename T>
struct StateBoundary {
  const T* V0;
  const T* Vd0;
  const T* Ft;
  T A0[36];
  T At[36];
};
// Kernel argument type: the full struct for the per-state instantiation, an
// empty tag otherwise (so the model-boundary kernels keep their parameter list).
struct NoStateBoundary {};
template <typename T, bool SB> struct SBArg { typedef NoStateBoundary type; };
template <typename T> struct SBArg<T, true> { typedef StateBoundary<T> type; };

// Kernel-parameter image for the compile-time-N kernels (lives in the constant
// bank; every access has a compile-time offset so the DFMAs take it directly).
template <typename T, int N>
struct RneaParams {
  LinkConst<T> L[N];
  Boundary<T> bnd;
};

struct ModelHost;   // defined in capi.cu

enum Strategy { kAuto = 0, kThread = 1, kWarpScan = 2, kGeneric = 3 };

// Launchers (rnea_thread.cu / rnea_generic.cu / rnea_warp.cu / aba.cu).
// All return cudaGetLastError() after enqueue.  `launches` is incremented by
// the number of kernels enqueued.  FD launchers take an optional per-state
// status array (device int32[B], nullptr = none): 0, or the 1-based link of the
// failing pivot (Omega_i <= 0 in the ABI sweep, tip-most first; JSIIA: the first
// non-positive Cholesky pivot).
// prism_mask: bit i set = link i prismatic (DH kernels; n <= 32 here).
template <typename T>
cudaError_t launch_rnea_thread(int n, const LinkDHc<T>* L_host, const Boundary<T>& bnd,
                               int64_t B, const T* q, const T* qd, const T* qdd, T* tau,
                               cudaStream_t st, int* launches, bool* supported, uint32_t prism_mask = 0,
                               const StateBoundary<T>* sb = nullptr);
// Short chains (n <= 12 fp64 / 32 fp32): the register-resident, fully
// unrolled THREAD kernel (rnea_small.cu); launch_rnea_thread dispatches to it.
bool small_kernel_has_n(int n, bool fp64, int64_t batch);
template <typename T>
cudaError_t launch_rnea_small(int n, const LinkDHc<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                              const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                              uint32_t prism_mask, const StateBoundary<T>* sb = nullptr);
template <typename T>
cudaError_t launch_rnea_generic(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd,
                                int64_t B, const T* q, const T* qd, const T* qdd, T* tau,
                                T* ws, int64_t ws_slots, cudaStream_t st, int* launches,
                                const StateBoundary<T>* sb = nullptr);
// qdd == nullptr: qdd = 0; tau == nullptr: not stored; fhat != nullptr: the
// per-link bias wrench Fhat (joint frame) is stored as [n][6][B].
template <typename T>
cudaError_t launch_rnea_warp(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd,
                             int64_t B, const T* q, const T* qd, const T* qdd, T* tau,
                             cudaStream_t st, int* launches, bool* supported, T* fhat = nullptr,
                             const StateBoundary<T>* sb = nullptr);
template <typename T>
cudaError_t launch_aba(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd,
                       int64_t B, const T* q, const T* qd, const T* tau, T* qdd,
                       T* ws, int64_t ws_slots, cudaStream_t st, int* launches, int32_t* status,
                       const StateBoundary<T>* sb = nullptr);

template <typename T>
cudaError_t launch_rnea_warp13(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd,
                               int64_t B, const T* q, const T* qd, const T* qdd, T* tau,
                               cudaStream_t st, int* launches, bool* supported);
template <typename T>
cudaError_t launch_rnea_warp15(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd,
                               int64_t B, const T* q, const T* qd, const T* qdd, T* tau,
                               cudaStream_t st, int* launches, bool* supported);
template <typename T>
cudaError_t launch_rnea_block(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd,
                              int64_t B, const T* q, const T* qd, const T* qdd, T* tau,
                              cudaStream_t st, int* launches, bool* supported);
// prism: device uint8[n], 1 = prismatic link (nullptr: all revolute).
template <typename T>
cudaError_t launch_rnea_rev(int n, const LinkDHc<T>* L_dev, const Boundary<T>& bnd,
                            int64_t B, const T* q, const T* qd, const T* qdd, T* tau,
                            cudaStream_t st, int* launches, const unsigned char* prism = nullptr,
                            const StateBoundary<T>* sb = nullptr);
// The register-resident THREAD kernel in joint frames (rnea_small_jf.cu): any joints,
// short chains (fp64 n <= 8, fp32 n <= 12), for models without a (well-conditioned) DH form.
bool small_jf_has_n(int n, bool fp64);
template <typename T>
cudaError_t launch_rnea_small_jf(int n, const LinkConst<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                                 const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                                 const StateBoundary<T>* sb = nullptr);
// REVERSE in joint frames (rnea_rev_jf.cu): any joints (screw included), any n whose
// constants fit shared memory; for models without a (well-conditioned) DH form.
bool rev_jf_has_n(int n, bool fp64);
template <typename T>
cudaError_t launch_rnea_rev_jf(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd, int64_t B, const T* q,
                               const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                               const StateBoundary<T>* sb = nullptr);
// CHUNK (rnea_chunk.cu): `lanes` in {2, 4, 8, 16, 32} lanes per state; ws: device
// workspace of chunk_ws_elems(n, B, lanes) elements.
template <typename T>
cudaError_t launch_rnea_chunk(int n, int lanes, const LinkDHc<T>* L_dev, const Boundary<T>& bnd, int64_t B,
                              const T* q, const T* qd, const T* qdd, T* tau, cudaStream_t st, int* launches,
                              const unsigned char* prism, T* ws);
size_t chunk_ws_elems(int n, int64_t B, int lanes);
int chunk_default_lanes(int n);
template <typename T>
cudaError_t launch_aba_dh(int n, const LinkDH<T>* L_dev, const Boundary<T>& bnd,
                          int64_t B, const T* q, const T* qd, const T* tau, T* qdd,
                          T* ws, int64_t ws_slots, cudaStream_t st, int* launches, int32_t* status,
                          const unsigned char* prism = nullptr, const StateBoundary<T>* sb = nullptr);
template <typename T>
cudaError_t launch_fd_scan(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd,
                           int64_t B, const T* q, const T* qd, const T* tau, T* qdd, T* ws,
                           cudaStream_t st, int* launches, bool* supported, int32_t* status);
template <typename T>
cudaError_t launch_fd_merged(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd,
                             int64_t B, const T* q, const T* qd, const T* tau, T* qdd, T* ws,
                             cudaStream_t st, int* launches, bool* supported, int32_t* status);
size_t fd_scan_ws_elems(int n, int64_t B);     // workspace (elements) of either scan FD
template <typename T>
cudaError_t launch_jsiia(int n, const LinkConst<T>* L_dev, const Boundary<T>& bnd,
                         int64_t B, const T* q, const T* qd, const T* tau, T* qdd,
                         cudaStream_t st, int* launches, bool* supported, int32_t* status, T* ws);
size_t jsiia_ws_elems(int n, int64_t B);   // workspace of the CTA-wide JSIIA (n > 31), elements

// Workspace slots (threads) the generic / ABA kernels use: ws holds
// per-link doubles for each slot (see the .cu files for the layout).
int64_t generic_ws_slots(int64_t B);
int generic_ws_per_link();
int aba_ws_per_link();
// Short chains (n <= 16 fp64 / 20 fp32, DH frames): ABA with the per-link workspace in registers
// (aba_small.cuh); capi dispatches to it before launch_aba_dh.
bool aba_small_has_n(int n, bool fp64);
template <typename T>
cudaError_t launch_aba_small(int n, const LinkDH<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                             const T* qd, const T* tau, T* qdd, cudaStream_t st, int* launches, int32_t* status,
                             uint32_t prism_mask, const StateBoundary<T>* sb);

// The register ABA in joint frames (aba_small_jf.cu): any joints, fp64 n <= 8 / fp32 n <= 12.
bool aba_small_jf_has_n(int n, bool fp64);
template <typename T>
cudaError_t launch_aba_small_jf(int n, const LinkConst<T>* L_host, const Boundary<T>& bnd, int64_t B, const T* q,
                                const T* qd, const T* tau, T* qdd, cudaStream_t st, int* launches, int32_t* status,
                                const StateBoundary<T>* sb);

bool thread_kernel_has_n(int n, bool fp64);
int num_sms();

}  // namespace rd
