/*
 * rd.h -- C ABI of librd.so: batched rigid-body dynamics of an n-link serial
 * chain on NVIDIA B200 (sm_100a), after arXiv 1609.04493 (PAPER.md, cited P:n).
 *
 * The library evaluates, for B independent states,
 *   inverse dynamics  tau  = ID(q, qd, qdd, V_0, Vdot_0, F_{n+1})   Eq. (3)
 *                     by the RNEA forward/backward recursions of Eq. (1)-(2)
 *                     (P:60-78), i.e. the two scans of Alg. 1;
 *   forward dynamics  qdd  = FD(q, qd, tau, V_0, Vdot_0, F_{n+1})   Eq. (4)
 *                     by the articulated-body algorithm, Eq. (7)-(8)
 *                     and Alg. 3, or by JSIIA, Eq. (6), (17), Alg. 2.
 *
 * Conventions (A1-A3): twists (v, w) linear first; wrenches (f, m);
 * f_{i-1,i} = M_i exp([S_i] q_i) maps link-i coordinates to link-(i-1)
 * coordinates; S_i and J_i are given in the link-i frame; gravity g
 * enters as Vdot_0 = (-g, 0) (A3); V_0 = 0 and F_{n+1} = 0 unless set with
 * rd_model_set_boundary.
 *
 * Memory: batch arrays are structure-of-arrays, link-major: x[i*batch + b] for
 * link i (0-based) and state b; `lda` variants are not provided.  Device
 * pointers must be naturally aligned (8 B fp64, 4 B fp32) device memory of the
 * current CUDA device (checked: RD_E_ARG otherwise); outputs must not alias inputs.  The caller owns every I/O buffer; the model
 * owns its constants and any workspace.
 *
 * Errors: every call returns rd_status_t; RD_OK == 0.  rd_last_error() returns
 * a thread-local message for the last failing call on the calling thread.  No
 * C++ exception crosses the ABI.  Kernel launches are asynchronous on `stream`
 * (a cudaStream_t; NULL = legacy default stream) and the call returns after
 * enqueue; a launch failure returns RD_E_CUDA.  batch == 0 is a no-op (RD_OK).
 * Per-state numerical failure in FD (Omega_i = S_i^T Jhat_i S_i <= 0, A11)
 * does not abort other states: that state's qdd is NaN.
 */
#ifndef RD_H_
#define RD_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rd_model_s* rd_model_t;

typedef enum {
  RD_OK = 0,
  RD_E_ARG = 1,          /* bad argument: n < 1, null/misaligned/aliased pointer, batch < 0 */
  RD_E_MODEL = 2,        /* invalid model: non-unit twist, non-rigid M, non-SPD/non-rigid J */
  RD_E_CUDA = 3,         /* CUDA error (no device, launch failure, ...) */
  RD_E_NOMEM = 4,        /* device or host allocation failed */
  RD_E_UNSUPPORTED = 5   /* valid request this build does not support */
} rd_status_t;

/* In-robot parallelisation strategy of the inverse-dynamics kernel (north_star (2)). */
/* THREAD, REVERSE and CHUNK run in Denavit-Hartenberg frames built from the model at
 * creation.  They apply to chains of revolute (zero pitch) and prismatic joints whose DH
 * origins lie within 50 link lengths of their joints; a model with screw joints, or with
 * nearly parallel consecutive axes (DH origin farther out: ill-conditioned DH maps,
 * DESIGN.md 8.5), runs on the joint-frame kernels instead (any joints): THREAD as the
 * joint-frame register kernel (fp64 n <= 8, fp32 n <= 12) or else REVERSE, REVERSE in
 * joint frames, CHUNK as GENERIC. */
typedef enum {
  RD_STRAT_AUTO = 0,      /* chosen per (n, dtype, batch) from the measured table */
  RD_STRAT_THREAD = 1,    /* one thread per state, serial recursion; revolute (zero pitch) and prismatic
                             joints.  Short chains (fp64 n <= 12, <= 16 up to 300k states; fp32 n <= 32
                             except 25, 26) keep
                             the whole per-link stash in registers (fully
                             unrolled register kernel); longer ones stash on chip (TMEM + shared memory),
                             n <= 30 fp64 / 32 fp32; otherwise falls back to REVERSE */
  RD_STRAT_WARP_SCAN = 2, /* one warp per state, lane = link, Kogge-Stone shuffle scans */
  RD_STRAT_GENERIC = 3,   /* one thread per state, any n, any joints, stash in a global workspace */
  RD_STRAT_REVERSE = 4,   /* one thread per state, any n, any joints (DH frames for revolute / prismatic
                             chains, joint frames otherwise), no stash: the backward sweep re-derives
                             V, Vdot by inverting the forward maps */
  RD_STRAT_BLOCK_SCAN = 5, /* one CTA per state, thread = link, CTA-wide scans: the single-robot latency
                              mode for long chains (n <= 512) */
  RD_STRAT_WARP_SCAN_EQ13 = 6, /* the paper's operators literally: warp per state, one Eq. (13) semigroup scan
                                  for V and Vdot (Eq. 12) and the Eq. (16) affine backward scan, body frame;
                                  n <= 32 */
  RD_STRAT_WARP_SCAN_EQ15 = 7, /* the synchronous Eq. (15) scan literally: warp per state, one scan of the
                                  28x28 operators on (Vdot, Q, V, Fhat, 1) (starred blocks: reading A6),
                                  then the Eq. (16) backward scan; n <= 32; slow (one warp per SM) */
  RD_STRAT_CHUNK = 8      /* L lanes per state (L = lanes_per_state of rd_model_set_strategy, a power of
                             two in [2, 32]; 0 = chosen from n), lane j runs the serial recursions over
                             a chunk of ceil(n/L) consecutive links and the L chunk results are combined
                             by log2(L)-round shuffle scans of the Eq. (13) semigroup (forward) and of
                             the Eq. (16) affine wrench maps (backward), at chunk granularity;
                             revolute (zero pitch) and prismatic joints, any n; screw joints: GENERIC */
} rd_strategy_t;

/* Forward-dynamics algorithm. */
typedef enum {
  RD_FD_ABA = 0,          /* articulated-body algorithm, Eq. (7)-(8), Alg. 3 (default); one thread per
                             state; revolute/prismatic chains of n <= 16 (fp64) / 20 (fp32) keep the per-link workspace in
                             registers, longer ones in a per-call global workspace */
  RD_FD_JSIIA = 1,        /* joint-space inertia inversion, Eq. (6)/(17), Alg. 2: n+1 IDs per state
                             (one per lane of a warp, n <= 31, or per thread of a CTA, n <= 256) +
                             Cholesky solve; n > 256 -> RD_E_UNSUPPORTED */
  RD_FD_ABA_SCAN = 2,     /* the paper's hybrid ABIA, Alg. 3, all on the GPU: tau_bias by the warp-scan
                             ID, serial ABI (Eq. 7) per state, then the Eq. (18) zhat and Eq. (19)
                             lambda scans across the links of a warp (n <= 32) or of a CTA
                             (32 < n <= 256, warp scans + a scan of the warp totals) */
  RD_FD_ABA_MERGED = 3    /* as RD_FD_ABA_SCAN, but tau_hat, zhat and chat come from ONE backward scan
                             of the merged Eq. (20) operators (Omega^{-1} reading A7,
                             seeding A8) over the n+1 lanes of a warp; n <= 31 */
} rd_fd_algo_t;

/* Library version string. */
const char* rd_version(void);

/* Thread-local message of the last failing call ("" if none). */
const char* rd_last_error(void);

/* Create a model (P:25-36 nomenclature).  All arrays are HOST memory, row-major:
 *   M[n][4][4]  home transform M_i = f_{i-1,i}(q_i = 0), frame i -> frame i-1;
 *               rotation block orthonormal with det +1 (tol 1e-9), last row 0 0 0 1;
 *   S[n][6]     joint twist S_i = (v, w) in the link-i frame: revolute/screw
 *               |w| = 1, or prismatic w = 0 and |v| = 1 (tol 1e-9);
 *   J[n][6][6]  spatial inertia J_i about the link-i origin, (v, w) ordering,
 *               rigid-body structure [[m I, -m[c]], [m[c], I_o]], symmetric (tol
 *               1e-9 relative), m > 0 and positive-definite rotational inertia about
 *               the centre of mass (the 6x6 is then SPD);
 *   gravity[3]  base-frame gravity, realised as Vdot_0 = (-g, 0) (A3).
 * On RD_E_MODEL the message lists every violation with its 1-based link index.
 * The model is immutable afterwards except through rd_model_set_*; it holds
 * device copies of the constants on the device current at creation.
 */
rd_status_t rd_model_create(int32_t n, const double* M, const double* S, const double* J,
                            const double gravity[3], rd_model_t* out);

rd_status_t rd_model_destroy(rd_model_t m);

/* Number of links n (-1 for a NULL model). */
int32_t rd_model_n(rd_model_t m);

/* CUDA device ordinal the model was created on (-1 for a NULL model); every
 * device pointer passed with this model must be memory of that device. */
int32_t rd_model_device(rd_model_t m);

/* Override the inverse-dynamics strategy (RD_STRAT_AUTO restores the table).
 * lanes_per_state: RD_STRAT_CHUNK only -- 0 (choose from n) or a power of two in
 * [2, 32]; must be 0 for every other strategy.  RD_E_ARG otherwise. */
rd_status_t rd_model_set_strategy(rd_model_t m, rd_strategy_t s, int32_t lanes_per_state);

/* Strategy the next rd_inverse_dynamics_* call on `batch` states will use. */
rd_strategy_t rd_model_resolve_strategy(rd_model_t m, int64_t batch, int32_t fp64);

/* Full boundary data of Eq. (3)/(4): base twist V_0, base acceleration
 * Vdot_0 (replaces the gravity-derived value; pass NULL to keep it) and tip
 * wrench F_{n+1} acting on link n, expressed in frame n (f_{n,n+1} = I, A5).
 * Host arrays of 6 doubles, NULL = zero (Vdot_0: NULL = keep gravity). */
rd_status_t rd_model_set_boundary(rd_model_t m, const double V0[6], const double Vdot0[6],
                                  const double Ftip[6]);

/* Inverse dynamics (Eq. 1-2) on DEVICE arrays [n][batch]; tau is written. */
rd_status_t rd_inverse_dynamics_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                    const double* qdd, double* tau, void* stream);
rd_status_t rd_inverse_dynamics_f32(rd_model_t m, int64_t batch, const float* q, const float* qd,
                                    const float* qdd, float* tau, void* stream);

/* Forward dynamics (Eq. 4) on DEVICE arrays [n][batch]; qdd is written.
 * Concurrency (ID and FD alike): a model may be used by several host threads and
 * streams at once.  Calls that need a workspace (GENERIC ID, every FD algorithm)
 * allocate it per call, stream-ordered, from the model's memory pool
 * (cudaMallocFromPoolAsync before the kernels, cudaFreeAsync after them on the
 * call's stream), so concurrent calls never share scratch memory and a call
 * captured in a CUDA graph owns its workspace in the graph.  The model's
 * constants are read-only after creation; rd_model_set_* must not race with
 * calls on the same model. */
rd_status_t rd_forward_dynamics_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                    const double* tau, double* qdd, void* stream);
rd_status_t rd_forward_dynamics_f32(rd_model_t m, int64_t batch, const float* q, const float* qd,
                                    const float* tau, float* qdd, void* stream);
rd_status_t rd_model_set_fd_algo(rd_model_t m, rd_fd_algo_t algo);

/* Forward dynamics with a per-state status array (NEXT-4, SURVEY §8(b) "Errors";
 * A11).  As rd_forward_dynamics_*, plus status: DEVICE int32[batch] (NULL =
 * none, same as the plain call), written for every state: 0 = all pivots
 * positive; k > 0 = the algorithm's pivot at 1-based link k was not positive
 * (ABA / ABA_SCAN / ABA_MERGED: the tip-most link with Omega_k = S_k^T Jhat_k S_k
 * <= 0 in the ABI sweep, Eq. 7; JSIIA: the first non-positive Cholesky pivot of
 * M(q)).  A failing state's qdd is NaN and other states are unaffected.
 * status must be 4-byte aligned device memory not overlapping qdd (RD_E_ARG). */
/* Per-state boundary data (NEXT-4; the full signature of Eq. (3)/(4), P:79-92,
 * with V_0, Vdot_0, F_{n+1} varying per state): V0, Vdot0 (base frame) and Ftip
 * (acting on link n, in the user's link-n frame; f_{n,n+1} = I, A5) are DEVICE
 * arrays of layout [6][batch], component-major (x[k*batch + b]); any of them
 * NULL = the model's value (gravity / rd_model_set_boundary).  Same alignment /
 * device / aliasing rules as the state arrays (RD_E_ARG).  ID runs on THREAD,
 * WARP_SCAN, GENERIC or REVERSE (AUTO picks among them; an explicit
 * WARP_SCAN_EQ13/EQ15 strategy -> RD_E_UNSUPPORTED); FD on ABA only (other FD
 * algorithms -> RD_E_UNSUPPORTED).  status as in rd_forward_dynamics_ex_*. */
rd_status_t rd_inverse_dynamics_bnd_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                        const double* qdd, const double* V0, const double* Vdot0,
                                        const double* Ftip, double* tau, void* stream);
rd_status_t rd_inverse_dynamics_bnd_f32(rd_model_t m, int64_t batch, const float* q, const float* qd,
                                        const float* qdd, const float* V0, const float* Vdot0,
                                        const float* Ftip, float* tau, void* stream);
rd_status_t rd_forward_dynamics_bnd_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                        const double* tau, const double* V0, const double* Vdot0,
                                        const double* Ftip, double* qdd, int32_t* status, void* stream);
rd_status_t rd_forward_dynamics_bnd_f32(rd_model_t m, int64_t batch, const float* q, const float* qd,
                                        const float* tau, const float* V0, const float* Vdot0,
                                        const float* Ftip, float* qdd, int32_t* status, void* stream);

rd_status_t rd_forward_dynamics_ex_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                       const double* tau, double* qdd, int32_t* status, void* stream);
rd_status_t rd_forward_dynamics_ex_f32(rd_model_t m, int64_t batch, const float* q, const float* qd,
                                       const float* tau, float* qdd, int32_t* status, void* stream);

/* End-to-end inverse dynamics on HOST arrays [n][batch] (pageable or pinned):
 * the library streams the batch through device buffers in chunks, overlapping
 * host->device copies, the kernel and device->host copies on its own streams,
 * and returns after tau is complete in host memory (synchronous).  The strategy
 * is resolved once for the whole batch (every chunk runs it), so the result is
 * bit-identical to rd_inverse_dynamics_f64 on the same batch.  Host calls on one
 * model are serialised internally (the staging buffers are per model). */
rd_status_t rd_inverse_dynamics_host_f64(rd_model_t m, int64_t batch, const double* q,
                                         const double* qd, const double* qdd, double* tau);
/* Forward dynamics on HOST float64 arrays [n][batch] (same pipeline and rules as
 * rd_inverse_dynamics_host_f64; the model's FD algorithm). */
rd_status_t rd_forward_dynamics_host_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                         const double* tau, double* qdd);

/* Number of kernel launches the last rd_* compute call on this thread enqueued. */
int32_t rd_last_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* RD_H_ */
