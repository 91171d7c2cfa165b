// capi.cu -- the C ABI of librd.so (include/rd.h): model validation, the
// joint-frame re-parameterisation, strategy dispatch, and the host-buffer
// (end-to-end) pipeline.  No torch types, no exceptions across the ABI.
#include <cuda_runtime.h>
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rd.h"
#include "rd_internal.h"

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;

rd_status_t fail(rd_status_t st, const std::string& msg) {
  g_err = msg;
  return st;
}

rd_status_t cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return RD_E_CUDA;
}

// ------------------------------------------------------------ small host algebra
typedef double Mat3[3][3];
typedef double Mat6[6][6];

void skew(const double* a, Mat3 K) {
  K[0][0] = 0; K[0][1] = -a[2]; K[0][2] = a[1];
  K[1][0] = a[2]; K[1][1] = 0; K[1][2] = -a[0];
  K[2][0] = -a[1]; K[2][1] = a[0]; K[2][2] = 0;
}

// Rigid transform (R, p) as 4x4 row-major.
struct Rigid { double R[3][3]; double p[3]; };

Rigid rigid_from4(const double* M) {
  Rigid g;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) g.R[i][j] = M[4 * i + j];
    g.p[i] = M[4 * i + 3];
  }
  return g;
}
Rigid rigid_mul(const Rigid& a, const Rigid& b) {
  Rigid c;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += a.R[i][k] * b.R[k][j];
      c.R[i][j] = s;
    }
    double t = a.p[i];
    for (int k = 0; k < 3; ++k) t += a.R[i][k] * b.p[k];
    c.p[i] = t;
  }
  return c;
}
Rigid rigid_inv(const Rigid& a) {
  Rigid c;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c.R[i][j] = a.R[j][i];
  for (int i = 0; i < 3; ++i) {
    double t = 0;
    for (int k = 0; k < 3; ++k) t -= a.R[k][i] * a.p[k];
    c.p[i] = t;
  }
  return c;
}
Rigid rigid_identity() {
  Rigid g;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) g.R[i][j] = (i == j);
    g.p[i] = 0;
  }
  return g;
}
// Ad_g for (v, w) twists: [[R, [p]R], [0, R]].
void adjoint(const Rigid& g, Mat6 A) {
  Mat3 P;
  skew(g.p, P);
  for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) A[i][j] = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      A[i][j] = g.R[i][j];
      A[3 + i][3 + j] = g.R[i][j];
      double s = 0;
      for (int k = 0; k < 3; ++k) s += P[i][k] * g.R[k][j];
      A[i][3 + j] = s;
    }
}

// Rotation whose third column is the unit vector a.
void frame_with_z(const double* a, double R[3][3]) {
  double e[3] = {0, 0, 0};
  int k = 0;
  for (int i = 1; i < 3; ++i)
    if (std::fabs(a[i]) < std::fabs(a[k])) k = i;
  e[k] = 1.0;
  double d = e[0] * a[0] + e[1] * a[1] + e[2] * a[2];
  double x[3] = {e[0] - d * a[0], e[1] - d * a[1], e[2] - d * a[2]};
  double nx = std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
  for (int i = 0; i < 3; ++i) x[i] /= nx;
  double y[3] = {a[1] * x[2] - a[2] * x[1], a[2] * x[0] - a[0] * x[2], a[0] * x[1] - a[1] * x[0]};
  for (int i = 0; i < 3; ++i) { R[i][0] = x[i]; R[i][1] = y[i]; R[i][2] = a[i]; }
}

bool cholesky6(const Mat6 A) {
  double L[6][6] = {};
  for (int j = 0; j < 6; ++j) {
    double d = A[j][j];
    for (int k = 0; k < j; ++k) d -= L[j][k] * L[j][k];
    if (!(d > 0)) return false;
    L[j][j] = std::sqrt(d);
    for (int i = j + 1; i < 6; ++i) {
      double s = A[i][j];
      for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
      L[i][j] = s / L[j][j];
    }
  }
  return true;
}

}  // namespace

// ------------------------------------------------------------------ the model
struct rd_model_s {
  int n = 0;
  int device = 0;
  bool all_revolute = false;       // every joint revolute with zero pitch
  rd_strategy_t strategy = RD_STRAT_AUTO;
  int chunk_lanes = 0;             // RD_STRAT_CHUNK: lanes per state (0 = from n)
  rd_fd_algo_t fd_algo = RD_FD_ABA;
  std::vector<rd::LinkConst<double>> L64;
  std::vector<rd::LinkConst<float>> L32;
  std::vector<Rigid> T;            // joint frame of link i expressed in the user's link-i frame
  bool dh_ok = false;              // DH frames built (every joint revolute with zero pitch, or prismatic)
  bool dh_eligible = false;        // no screw joints
  std::vector<unsigned char> prism;  // per link: 1 = prismatic
  bool has_prism = false;
  uint32_t prism_mask = 0;         // bit i = prism[i] (links < 32)
  unsigned char* dPrism = nullptr; // device copy of prism (REVERSE kernel)
  std::vector<rd::LinkDH<double>> D64;
  std::vector<rd::LinkDH<float>> D32;
  rd::LinkDH<double>* dD64 = nullptr;
  rd::LinkDH<float>* dD32 = nullptr;
  std::vector<rd::LinkDHc<double>> C64;   // thread kernel: the same frames, inertia about the CoM
  std::vector<rd::LinkDHc<float>> C32;
  rd::LinkDHc<double>* dC64 = nullptr;   // device copies (REVERSE kernel)
  rd::LinkDHc<float>* dC32 = nullptr;
  Rigid D0;                        // DH base frame in the user's base frame
  rd::Boundary<double> bdh64;
  rd::Boundary<float> bdh32;
  double gravity[3] = {0, 0, 0};
  double V0[6] = {0}, Vd0[6] = {0}, Ftip_user[6] = {0};
  rd::Boundary<double> b64;
  rd::Boundary<float> b32;
  double sbA0dh[36] = {0};         // per-state boundary: user base twist -> DH base frame
  double sbAt[36] = {0};           // per-state boundary: user frame-n wrench -> kernel frame n
  rd::LinkConst<double>* dL64 = nullptr;
  rd::LinkConst<float>* dL32 = nullptr;
  // Workspace of the GENERIC ID and the FD kernels: allocated PER CALL, stream-ordered
  // (cudaMallocFromPoolAsync before the launch, cudaFreeAsync after it, on the call's
  // stream) from this model's memory pool, which keeps freed blocks cached (release
  // threshold = max).  Concurrent calls on different streams therefore never share
  // a workspace, and a call captured in a CUDA graph gets graph-owned memory.
  cudaMemPool_t pool = nullptr;
  std::mutex pool_mu;
  // host-buffer pipeline (rd_*_host_f64): serialised by host_mu for the whole call
  void* hbuf[2] = {nullptr, nullptr};
  size_t hbuf_bytes = 0;
  cudaStream_t hstream[2] = {nullptr, nullptr};
  std::mutex host_mu;
};

namespace {

void rebuild_boundary(rd_model_t m) {
  // Base quantities are unchanged by the joint frames (T_0 = I); the tip wrench
  // is expressed in link n's joint frame: F' = Ad_{T_n}^T F (power pairing).
  Mat6 A;
  adjoint(m->T[m->n - 1], A);
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) m->sbAt[6 * j + i] = A[i][j];    // F' = A^T F
  double Ft[6];
  for (int j = 0; j < 6; ++j) {
    double s = 0;
    for (int i = 0; i < 6; ++i) s += A[i][j] * m->Ftip_user[i];
    Ft[j] = s;
  }
  for (int k = 0; k < 6; ++k) {
    m->b64.V0[k] = m->V0[k];
    m->b64.Vd0[k] = m->Vd0[k];
    m->b64.Ftip[k] = Ft[k];
    m->b32.V0[k] = (float)m->V0[k];
    m->b32.Vd0[k] = (float)m->Vd0[k];
    m->b32.Ftip[k] = (float)Ft[k];
  }
  if (m->dh_ok) {
    // DH base frame D0 is fixed to the base: V''_0 = Ad_{D0^-1} V_0 (same for Vdot_0);
    // the last DH frame equals link n's joint frame, so F_{n+1} is unchanged.
    Mat6 Ai;
    adjoint(rigid_inv(m->D0), Ai);
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) m->sbA0dh[6 * i + j] = Ai[i][j];
    for (int j = 0; j < 6; ++j) {
      double sv = 0, sa = 0;
      for (int k = 0; k < 6; ++k) { sv += Ai[j][k] * m->V0[k]; sa += Ai[j][k] * m->Vd0[k]; }
      m->bdh64.V0[j] = sv; m->bdh64.Vd0[j] = sa; m->bdh64.Ftip[j] = Ft[j];
      m->bdh32.V0[j] = (float)sv; m->bdh32.Vd0[j] = (float)sa; m->bdh32.Ftip[j] = (float)Ft[j];
    }
  }
}

// Modified-DH (Craig) frames for a chain of revolute (zero pitch) and prismatic
// joints, from the joint frames (a prismatic joint slides along z_i: d = d0 + q):
// joint frame i has z_i = the joint axis (Mp[i]: frame i in frame i-1).  Frame
// D_i keeps z_i and puts its origin/x-axis on the common normal of axes i and
// i+1 (any perpendicular for parallel axes; the joint frame itself for i = n);
// D_0 := D_1, so f''_{0,1} = Rz(q_1).  Then D_{i-1}^-1 D_i = Rx(alpha) Tx(a)
// Rz(th0) Tz(d) and the per-link parameters are read off that transform
// (verified to 1e-10; otherwise the THREAD strategy is not used).
bool build_dh(rd_model_t m, const std::vector<Rigid>& Mp, const std::vector<std::array<double, 36>>& Jp) {
  const int n = m->n;
  // Every DH frame is built LOCALLY, as its pose D[i] in joint frame i from the axes
  // of joints i and i+1 (joint frame i+1 in frame i is Mp[i+1]); then
  // D_{i-1}^-1 D_i = D[i-1]^-1 Mp[i] D[i].  Building them from the base-frame poses
  // G_i = Mp[0] ... Mp[i] instead carried the rounding of i products into every
  // relative transform: ~1e-13 (n = 30) to ~1e-10 (n = 1000) relative torque error.
  std::vector<Rigid> D(n);
  auto dot = [](const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; };
  auto cross = [](const double* a, const double* b, double* c) {
    c[0] = a[1] * b[2] - a[2] * b[1]; c[1] = a[2] * b[0] - a[0] * b[2]; c[2] = a[0] * b[1] - a[1] * b[0];
  };
  for (int i = 0; i < n; ++i) {
    const double z[3] = {0, 0, 1}, o[3] = {0, 0, 0};
    double x[3], P[3];
    if (i == n - 1) {
      x[0] = 1; x[1] = 0; x[2] = 0;
      for (int k = 0; k < 3; ++k) P[k] = o[k];
    } else {
      const Rigid& N = Mp[i + 1];                       // joint frame i+1 in joint frame i
      const double z2[3] = {N.R[0][2], N.R[1][2], N.R[2][2]}, o2[3] = {N.p[0], N.p[1], N.p[2]};
      double cz[3];
      cross(z, z2, cz);
      const double cn = std::sqrt(dot(cz, cz));
      double w0[3] = {o[0] - o2[0], o[1] - o2[1], o[2] - o2[2]};
      if (cn > 1e-9) {
        const double b = dot(z, z2), dd = dot(z, w0), e = dot(z2, w0), den = 1 - b * b;
        const double s1 = (b * e - dd) / den, t2 = (e - b * dd) / den;
        double Q[3];
        for (int k = 0; k < 3; ++k) { P[k] = o[k] + s1 * z[k]; Q[k] = o2[k] + t2 * z2[k]; }
        double r[3] = {Q[0] - P[0], Q[1] - P[1], Q[2] - P[2]};
        const double rn = std::sqrt(dot(r, r));
        if (rn > 1e-12) for (int k = 0; k < 3; ++k) x[k] = r[k] / rn;
        else for (int k = 0; k < 3; ++k) x[k] = cz[k] / cn;
      } else {
        double r[3] = {o2[0] - o[0], o2[1] - o[1], o2[2] - o[2]};
        const double rz = dot(r, z);
        for (int k = 0; k < 3; ++k) r[k] -= rz * z[k];
        const double rn = std::sqrt(dot(r, r));
        if (rn > 1e-12) for (int k = 0; k < 3; ++k) x[k] = r[k] / rn;
        else { x[0] = 1; x[1] = 0; x[2] = 0; }
        for (int k = 0; k < 3; ++k) P[k] = o[k];
      }
    }
    double y[3];
    cross(z, x, y);
    for (int k = 0; k < 3; ++k) {
      D[i].R[k][0] = x[k]; D[i].R[k][1] = y[k]; D[i].R[k][2] = z[k];
      D[i].p[k] = P[k];
    }
  }
  // Conditioning: nearly parallel consecutive axes put the common normal, and so the
  // DH origin, far from the links; the DH maps then carry large, cancelling moment
  // arms.  Measured (tools/near_parallel_accuracy.py, profiles/r02/near_parallel.csv):
  // DH origin at 20 / 60 / 200 / 600 link lengths -> 5.6e-12 / 5.8e-11 / 7.5e-9 /
  // 6.7e-8 relative torque error.  Beyond kDhMaxStretch the model keeps the
  // joint-frame kernels only (exact to ~1e-14).
  constexpr double kDhMaxStretch = 50.0;
  double lref = 1e-9;
  for (int i = 0; i < n; ++i)
    lref = std::max(lref, std::sqrt(Mp[i].p[0] * Mp[i].p[0] + Mp[i].p[1] * Mp[i].p[1] + Mp[i].p[2] * Mp[i].p[2]));
  for (int i = 0; i < n; ++i) {
    const double off = std::sqrt(D[i].p[0] * D[i].p[0] + D[i].p[1] * D[i].p[1] + D[i].p[2] * D[i].p[2]);
    if (!(off <= kDhMaxStretch * lref)) return false;
  }
  m->D0 = rigid_mul(Mp[0], D[0]);                      // DH base frame in the user's base frame
  m->D64.resize(n);
  m->D32.resize(n);
  m->C64.resize(n);
  m->C32.resize(n);
  for (int i = 0; i < n; ++i) {
    const Rigid Mi = (i == 0) ? rigid_identity() : rigid_mul(rigid_inv(D[i - 1]), rigid_mul(Mp[i], D[i]));
    const double ca = Mi.R[2][2], sa = -Mi.R[1][2];
    const double ct = Mi.R[0][0], st = -Mi.R[0][1];
    const double a = Mi.p[0], d = -sa * Mi.p[1] + ca * Mi.p[2];
    // verify the DH form R = Rx(alpha) Rz(th0), p = (a, -sa d, ca d)
    const double Rr[3][3] = {{ct, -st, 0}, {ca * st, ca * ct, -sa}, {sa * st, sa * ct, ca}};
    double err = std::fabs(Mi.p[1] + sa * d) + std::fabs(Mi.p[2] - ca * d);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) err += std::fabs(Mi.R[r][c] - Rr[r][c]);
    if (!(err < 1e-10)) return false;
    // Inertia in the DH frame from the joint-frame inertia (the joint frame sits at the
    // link, the DH origin can be metres away on the common normal): centre of mass
    // c_j and rotational inertia I_c about it in the joint frame, then
    // c = R_E^T (c_j - p_E), I_c' = R_E^T I_c R_E for E = G_i^-1 D_i, and the
    // inertia about the DH origin I = I_c' + m (|c|^2 1 - c c^T).  (Congruence of
    // the 6x6 J by Ad_E instead forms m |p_E|^2-sized terms and recovers I_c by
    // cancellation: ~1e-11 relative torque error on long random chains.)
    const Rigid& E = D[i];                                // DH frame i in joint frame i
    const std::array<double, 36>& Jj = Jp[i];
    const double mj = (Jj[0] + Jj[7] + Jj[14]) / 3.0;
    const double hj[3] = {0.5 * (Jj[6 * 5 + 1] - Jj[6 * 4 + 2]), 0.5 * (Jj[6 * 3 + 2] - Jj[6 * 5 + 0]),
                          0.5 * (Jj[6 * 4 + 0] - Jj[6 * 3 + 1])};
    const double cj[3] = {hj[0] / mj, hj[1] / mj, hj[2] / mj};
    double Icj[3][3];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) Icj[r][c] = 0.5 * (Jj[6 * (3 + r) + 3 + c] + Jj[6 * (3 + c) + 3 + r]);
    const double cj2 = cj[0] * cj[0] + cj[1] * cj[1] + cj[2] * cj[2];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) Icj[r][c] -= mj * ((r == c ? cj2 : 0.0) - cj[r] * cj[c]);
    double cd[3], Icd[3][3];
    for (int r = 0; r < 3; ++r) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += E.R[k][r] * (cj[k] - E.p[k]);
      cd[r] = s;
    }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double s = 0;
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) s += E.R[k][r] * Icj[k][l] * E.R[l][c];
        Icd[r][c] = s;
      }
    const double cd2 = cd[0] * cd[0] + cd[1] * cd[1] + cd[2] * cd[2];
    rd::LinkDH<double>& L = m->D64[i];
    L.ca = ca; L.sa = sa;
    L.a = a; L.d = d;
    L.th0 = std::atan2(st, ct);
    L.cth0 = std::cos(L.th0);
    L.sth0 = std::sin(L.th0);
    L.m = mj;
    for (int k = 0; k < 3; ++k) L.h[k] = mj * cd[k];
    L.I[0] = Icd[0][0] + mj * (cd2 - cd[0] * cd[0]);
    L.I[1] = Icd[1][1] + mj * (cd2 - cd[1] * cd[1]);
    L.I[2] = Icd[2][2] + mj * (cd2 - cd[2] * cd[2]);
    L.I[3] = 0.5 * (Icd[0][1] + Icd[1][0]) - mj * cd[0] * cd[1];
    L.I[4] = 0.5 * (Icd[0][2] + Icd[2][0]) - mj * cd[0] * cd[2];
    L.I[5] = 0.5 * (Icd[1][2] + Icd[2][1]) - mj * cd[1] * cd[2];
    rd::LinkDH<float>& F = m->D32[i];
    F.ca = (float)L.ca; F.sa = (float)L.sa; F.a = (float)L.a; F.d = (float)L.d;
    F.th0 = (float)L.th0; F.m = (float)L.m;
    F.cth0 = (float)L.cth0; F.sth0 = (float)L.sth0;
    for (int k = 0; k < 3; ++k) F.h[k] = (float)L.h[k];
    for (int k = 0; k < 6; ++k) F.I[k] = (float)L.I[k];
    // inertia about the centre of mass c = h / m: I_c = I - m (|c|^2 1 - c c^T)
    rd::LinkDHc<double>& Lc = m->C64[i];
    Lc.ca = L.ca; Lc.sa = L.sa; Lc.a = L.a; Lc.d = L.d;
    Lc.th0 = L.th0; Lc.cth0 = L.cth0; Lc.sth0 = L.sth0; Lc.m = L.m;
    for (int k = 0; k < 3; ++k) Lc.c[k] = cd[k];                    // direct, no cancellation
    Lc.Ic[0] = Icd[0][0]; Lc.Ic[1] = Icd[1][1]; Lc.Ic[2] = Icd[2][2];
    Lc.Ic[3] = 0.5 * (Icd[0][1] + Icd[1][0]);
    Lc.Ic[4] = 0.5 * (Icd[0][2] + Icd[2][0]);
    Lc.Ic[5] = 0.5 * (Icd[1][2] + Icd[2][1]);
    rd::LinkDHc<float>& Fc = m->C32[i];
    Fc.ca = (float)Lc.ca; Fc.sa = (float)Lc.sa; Fc.a = (float)Lc.a; Fc.d = (float)Lc.d;
    Fc.th0 = (float)Lc.th0; Fc.cth0 = (float)Lc.cth0; Fc.sth0 = (float)Lc.sth0; Fc.m = (float)Lc.m;
    for (int k = 0; k < 3; ++k) Fc.c[k] = (float)Lc.c[k];
    for (int k = 0; k < 6; ++k) Fc.Ic[k] = (float)Lc.Ic[k];
  }
  return true;
}

// Stream-ordered workspace of one call (see rd_model_s::pool).  The pool is
// created on first use on the model's device.
rd_status_t ws_alloc(rd_model_t m, size_t bytes, cudaStream_t s, void** out) {
  *out = nullptr;
  {
    std::lock_guard<std::mutex> lk(m->pool_mu);
    if (!m->pool) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = m->device;
      cudaError_t e = cudaMemPoolCreate(&m->pool, &props);
      if (e != cudaSuccess) { m->pool = nullptr; return cuda_fail(e, "workspace pool create"); }
      uint64_t keep = UINT64_MAX;
      e = cudaMemPoolSetAttribute(m->pool, cudaMemPoolAttrReleaseThreshold, &keep);
      if (e != cudaSuccess) return cuda_fail(e, "workspace pool attribute");
    }
  }
  cudaError_t e = cudaMallocFromPoolAsync(out, bytes, m->pool, s);
  if (e != cudaSuccess) {
    *out = nullptr;
    return fail(RD_E_NOMEM, std::string("workspace cudaMallocFromPoolAsync: ") + cudaGetErrorString(e));
  }
  return RD_OK;
}

// Frees the call's workspace on its stream after the launches (stream order).
struct WsScope {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~WsScope() { if (p) cudaFreeAsync(p, s); }
};

// Device-memory check: the pointer must be device (or managed) memory of the
// model's device.  A small per-thread cache of recently verified (address, device)
// pairs skips cudaPointerGetAttributes (~1 us per pointer, which dominated the
// host side of small-batch calls).  Under UVA an address denotes one allocation
// at a time, so a cached device address cannot later denote host memory; a
// freed and re-mapped address on ANOTHER device is the one case the cache can
// miss, and it is re-verified whenever the cached device differs from the model's.
struct PtrCacheEntry { uintptr_t addr; int device; };
thread_local PtrCacheEntry g_ptr_cache[16] = {};
thread_local int g_ptr_next = 0;

template <typename T>
bool is_device_ptr(const T* p, int device) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p);
  for (const PtrCacheEntry& c : g_ptr_cache)
    if (c.addr == a0 && c.device == device) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const bool dev = (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) && a.device == device;
  if (dev) {
    g_ptr_cache[g_ptr_next] = PtrCacheEntry{a0, device};
    g_ptr_next = (g_ptr_next + 1) % 16;
  }
  return dev;
}

template <typename T>
rd_status_t check_io(rd_model_t m, int64_t batch, const T* a, const T* b, const T* c, const T* out, bool device) {
  if (!m) return fail(RD_E_ARG, "null model");
  if (batch < 0) return fail(RD_E_ARG, "batch < 0");
  if (batch == 0) return RD_OK;
  const T* ins[3] = {a, b, c};
  const char* names[4] = {"q", "qd", "third input", "output"};
  const T* all[4] = {a, b, c, out};
  for (int k = 0; k < 4; ++k) {
    if (!all[k]) return fail(RD_E_ARG, std::string("null pointer: ") + names[k]);
    if (reinterpret_cast<uintptr_t>(all[k]) % sizeof(T) != 0) return fail(RD_E_ARG, std::string("misaligned pointer: ") + names[k]);
    if (device && !is_device_ptr(all[k], m->device))
      return fail(RD_E_ARG, std::string("not device memory of the model's device: ") + names[k]);
  }
  const size_t bytes = (size_t)m->n * (size_t)batch * sizeof(T);
  for (int k = 0; k < 3; ++k) {
    const char* lo = reinterpret_cast<const char*>(ins[k]);
    const char* olo = reinterpret_cast<const char*>(out);
    if (olo < lo + bytes && lo < olo + bytes) return fail(RD_E_ARG, std::string("output aliases input ") + names[k]);
  }
  int dev = -1;
  cudaGetDevice(&dev);
  if (device && dev != m->device) return fail(RD_E_ARG, "current CUDA device differs from the model's device");
  return RD_OK;
}

template <typename T> const rd::LinkConst<T>* jf_consts(rd_model_t m);     // host copies (kernel parameters)
template <> const rd::LinkConst<double>* jf_consts<double>(rd_model_t m) { return m->L64.data(); }
template <> const rd::LinkConst<float>* jf_consts<float>(rd_model_t m) { return m->L32.data(); }
template <typename T> const rd::LinkConst<T>* dev_consts(rd_model_t m);
template <> const rd::LinkConst<double>* dev_consts<double>(rd_model_t m) { return m->dL64; }
template <> const rd::LinkConst<float>* dev_consts<float>(rd_model_t m) { return m->dL32; }
template <typename T> const rd::LinkDH<T>* dh_consts(rd_model_t m);
template <> const rd::LinkDH<double>* dh_consts<double>(rd_model_t m) { return m->D64.data(); }
template <> const rd::LinkDH<float>* dh_consts<float>(rd_model_t m) { return m->D32.data(); }
template <typename T> const rd::LinkDHc<T>* dhc_consts(rd_model_t m);
template <> const rd::LinkDHc<double>* dhc_consts<double>(rd_model_t m) { return m->C64.data(); }
template <> const rd::LinkDHc<float>* dhc_consts<float>(rd_model_t m) { return m->C32.data(); }
template <typename T> const rd::LinkDHc<T>* dhc_dev(rd_model_t m);
template <> const rd::LinkDHc<double>* dhc_dev<double>(rd_model_t m) { return m->dC64; }
template <> const rd::LinkDHc<float>* dhc_dev<float>(rd_model_t m) { return m->dC32; }
template <typename T> const rd::LinkDH<T>* dh_dev(rd_model_t m);
template <> const rd::LinkDH<double>* dh_dev<double>(rd_model_t m) { return m->dD64; }
template <> const rd::LinkDH<float>* dh_dev<float>(rd_model_t m) { return m->dD32; }
template <typename T> const rd::Boundary<T>& dh_bnd(rd_model_t m);
template <> const rd::Boundary<double>& dh_bnd<double>(rd_model_t m) { return m->bdh64; }
template <> const rd::Boundary<float>& dh_bnd<float>(rd_model_t m) { return m->bdh32; }
template <typename T> const rd::Boundary<T>& bnd(rd_model_t m);
template <> const rd::Boundary<double>& bnd<double>(rd_model_t m) { return m->b64; }
template <> const rd::Boundary<float>& bnd<float>(rd_model_t m) { return m->b32; }

// Strategy table, measured on B200 as device time
// per call (CUDA-graph replay; profiles/r02/auto_grid_f64.csv, auto_grid_f32.csv).
// DH chains (revolute / prismatic joints):
//  * the register-resident THREAD kernel (rnea_small.cu; fp64 n <= 12, fp32 n <= 32
//    but 25, 26) except WARP_SCAN for the smallest batches of
//    the longer chains and REVERSE for fp32 n >= 24 at 4-16k states (below);
//  * n <= 32: WARP_SCAN (warp per state, lane = link; the latency regime of the
//    paper) for batch <= 1536 (fp64: n >= 7; fp32: n >= 20), e.g. n = 30,
//    B = 1000: 6.1 us vs 9.7 (CHUNK 16) / 10.4 (BLOCK_SCAN); up to 3072 for n >= 24
//    (n = 30, B = 2048: 10.4 vs 11.3 us CHUNK 8); CHUNK with 8 / 4 lanes for
//    16 <= n <= 32 at batches up to 3072 / 6144 (n = 30, B = 4096: 13.2 vs
//    14.0 us REVERSE); THREAD above the thread crossover (fp64 32768, fp32 49152;
//    n = 30, B = 65536: 38 vs 43 us) when the on-chip stash fits (n <= 30 fp64 /
//    32 fp32); REVERSE in between;
//  * n > 32: BLOCK_SCAN (CTA per state) for batch <= 512 (<= 1024 fp32 n < 100);
//    CHUNK with 16 (32 for n >= 150) lanes up to 1536, 8 lanes up to 3072, 4 (8 for
//    n >= 150) lanes up to 6144 (n = 100, B = 1000 / 2048 / 4096: 16 / 19 / 27 us vs
//    BLOCK_SCAN 33 / REVERSE 40 us); REVERSE above (and for n > 300 from 3072 on).
// Screw joints (no DH form): WARP_SCAN for n <= 32 and batch <= 4096, BLOCK_SCAN
// for longer chains and batch <= 1024, else GENERIC.
constexpr int64_t kWarpScanMaxBatch = 4096;     // joint-frame chains
constexpr int64_t kBlockScanMaxBatch = 1024;
constexpr int64_t kThreadMinBatch64 = 32768, kThreadMinBatch32 = 49152;

struct Plan {
  rd_strategy_t s;
  int lanes;        // CHUNK: lanes per state
};

Plan resolve_plan(rd_model_t m, int64_t batch, bool fp64) {
  const int n = m->n;
  // THREAD: the DH kernels, or the joint-frame register kernel for short chains
  const bool thread_ok = m->dh_ok ? rd::thread_kernel_has_n(n, fp64) : rd::small_jf_has_n(n, fp64);
  const bool warp_ok = n <= 32;
  // REVERSE exists in DH frames and in joint frames (any joints; constants in shared memory)
  const bool rev_ok = m->dh_ok || rd::rev_jf_has_n(n, fp64);
  switch (m->strategy) {
    case RD_STRAT_GENERIC: return {RD_STRAT_GENERIC, 0};
    case RD_STRAT_THREAD: return {thread_ok ? RD_STRAT_THREAD : (rev_ok ? RD_STRAT_REVERSE : RD_STRAT_GENERIC), 0};
    case RD_STRAT_WARP_SCAN: return {warp_ok ? RD_STRAT_WARP_SCAN : RD_STRAT_GENERIC, 0};
    case RD_STRAT_REVERSE: return {rev_ok ? RD_STRAT_REVERSE : RD_STRAT_GENERIC, 0};
    case RD_STRAT_BLOCK_SCAN: return {n <= 512 ? RD_STRAT_BLOCK_SCAN : RD_STRAT_GENERIC, 0};
    case RD_STRAT_WARP_SCAN_EQ13: return {warp_ok ? RD_STRAT_WARP_SCAN_EQ13 : RD_STRAT_GENERIC, 0};
    case RD_STRAT_WARP_SCAN_EQ15: return {warp_ok ? RD_STRAT_WARP_SCAN_EQ15 : RD_STRAT_GENERIC, 0};
    case RD_STRAT_CHUNK:
      if (!m->dh_ok) return {RD_STRAT_GENERIC, 0};
      return {RD_STRAT_CHUNK, m->chunk_lanes ? m->chunk_lanes : rd::chunk_default_lanes(n)};
    default: break;
  }
  if (m->dh_ok) {
    // the register-resident THREAD kernel (rnea_small.cu: fp64 n <= 12, fp32 n <= 32
    // but 25, 26) wherever it is not beaten
    // (profiles/r02/small_grid{,2,3}_f{64,32}.csv): n = 7, B = 256: 3.0 us vs 5.7
    // WARP_SCAN / 5.8 REVERSE, B = 1e6: 89 vs 161 us REVERSE; fp32 n = 30, 1e6: 0.218
    // vs 0.241 ms (stash kernel).  The warp scan keeps the smallest batches of the
    // longer chains (fp32 n = 30, B = 1024: 4.9 vs 8.5 us) and REVERSE the fp32
    // 8-16k band for n >= 24 (n = 30, 16384: 9.8 vs 11.0 us).
    if (rd::small_kernel_has_n(n, fp64, batch)) {
      if (fp64 && n >= 12 && batch <= 1024) return {RD_STRAT_WARP_SCAN, 0};
      if (!fp64 && ((n >= 16 && batch <= 1024) || (n >= 20 && batch <= 2048))) return {RD_STRAT_WARP_SCAN, 0};
      if (!fp64 && n >= 24 && batch > 4096 && batch <= 16384) return {RD_STRAT_REVERSE, 0};
      return {RD_STRAT_THREAD, 0};
    }
    if (warp_ok) {
      if (batch <= 1536 && n >= (fp64 ? 7 : 20)) return {RD_STRAT_WARP_SCAN, 0};
      if (batch <= 3072 && n >= 24) return {RD_STRAT_WARP_SCAN, 0};
      if (n >= 16 && batch <= 3072) return {RD_STRAT_CHUNK, 8};
      if (n >= 24 && batch <= 6144) return {RD_STRAT_CHUNK, 4};
      if (thread_ok && batch > (fp64 ? kThreadMinBatch64 : kThreadMinBatch32)) return {RD_STRAT_THREAD, 0};
      return {RD_STRAT_REVERSE, 0};
    }
    const int64_t block_max = (!fp64 && n < 100) ? 1024 : 512;
    if (n <= 512 && batch <= block_max) return {RD_STRAT_BLOCK_SCAN, 0};
    if (batch <= 1536) return {RD_STRAT_CHUNK, n >= 150 ? 32 : 16};
    if (batch <= 3072) return {RD_STRAT_CHUNK, 8};
    if (batch <= 6144 && n <= 300) return {RD_STRAT_CHUNK, n >= 150 ? 8 : 4};
    return {RD_STRAT_REVERSE, 0};
  }
  // joint frames (screw joints, or no well-conditioned DH form): warp scan for small
  // batches, then the joint-frame REVERSE, which needs no workspace: 1.6-2.3x GENERIC
  // from n = 30 (n = 30, 1e6: 0.744 vs 1.191 ms; n = 100, 4096: 0.052 vs 0.118 ms) and
  // 2.5x the warp scan for short chains at 4096 states (n = 7: 7.1 vs 17.7 us); GENERIC
  // keeps short chains at large batches (n = 7, 1e5: 21.7 vs 24.0 us)
  // (profiles/r02/jf_time.csv)
  if (thread_ok) return {RD_STRAT_THREAD, 0};                  // joint-frame register kernel (short chains)
  if (warp_ok && batch <= (n >= 16 ? kWarpScanMaxBatch : 1024)) return {RD_STRAT_WARP_SCAN, 0};
  if (!warp_ok && n <= 512 && batch <= kBlockScanMaxBatch) return {RD_STRAT_BLOCK_SCAN, 0};
  if (rev_ok && !(n <= 8 && batch > 32768)) return {RD_STRAT_REVERSE, 0};
  return {RD_STRAT_GENERIC, 0};
}

rd_strategy_t resolve(rd_model_t m, int64_t batch, bool fp64) { return resolve_plan(m, batch, fp64).s; }

// Per-state boundary arrays (NEXT-4): validated device arrays [6][batch] -> the
// kernel-side StateBoundary for joint-frame (jf) and DH kernels.
struct UserStateBoundary {
  const void* V0;
  const void* Vd0;
  const void* Ft;
};
template <typename T>
rd_status_t check_state_boundary(rd_model_t m, int64_t batch, const UserStateBoundary& u, const T* out) {
  const void* p[3] = {u.V0, u.Vd0, u.Ft};
  const char* names[3] = {"V0", "Vdot0", "Ftip"};
  const size_t bytes = (size_t)6 * batch * sizeof(T), ob = (size_t)m->n * batch * sizeof(T);
  for (int k = 0; k < 3; ++k) {
    if (!p[k]) continue;
    if (reinterpret_cast<uintptr_t>(p[k]) % sizeof(T) != 0) return fail(RD_E_ARG, std::string("misaligned pointer: ") + names[k]);
    if (!is_device_ptr(reinterpret_cast<const T*>(p[k]), m->device))
      return fail(RD_E_ARG, std::string("not device memory of the model's device: ") + names[k]);
    const char* lo = reinterpret_cast<const char*>(p[k]);
    const char* o = reinterpret_cast<const char*>(out);
    if (lo < o + ob && o < lo + bytes) return fail(RD_E_ARG, std::string("output aliases ") + names[k]);
  }
  return RD_OK;
}
template <typename T>
void make_state_boundary(rd_model_t m, const UserStateBoundary& u, bool dh, rd::StateBoundary<T>* sb) {
  sb->V0 = reinterpret_cast<const T*>(u.V0);
  sb->Vd0 = reinterpret_cast<const T*>(u.Vd0);
  sb->Ft = reinterpret_cast<const T*>(u.Ft);
  for (int i = 0; i < 36; ++i) {
    sb->A0[i] = dh ? (T)m->sbA0dh[i] : (T)((i % 7) == 0 ? 1.0 : 0.0);   // joint frames: T_0 = I
    sb->At[i] = (T)m->sbAt[i];                                        // last DH frame = joint frame n
  }
}

// force: the strategy resolved by the caller (the host pipeline resolves it ONCE for
// the whole batch, so host and device results are bit-identical at any batch size);
// RD_STRAT_AUTO = resolve here for this call's batch.
template <typename T>
rd_status_t inverse_dynamics(rd_model_t m, int64_t batch, const T* q, const T* qd, const T* qdd, T* tau,
                             void* stream, const UserStateBoundary* usb = nullptr,
                             Plan force = Plan{RD_STRAT_AUTO, 0}) {
  g_launches = 0;
  rd_status_t st = check_io<T>(m, batch, q, qd, qdd, tau, true);
  if (st != RD_OK || batch == 0) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Plan plan = force.s != RD_STRAT_AUTO ? force : resolve_plan(m, batch, sizeof(T) == 8);
  rd_strategy_t strat = plan.s;
  rd::StateBoundary<T> sbj, sbd;                 // joint-frame / DH variants
  const rd::StateBoundary<T>* pj = nullptr;
  const rd::StateBoundary<T>* pd = nullptr;
  if (usb) {
    st = check_state_boundary<T>(m, batch, *usb, tau);
    if (st != RD_OK) return st;
    make_state_boundary<T>(m, *usb, false, &sbj);
    make_state_boundary<T>(m, *usb, true, &sbd);
    pj = &sbj;
    pd = &sbd;
    if (strat == RD_STRAT_BLOCK_SCAN || strat == RD_STRAT_CHUNK) strat = RD_STRAT_REVERSE;   // (GENERIC if no REVERSE fits)
    if (strat == RD_STRAT_WARP_SCAN_EQ13 || strat == RD_STRAT_WARP_SCAN_EQ15)
      return fail(RD_E_UNSUPPORTED, "per-state boundary data: strategies THREAD, WARP_SCAN, GENERIC, REVERSE only");
  }
  cudaError_t e = cudaSuccess;
  if (strat == RD_STRAT_THREAD) {
    bool ok = false;
    if (m->dh_ok) {
      e = rd::launch_rnea_thread<T>(m->n, dhc_consts<T>(m), dh_bnd<T>(m), batch, q, qd, qdd, tau, s, &g_launches,
                                    &ok, m->prism_mask, pd);
    } else if (rd::small_jf_has_n(m->n, sizeof(T) == 8)) {
      e = rd::launch_rnea_small_jf<T>(m->n, jf_consts<T>(m), bnd<T>(m), batch, q, qd, qdd, tau, s, &g_launches, pj);
      ok = true;
    }
    if (!ok) strat = RD_STRAT_REVERSE;                 // (GENERIC if no REVERSE fits)
  } else if (strat == RD_STRAT_WARP_SCAN) {
    bool ok = false;
    e = rd::launch_rnea_warp<T>(m->n, dev_consts<T>(m), bnd<T>(m), batch, q, qd, qdd, tau, s, &g_launches, &ok,
                                nullptr, pj);
    if (!ok) strat = RD_STRAT_GENERIC;
  }
  if (strat == RD_STRAT_WARP_SCAN_EQ13) {
    bool ok = false;
    e = rd::launch_rnea_warp13<T>(m->n, dev_consts<T>(m), bnd<T>(m), batch, q, qd, qdd, tau, s, &g_launches, &ok);
    if (!ok) strat = RD_STRAT_GENERIC;
  }
  if (strat == RD_STRAT_WARP_SCAN_EQ15) {
    bool ok = false;
    e = rd::launch_rnea_warp15<T>(m->n, dev_consts<T>(m), bnd<T>(m), batch, q, qd, qdd, tau, s, &g_launches, &ok);
    if (!ok) strat = RD_STRAT_GENERIC;
  }
  if (strat == RD_STRAT_BLOCK_SCAN) {
    bool ok = false;
    e = rd::launch_rnea_block<T>(m->n, dev_consts<T>(m), bnd<T>(m), batch, q, qd, qdd, tau, s, &g_launches, &ok);
    if (!ok) strat = RD_STRAT_GENERIC;
  }
  if (strat == RD_STRAT_CHUNK) {
    const int lanes = plan.lanes ? plan.lanes : rd::chunk_default_lanes(m->n);
    WsScope ws;
    ws.s = s;
    st = ws_alloc(m, rd::chunk_ws_elems(m->n, batch, lanes) * sizeof(T), s, &ws.p);
    if (st != RD_OK) return st;
    e = rd::launch_rnea_chunk<T>(m->n, lanes, dhc_dev<T>(m), dh_bnd<T>(m), batch, q, qd, qdd, tau, s, &g_launches,
                                 m->has_prism ? m->dPrism : nullptr, reinterpret_cast<T*>(ws.p));
  }
  if (strat == RD_STRAT_REVERSE) {
    if (m->dh_ok)
      e = rd::launch_rnea_rev<T>(m->n, dhc_dev<T>(m), dh_bnd<T>(m), batch, q, qd, qdd, tau, s, &g_launches,
                                 m->has_prism ? m->dPrism : nullptr, pd);
    else if (rd::rev_jf_has_n(m->n, sizeof(T) == 8))    // joint frames: screw joints / ill-conditioned DH
      e = rd::launch_rnea_rev_jf<T>(m->n, dev_consts<T>(m), bnd<T>(m), batch, q, qd, qdd, tau, s, &g_launches, pj);
    else
      strat = RD_STRAT_GENERIC;
  }
  if (strat == RD_STRAT_GENERIC) {
    const int64_t slots = rd::generic_ws_slots(batch);
    WsScope ws;
    ws.s = s;
    st = ws_alloc(m, (size_t)slots * m->n * rd::generic_ws_per_link() * sizeof(T), s, &ws.p);
    if (st != RD_OK) return st;
    e = rd::launch_rnea_generic<T>(m->n, dev_consts<T>(m), bnd<T>(m), batch, q, qd, qdd, tau,
                                   reinterpret_cast<T*>(ws.p), slots, s, &g_launches, pj);
  }
  if (e != cudaSuccess) return cuda_fail(e, "inverse dynamics launch");
  return RD_OK;
}

template <typename T>
rd_status_t forward_dynamics(rd_model_t m, int64_t batch, const T* q, const T* qd, const T* tau, T* qdd,
                             void* stream, int32_t* status = nullptr, const UserStateBoundary* usb = nullptr) {
  g_launches = 0;
  rd_status_t st = check_io<T>(m, batch, q, qd, tau, qdd, true);
  if (st != RD_OK || batch == 0) return st;
  if (status) {
    if (reinterpret_cast<uintptr_t>(status) % sizeof(int32_t) != 0) return fail(RD_E_ARG, "misaligned pointer: status");
    if (!is_device_ptr(status, m->device)) return fail(RD_E_ARG, "not device memory of the model's device: status");
    const char* so = reinterpret_cast<const char*>(status);
    const char* qo = reinterpret_cast<const char*>(qdd);
    const size_t sb = (size_t)batch * sizeof(int32_t), qb = (size_t)m->n * (size_t)batch * sizeof(T);
    if (so < qo + qb && qo < so + sb) return fail(RD_E_ARG, "status aliases qdd");
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  rd::StateBoundary<T> sbj, sbd;
  if (usb) {
    st = check_state_boundary<T>(m, batch, *usb, qdd);
    if (st != RD_OK) return st;
    if (m->fd_algo != RD_FD_ABA) return fail(RD_E_UNSUPPORTED, "per-state boundary data: FD algorithm ABA only");
    make_state_boundary<T>(m, *usb, false, &sbj);
    make_state_boundary<T>(m, *usb, true, &sbd);
  }
  WsScope ws;                                       // this call's workspace, freed in stream order
  ws.s = s;
  if (m->fd_algo == RD_FD_JSIIA) {
    if (m->n > 256) return fail(RD_E_UNSUPPORTED, "JSIIA forward dynamics supports n <= 256 (use RD_FD_ABA)");
    T* jws = nullptr;
    if (m->n > 31) {                                  // CTA-wide JSIIA: per-CTA M in the workspace
      st = ws_alloc(m, rd::jsiia_ws_elems(m->n, batch) * sizeof(T), s, &ws.p);
      if (st != RD_OK) return st;
      jws = reinterpret_cast<T*>(ws.p);
    }
    bool ok = false;
    cudaError_t e = rd::launch_jsiia<T>(m->n, dev_consts<T>(m), bnd<T>(m), batch, q, qd, tau, qdd, s,
                                        &g_launches, &ok, status, jws);
    if (!ok) return fail(RD_E_UNSUPPORTED, "JSIIA forward dynamics supports n <= 256 (use RD_FD_ABA)");
    if (e != cudaSuccess) return cuda_fail(e, "forward dynamics (JSIIA) launch");
    return RD_OK;
  }
  if (m->fd_algo == RD_FD_ABA_SCAN || m->fd_algo == RD_FD_ABA_MERGED) {
    const bool merged = m->fd_algo == RD_FD_ABA_MERGED;
    if (merged ? m->n > 31 : m->n > 256)
      return fail(RD_E_UNSUPPORTED, merged ? "merged-scan ABIA forward dynamics supports n <= 31 (use RD_FD_ABA)"
                                           : "scan-ABIA forward dynamics supports n <= 256 (use RD_FD_ABA)");
    st = ws_alloc(m, rd::fd_scan_ws_elems(m->n, batch) * sizeof(T), s, &ws.p);
    if (st != RD_OK) return st;
    bool ok = false;
    cudaError_t e = merged
        ? rd::launch_fd_merged<T>(m->n, dev_consts<T>(m), bnd<T>(m), batch, q, qd, tau, qdd,
                                  reinterpret_cast<T*>(ws.p), s, &g_launches, &ok, status)
        : rd::launch_fd_scan<T>(m->n, dev_consts<T>(m), bnd<T>(m), batch, q, qd, tau, qdd,
                                reinterpret_cast<T*>(ws.p), s, &g_launches, &ok, status);
    if (!ok) return fail(RD_E_UNSUPPORTED, merged ? "merged-scan ABIA forward dynamics supports n <= 31 (use RD_FD_ABA)"
                                                  : "scan-ABIA forward dynamics supports n <= 256 (use RD_FD_ABA)");
    if (e != cudaSuccess) return cuda_fail(e, "forward dynamics (scan ABIA) launch");
    return RD_OK;
  }
  if (m->dh_ok && rd::aba_small_has_n(m->n, sizeof(T) == 8)) {   // short chain: workspace in registers
    cudaError_t e = rd::launch_aba_small<T>(m->n, dh_consts<T>(m), dh_bnd<T>(m), batch, q, qd, tau, qdd, s,
                                            &g_launches, status, m->prism_mask, usb ? &sbd : nullptr);
    if (e != cudaSuccess) return cuda_fail(e, "forward dynamics (register ABA) launch");
    return RD_OK;
  }
  if (!m->dh_ok && rd::aba_small_jf_has_n(m->n, sizeof(T) == 8)) {   // same in joint frames (any joints)
    cudaError_t e = rd::launch_aba_small_jf<T>(m->n, jf_consts<T>(m), bnd<T>(m), batch, q, qd, tau, qdd, s,
                                               &g_launches, status, usb ? &sbj : nullptr);
    if (e != cudaSuccess) return cuda_fail(e, "forward dynamics (joint-frame register ABA) launch");
    return RD_OK;
  }
  const int64_t slots = rd::generic_ws_slots(batch);
  st = ws_alloc(m, (size_t)slots * m->n * rd::aba_ws_per_link() * sizeof(T), s, &ws.p);
  if (st != RD_OK) return st;
  cudaError_t e = m->dh_ok
      ? rd::launch_aba_dh<T>(m->n, dh_dev<T>(m), dh_bnd<T>(m), batch, q, qd, tau, qdd,
                             reinterpret_cast<T*>(ws.p), slots, s, &g_launches, status,
                             m->has_prism ? m->dPrism : nullptr, usb ? &sbd : nullptr)
      : rd::launch_aba<T>(m->n, dev_consts<T>(m), bnd<T>(m), batch, q, qd, tau, qdd,
                          reinterpret_cast<T*>(ws.p), slots, s, &g_launches, status, usb ? &sbj : nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "forward dynamics launch");
  return RD_OK;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char* rd_version(void) { return "rd 0.1 (sm_100a; arXiv 1609.04493 batched scan-RNEA)"; }
const char* rd_last_error(void) { return g_err.c_str(); }
int32_t rd_last_launch_count(void) { return g_launches; }

rd_status_t rd_model_create(int32_t n, const double* M, const double* S, const double* J,
                            const double gravity[3], rd_model_t* out) {
  if (!out) return fail(RD_E_ARG, "null output handle");
  *out = nullptr;
  if (n < 1) return fail(RD_E_ARG, "n < 1");
  if (!M || !S || !J || !gravity) return fail(RD_E_ARG, "null model array");
  std::string viol;
  auto add = [&](int i, const std::string& s) {
    char buf[64];
    snprintf(buf, sizeof buf, "link %d: ", i + 1);
    if (!viol.empty()) viol += "; ";
    viol += buf + s;
  };
  for (int i = 0; i < n; ++i) {
    const double* Mi = M + 16 * i;
    const double* Si = S + 6 * i;
    const double* Ji = J + 36 * i;
    bool finite = true;
    for (int k = 0; k < 16; ++k) finite &= std::isfinite(Mi[k]);
    for (int k = 0; k < 6; ++k) finite &= std::isfinite(Si[k]);
    for (int k = 0; k < 36; ++k) finite &= std::isfinite(Ji[k]);
    if (!finite) { add(i, "non-finite entry"); continue; }
    // M: rigid transform
    double orth = 0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0;
        for (int k = 0; k < 3; ++k) s += Mi[4 * k + a] * Mi[4 * k + b];
        orth = std::max(orth, std::fabs(s - (a == b)));
      }
    double det = Mi[0] * (Mi[5] * Mi[10] - Mi[6] * Mi[9]) - Mi[1] * (Mi[4] * Mi[10] - Mi[6] * Mi[8]) +
                 Mi[2] * (Mi[4] * Mi[9] - Mi[5] * Mi[8]);
    if (orth > 1e-9) add(i, "home transform rotation not orthonormal (err " + std::to_string(orth) + ")");
    if (det < 0) add(i, "home transform rotation has det < 0");
    if (Mi[12] != 0 || Mi[13] != 0 || Mi[14] != 0 || Mi[15] != 1) add(i, "home transform last row is not 0 0 0 1");
    // S: unit twist
    double wn = std::sqrt(Si[3] * Si[3] + Si[4] * Si[4] + Si[5] * Si[5]);
    double vn = std::sqrt(Si[0] * Si[0] + Si[1] * Si[1] + Si[2] * Si[2]);
    if (wn > 1e-9) {
      if (std::fabs(wn - 1) > 1e-9) add(i, "joint twist angular norm " + std::to_string(wn) + " (must be 1)");
    } else if (std::fabs(vn - 1) > 1e-9) {
      add(i, "prismatic joint twist linear norm " + std::to_string(vn) + " (must be 1)");
    }
    // J: symmetric rigid-body spatial inertia, SPD
    double jmax = 0, asym = 0;
    for (int a = 0; a < 36; ++a) jmax = std::max(jmax, std::fabs(Ji[a]));
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) asym = std::max(asym, std::fabs(Ji[6 * a + b] - Ji[6 * b + a]));
    if (asym > 1e-9 * std::max(1.0, jmax)) add(i, "inertia not symmetric");
    double mass = Ji[0];
    double blk = 0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) blk = std::max(blk, std::fabs(Ji[6 * a + b] - (a == b ? mass : 0.0)));
    double skw = 0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) skw = std::max(skw, std::fabs(Ji[6 * (3 + a) + b] + Ji[6 * (3 + b) + a]));
    if (!(mass > 0)) add(i, "mass not positive");
    if (blk > 1e-9 * std::max(1.0, jmax)) add(i, "inertia upper-left block is not m*I (not a rigid body)");
    if (skw > 1e-9 * std::max(1.0, jmax)) add(i, "inertia off-diagonal block is not skew (not a rigid body)");
    Mat6 A;
    for (int a = 0; a < 6; ++a) for (int b = 0; b < 6; ++b) A[a][b] = 0.5 * (Ji[6 * a + b] + Ji[6 * b + a]);
    if (!cholesky6(A)) add(i, "inertia not positive definite");
  }
  if (!viol.empty()) return fail(RD_E_MODEL, viol);

  rd_model_t m = new (std::nothrow) rd_model_s;
  if (!m) return fail(RD_E_NOMEM, "host allocation");
  m->n = n;
  cudaGetDevice(&m->device);
  m->T.resize(n);
  m->L64.resize(n);
  m->L32.resize(n);
  m->all_revolute = true;
  m->dh_eligible = true;
  m->prism.assign(n, 0);
  std::vector<Rigid> Mps(n);
  std::vector<std::array<double, 36>> Jps(n);
  // Joint frames: T_i = (R_a, r) with R_a e_z = joint axis and r the point of
  // the axis closest to the link origin; then S'_i = Ad_{T_i^-1} S_i =
  // (beta e_z, alpha e_z), M'_i = T_{i-1}^-1 M_i T_i, J'_i = Ad_{T_i}^T J_i Ad_{T_i}.
  for (int i = 0; i < n; ++i) {
    const double* Si = S + 6 * i;
    double w[3] = {Si[3], Si[4], Si[5]}, v[3] = {Si[0], Si[1], Si[2]};
    double wn = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    Rigid Ti;
    double alpha, beta;
    if (wn > 1e-9) {
      for (int k = 0; k < 3; ++k) w[k] /= wn;
      frame_with_z(w, Ti.R);
      Ti.p[0] = w[1] * v[2] - w[2] * v[1];
      Ti.p[1] = w[2] * v[0] - w[0] * v[2];
      Ti.p[2] = w[0] * v[1] - w[1] * v[0];
      alpha = 1.0;
      beta = w[0] * v[0] + w[1] * v[1] + w[2] * v[2];   // pitch
      if (std::fabs(beta) < 1e-14) beta = 0.0;
    } else {
      double vv[3] = {v[0], v[1], v[2]};
      double vn = std::sqrt(vv[0] * vv[0] + vv[1] * vv[1] + vv[2] * vv[2]);
      for (int k = 0; k < 3; ++k) vv[k] /= vn;
      frame_with_z(vv, Ti.R);
      Ti.p[0] = Ti.p[1] = Ti.p[2] = 0;
      alpha = 0.0;
      beta = 1.0;
    }
    if (!(alpha == 1.0 && beta == 0.0)) m->all_revolute = false;
    if (alpha == 0.0) {
      m->prism[i] = 1;
      m->has_prism = true;
      if (i < 32) m->prism_mask |= 1u << i;
    } else if (beta != 0.0) {
      m->dh_eligible = false;                       // screw joint: no DH form with one variable
    }
    m->T[i] = Ti;
    Rigid Tprev = (i == 0) ? rigid_identity() : m->T[i - 1];
    Rigid Mp = rigid_mul(rigid_mul(rigid_inv(Tprev), rigid_from4(M + 16 * i)), Ti);
    Mps[i] = Mp;
    Mat6 A;
    adjoint(Ti, A);
    const double* Ji = J + 36 * i;
    double Jp[6][6];
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) {
        double s = 0;
        for (int k = 0; k < 6; ++k)
          for (int l = 0; l < 6; ++l) s += A[k][a] * Ji[6 * k + l] * A[l][b];
        Jp[a][b] = s;
        Jps[i][6 * a + b] = s;
      }
    rd::LinkConst<double>& C = m->L64[i];
    for (int a = 0; a < 3; ++a) {
      for (int b = 0; b < 3; ++b) C.Rm[3 * a + b] = Mp.R[a][b];
      C.pm[a] = Mp.p[a];
    }
    C.m = (Jp[0][0] + Jp[1][1] + Jp[2][2]) / 3.0;
    C.h[0] = 0.5 * (Jp[5][1] - Jp[4][2]);
    C.h[1] = 0.5 * (Jp[3][2] - Jp[5][0]);
    C.h[2] = 0.5 * (Jp[4][0] - Jp[3][1]);
    C.I[0] = Jp[3][3];
    C.I[1] = Jp[4][4];
    C.I[2] = Jp[5][5];
    C.I[3] = 0.5 * (Jp[3][4] + Jp[4][3]);
    C.I[4] = 0.5 * (Jp[3][5] + Jp[5][3]);
    C.I[5] = 0.5 * (Jp[4][5] + Jp[5][4]);
    C.alpha = alpha;
    C.beta = beta;
    rd::LinkConst<float>& F = m->L32[i];
    for (int k = 0; k < 9; ++k) F.Rm[k] = (float)C.Rm[k];
    for (int k = 0; k < 3; ++k) { F.pm[k] = (float)C.pm[k]; F.h[k] = (float)C.h[k]; }
    for (int k = 0; k < 6; ++k) F.I[k] = (float)C.I[k];
    F.m = (float)C.m;
    F.alpha = (float)C.alpha;
    F.beta = (float)C.beta;
  }
  for (int k = 0; k < 3; ++k) {
    m->gravity[k] = gravity[k];
    m->Vd0[k] = -gravity[k];     // reading A3: Vdot_0 = (-g, 0)
  }
  m->dh_ok = m->dh_eligible && build_dh(m, Mps, Jps);
  rebuild_boundary(m);
  cudaError_t e = cudaMalloc(&m->dL64, sizeof(rd::LinkConst<double>) * n);
  if (e == cudaSuccess) e = cudaMalloc(&m->dL32, sizeof(rd::LinkConst<float>) * n);
  if (e == cudaSuccess) e = cudaMemcpy(m->dL64, m->L64.data(), sizeof(rd::LinkConst<double>) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(m->dL32, m->L32.data(), sizeof(rd::LinkConst<float>) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && m->dh_ok) {
    e = cudaMalloc(&m->dD64, sizeof(rd::LinkDH<double>) * n);
    if (e == cudaSuccess) e = cudaMalloc(&m->dD32, sizeof(rd::LinkDH<float>) * n);
    if (e == cudaSuccess) e = cudaMemcpy(m->dD64, m->D64.data(), sizeof(rd::LinkDH<double>) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(m->dD32, m->D32.data(), sizeof(rd::LinkDH<float>) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&m->dC64, sizeof(rd::LinkDHc<double>) * n);
    if (e == cudaSuccess) e = cudaMalloc(&m->dC32, sizeof(rd::LinkDHc<float>) * n);
    if (e == cudaSuccess) e = cudaMemcpy(m->dC64, m->C64.data(), sizeof(rd::LinkDHc<double>) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(m->dC32, m->C32.data(), sizeof(rd::LinkDHc<float>) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && m->has_prism) e = cudaMalloc(&m->dPrism, n);
    if (e == cudaSuccess && m->has_prism) e = cudaMemcpy(m->dPrism, m->prism.data(), n, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    rd_model_destroy(m);
    return cuda_fail(e, "model upload");
  }
  *out = m;
  return RD_OK;
}

rd_status_t rd_model_destroy(rd_model_t m) {
  if (!m) return RD_OK;
  if (m->dL64) cudaFree(m->dL64);
  if (m->dL32) cudaFree(m->dL32);
  if (m->dD64) cudaFree(m->dD64);
  if (m->dD32) cudaFree(m->dD32);
  if (m->dC64) cudaFree(m->dC64);
  if (m->dC32) cudaFree(m->dC32);
  if (m->dPrism) cudaFree(m->dPrism);
  if (m->pool) cudaMemPoolDestroy(m->pool);
  for (int k = 0; k < 2; ++k) {
    if (m->hbuf[k]) cudaFree(m->hbuf[k]);
    if (m->hstream[k]) cudaStreamDestroy(m->hstream[k]);
  }
  delete m;
  return RD_OK;
}

int32_t rd_model_n(rd_model_t m) { return m ? m->n : -1; }
int32_t rd_model_device(rd_model_t m) { return m ? m->device : -1; }

rd_status_t rd_model_set_strategy(rd_model_t m, rd_strategy_t s, int32_t lanes_per_state) {
  if (!m) return fail(RD_E_ARG, "null model");
  if (s < RD_STRAT_AUTO || s > RD_STRAT_CHUNK) return fail(RD_E_ARG, "unknown strategy");
  if (s != RD_STRAT_CHUNK && lanes_per_state != 0) return fail(RD_E_ARG, "lanes_per_state is for RD_STRAT_CHUNK only");
  if (s == RD_STRAT_CHUNK && lanes_per_state != 0 &&
      (lanes_per_state < 2 || lanes_per_state > 32 || (lanes_per_state & (lanes_per_state - 1))))
    return fail(RD_E_ARG, "lanes_per_state must be 0 or a power of two in [2, 32]");
  m->strategy = s;
  m->chunk_lanes = s == RD_STRAT_CHUNK ? lanes_per_state : 0;
  return RD_OK;
}

rd_strategy_t rd_model_resolve_strategy(rd_model_t m, int64_t batch, int32_t fp64) {
  return m ? resolve(m, batch, fp64 != 0) : RD_STRAT_AUTO;
}

rd_status_t rd_model_set_fd_algo(rd_model_t m, rd_fd_algo_t algo) {
  if (!m) return fail(RD_E_ARG, "null model");
  if (algo != RD_FD_ABA && algo != RD_FD_JSIIA && algo != RD_FD_ABA_SCAN && algo != RD_FD_ABA_MERGED) return fail(RD_E_ARG, "unknown FD algorithm");
  m->fd_algo = algo;
  return RD_OK;
}

rd_status_t rd_model_set_boundary(rd_model_t m, const double V0[6], const double Vdot0[6], const double Ftip[6]) {
  if (!m) return fail(RD_E_ARG, "null model");
  for (int k = 0; k < 6; ++k) {
    m->V0[k] = V0 ? V0[k] : 0.0;
    m->Ftip_user[k] = Ftip ? Ftip[k] : 0.0;
    if (Vdot0) m->Vd0[k] = Vdot0[k];
  }
  if (!Vdot0) {
    for (int k = 0; k < 3; ++k) { m->Vd0[k] = -m->gravity[k]; m->Vd0[3 + k] = 0; }
  }
  rebuild_boundary(m);
  return RD_OK;
}

rd_status_t rd_inverse_dynamics_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                    const double* qdd, double* tau, void* stream) {
  return inverse_dynamics<double>(m, batch, q, qd, qdd, tau, stream);
}
rd_status_t rd_inverse_dynamics_f32(rd_model_t m, int64_t batch, const float* q, const float* qd,
                                    const float* qdd, float* tau, void* stream) {
  return inverse_dynamics<float>(m, batch, q, qd, qdd, tau, stream);
}
rd_status_t rd_forward_dynamics_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                    const double* tau, double* qdd, void* stream) {
  return forward_dynamics<double>(m, batch, q, qd, tau, qdd, stream);
}
rd_status_t rd_forward_dynamics_f32(rd_model_t m, int64_t batch, const float* q, const float* qd,
                                    const float* tau, float* qdd, void* stream) {
  return forward_dynamics<float>(m, batch, q, qd, tau, qdd, stream);
}
rd_status_t rd_inverse_dynamics_bnd_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                        const double* qdd, const double* V0, const double* Vdot0,
                                        const double* Ftip, double* tau, void* stream) {
  const UserStateBoundary u{V0, Vdot0, Ftip};
  return inverse_dynamics<double>(m, batch, q, qd, qdd, tau, stream, &u);
}
rd_status_t rd_inverse_dynamics_bnd_f32(rd_model_t m, int64_t batch, const float* q, const float* qd,
                                        const float* qdd, const float* V0, const float* Vdot0,
                                        const float* Ftip, float* tau, void* stream) {
  const UserStateBoundary u{V0, Vdot0, Ftip};
  return inverse_dynamics<float>(m, batch, q, qd, qdd, tau, stream, &u);
}
rd_status_t rd_forward_dynamics_bnd_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                        const double* tau, const double* V0, const double* Vdot0,
                                        const double* Ftip, double* qdd, int32_t* status, void* stream) {
  const UserStateBoundary u{V0, Vdot0, Ftip};
  return forward_dynamics<double>(m, batch, q, qd, tau, qdd, stream, status, &u);
}
rd_status_t rd_forward_dynamics_bnd_f32(rd_model_t m, int64_t batch, const float* q, const float* qd,
                                        const float* tau, const float* V0, const float* Vdot0,
                                        const float* Ftip, float* qdd, int32_t* status, void* stream) {
  const UserStateBoundary u{V0, Vdot0, Ftip};
  return forward_dynamics<float>(m, batch, q, qd, tau, qdd, stream, status, &u);
}
rd_status_t rd_forward_dynamics_ex_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                       const double* tau, double* qdd, int32_t* status, void* stream) {
  return forward_dynamics<double>(m, batch, q, qd, tau, qdd, stream, status);
}
rd_status_t rd_forward_dynamics_ex_f32(rd_model_t m, int64_t batch, const float* q, const float* qd,
                                       const float* tau, float* qdd, int32_t* status, void* stream) {
  return forward_dynamics<float>(m, batch, q, qd, tau, qdd, stream, status);
}

}  // extern "C"

namespace {
// Host-buffer pipeline: chunks of `chunk` states; chunk k uses device buffer set
// k%2 and stream k%2: H2D(q, qd, third) -> kernel -> D2H(out).  Two streams
// overlap chunk k+1's copies with chunk k's kernel (PCIe is full duplex).  The
// whole call holds the model's host_mu (the buffers and streams are per model),
// and the ID strategy is resolved ONCE for the whole batch, so every chunk runs
// the strategy a device call on the full batch would (bit-identical results).
// FD: false = inverse dynamics (third input qdd, output tau), true = forward
// dynamics (third input tau, output qdd; the model's FD algorithm).
constexpr int64_t kHostChunkBytes = 32ll << 20;   // per input array; measured: 4/8/16/32/64 MB ->
                                                  // 6.0/6.4/6.9/7.0/6.9e7 evals/s at C3 (PCIe-bound)
template <bool FD>
rd_status_t host_pipeline(rd_model_t m, int64_t batch, const double* q, const double* qd,
                          const double* third, double* out, int64_t chunk_bytes = kHostChunkBytes) {
  g_launches = 0;
  rd_status_t st = check_io<double>(m, batch, q, qd, third, out, false);
  if (st != RD_OK || batch == 0) return st;
  int dev = -1;
  cudaGetDevice(&dev);
  if (dev != m->device) return fail(RD_E_ARG, "current CUDA device differs from the model's device");
  std::lock_guard<std::mutex> lk(m->host_mu);
  const int n = m->n;
  const Plan plan = FD ? Plan{RD_STRAT_AUTO, 0} : resolve_plan(m, batch, true);
  const int64_t chunk = std::min<int64_t>(batch, std::max<int64_t>(4096, chunk_bytes / (8ll * n)));
  const size_t set_bytes = (size_t)4 * n * chunk * sizeof(double);
  if (m->hbuf_bytes < set_bytes) {
    for (int k = 0; k < 2; ++k) {
      if (m->hstream[k]) cudaStreamSynchronize(m->hstream[k]);
      if (m->hbuf[k]) cudaFree(m->hbuf[k]);
      m->hbuf[k] = nullptr;
    }
    m->hbuf_bytes = 0;
    for (int k = 0; k < 2; ++k) {
      cudaError_t e = cudaMalloc(&m->hbuf[k], set_bytes);
      if (e != cudaSuccess) return fail(RD_E_NOMEM, "host-path device buffers");
    }
    m->hbuf_bytes = set_bytes;
  }
  for (int k = 0; k < 2; ++k) {
    if (!m->hstream[k]) {
      cudaError_t e = cudaStreamCreateWithFlags(&m->hstream[k], cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_fail(e, "stream create");
    }
  }
  int launches = 0;
  rd_status_t result = RD_OK;
  for (int64_t b0 = 0, k = 0; b0 < batch; b0 += chunk, ++k) {
    const int64_t bc = std::min(chunk, batch - b0);
    cudaStream_t s = m->hstream[k & 1];
    double* base = reinterpret_cast<double*>(m->hbuf[k & 1]);
    double* dq = base;
    double* dqd = base + (size_t)n * chunk;
    double* d3 = base + (size_t)2 * n * chunk;
    double* dout = base + (size_t)3 * n * chunk;
    const size_t hp = (size_t)batch * sizeof(double), dp = (size_t)bc * sizeof(double);
    cudaError_t e = cudaMemcpy2DAsync(dq, dp, q + b0, hp, dp, n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpy2DAsync(dqd, dp, qd + b0, hp, dp, n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpy2DAsync(d3, dp, third + b0, hp, dp, n, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { result = cuda_fail(e, "host path H2D"); break; }
    st = FD ? forward_dynamics<double>(m, bc, dq, dqd, d3, dout, s)
            : inverse_dynamics<double>(m, bc, dq, dqd, d3, dout, s, nullptr, plan);
    launches += g_launches;
    if (st != RD_OK) { result = st; break; }
    e = cudaMemcpy2DAsync(out + b0, hp, dout, dp, dp, n, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) { result = cuda_fail(e, "host path D2H"); break; }
  }
  // always drain both streams before releasing the lock (the buffers are reused)
  for (int k = 0; k < 2; ++k) {
    cudaError_t e = cudaStreamSynchronize(m->hstream[k]);
    if (e != cudaSuccess && result == RD_OK) result = cuda_fail(e, "host path sync");
  }
  g_launches = launches;
  return result;
}
}  // namespace

extern "C" {
rd_status_t rd_inverse_dynamics_host_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                         const double* qdd, double* tau) {
  return host_pipeline<false>(m, batch, q, qd, qdd, tau);
}
rd_status_t rd_forward_dynamics_host_f64(rd_model_t m, int64_t batch, const double* q, const double* qd,
                                         const double* tau, double* qdd) {
  return host_pipeline<true>(m, batch, q, qd, tau, qdd);
}

}  // extern "C"
