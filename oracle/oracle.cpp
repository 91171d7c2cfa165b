/*
 * oracle/oracle.cpp -- TEST INFRASTRUCTURE ONLY (never on the product path).
 *
 * Plain, slow, obviously-correct CPU reference for arXiv 1609.04493 ("a parallel
 * framework for fast computation of inverse and forward dynamics ... based on
 * prefix sums").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.  It shares no
 * code, header, table or helper with paper_1609_04493_b200/ (the CUDA path).
 *
 * Citation key: P:n = PAPER.md line n.  Readings of gaps/garbles are the A#
 * entries of DESIGN.md ("Readings of the paper").
 *
 * Conventions (A1-A3):
 *   twists xi = (v, w) linear first; wrenches F = (f, m) dual, so
 *   tau = S^T F is a plain dot product;
 *   Ad_g = [[R, [p]R], [0, R]];  ad_xi = [[w^, v^], [0, w^]];
 *   f_{i-1,i} maps link-i coordinates to link-(i-1) coordinates;
 *   S_i, V_i, Vdot_i, F_i, J_i are in the body frame of link i;
 *   gravity enters as Vdot_0 = (-g, 0), V_0 = 0, F_{n+1} = 0 (A3).
 *
 * Everything is dense 4x4 / 6x6 double arithmetic with no precomputation,
 * blocking or fusion beyond what each equation states.  All arrays are
 * row-major.  Per-link model arrays: M[n][4][4], S[n][6], J[n][6][6].
 * Batch arrays are link-major (x[i*B + b]).
 */
#include <cmath>
#include <cstring>
#include <cstdint>
#include <vector>
#include <array>
#include <thread>
#include <functional>
#include <stdexcept>
#include <string>

namespace {

typedef std::array<double, 3> V3;
typedef std::array<double, 6> V6;
typedef std::array<std::array<double, 3>, 3> M3;
typedef std::array<std::array<double, 4>, 4> M4;
typedef std::array<std::array<double, 6>, 6> M6;

// ---------------------------------------------------------------- basic algebra
M6 zero6() { M6 A{}; return A; }
M6 eye6() { M6 A{}; for (int i = 0; i < 6; ++i) A[i][i] = 1.0; return A; }
M4 eye4() { M4 A{}; for (int i = 0; i < 4; ++i) A[i][i] = 1.0; return A; }
V6 zv6() { V6 v{}; return v; }

M6 mul6(const M6& A, const M6& B) {
  M6 C{};
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      double s = 0;
      for (int k = 0; k < 6; ++k) s += A[i][k] * B[k][j];
      C[i][j] = s;
    }
  return C;
}
V6 mv6(const M6& A, const V6& x) {
  V6 y{};
  for (int i = 0; i < 6; ++i) {
    double s = 0;
    for (int k = 0; k < 6; ++k) s += A[i][k] * x[k];
    y[i] = s;
  }
  return y;
}
M6 tr6(const M6& A) {
  M6 B{};
  for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) B[i][j] = A[j][i];
  return B;
}
M6 add6(const M6& A, const M6& B) {
  M6 C{}; for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) C[i][j] = A[i][j] + B[i][j];
  return C;
}
M6 sub6(const M6& A, const M6& B) {
  M6 C{}; for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) C[i][j] = A[i][j] - B[i][j];
  return C;
}
M6 scale6(const M6& A, double s) {
  M6 C{}; for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) C[i][j] = A[i][j] * s;
  return C;
}
M6 outer6(const V6& a, const V6& b) {
  M6 C{}; for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) C[i][j] = a[i] * b[j];
  return C;
}
V6 addv(const V6& a, const V6& b) { V6 c{}; for (int i = 0; i < 6; ++i) c[i] = a[i] + b[i]; return c; }
V6 subv(const V6& a, const V6& b) { V6 c{}; for (int i = 0; i < 6; ++i) c[i] = a[i] - b[i]; return c; }
V6 scalev(const V6& a, double s) { V6 c{}; for (int i = 0; i < 6; ++i) c[i] = a[i] * s; return c; }
double dot6(const V6& a, const V6& b) { double s = 0; for (int i = 0; i < 6; ++i) s += a[i] * b[i]; return s; }

M4 mul4(const M4& A, const M4& B) {
  M4 C{};
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double s = 0;
      for (int k = 0; k < 4; ++k) s += A[i][k] * B[k][j];
      C[i][j] = s;
    }
  return C;
}

M3 skew(const V3& a) {
  M3 K{};
  K[0][1] = -a[2]; K[0][2] = a[1];
  K[1][0] = a[2];  K[1][2] = -a[0];
  K[2][0] = -a[1]; K[2][1] = a[0];
  return K;
}
M3 mul3(const M3& A, const M3& B) {
  M3 C{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += A[i][k] * B[k][j];
      C[i][j] = s;
    }
  return C;
}

M4 load4(const double* p) { M4 A{}; for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) A[i][j] = p[4 * i + j]; return A; }
M6 load6(const double* p) { M6 A{}; for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) A[i][j] = p[6 * i + j]; return A; }
V6 loadv(const double* p) { V6 a{}; for (int i = 0; i < 6; ++i) a[i] = p[i]; return a; }
void store4(const M4& A, double* p) { for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) p[4 * i + j] = A[i][j]; }
void store6(const M6& A, double* p) { for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) p[6 * i + j] = A[i][j]; }
void storev(const V6& a, double* p) { for (int i = 0; i < 6; ++i) p[i] = a[i]; }

// --------------------------------------------------------------- SE(3) / se(3)
// P:25-27 nomenclature: SE(3), se(3), Ad, ad.

// Inverse of a rigid transform g = (R, p): (R^T, -R^T p).
M4 inv4(const M4& g) {
  M4 h = eye4();
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) h[i][j] = g[j][i];
  for (int i = 0; i < 3; ++i) {
    double s = 0;
    for (int k = 0; k < 3; ++k) s += g[k][i] * g[k][3];
    h[i][3] = -s;
  }
  return h;
}

// Adjoint transformation Ad_g = [[R, [p]R], [0, R]] for (v, w) twists (A1).
M6 Ad(const M4& g) {
  M3 R{}; V3 p{};
  for (int i = 0; i < 3; ++i) { for (int j = 0; j < 3; ++j) R[i][j] = g[i][j]; p[i] = g[i][3]; }
  M3 PR = mul3(skew(p), R);
  M6 A{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      A[i][j] = R[i][j];
      A[i][3 + j] = PR[i][j];
      A[3 + i][3 + j] = R[i][j];
    }
  return A;
}

// adjoint map ad_xi = [[w^, v^], [0, w^]] (Lie bracket ad_xi(eta) = [xi, eta]).
M6 ad(const V6& xi) {
  M3 W = skew({xi[3], xi[4], xi[5]});
  M3 Vh = skew({xi[0], xi[1], xi[2]});
  M6 A{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      A[i][j] = W[i][j];
      A[i][3 + j] = Vh[i][j];
      A[3 + i][3 + j] = W[i][j];
    }
  return A;
}

// Exponential e^{[S] q} of a joint twist ("f_{i-1,i} = M_i e^{S_i q_i}").
// Closed form: revolute/screw (|w| = 1): R = I + sin q [w] + (1 - cos q)[w]^2,
// p = (I q + (1 - cos q)[w] + (q - sin q)[w]^2) v ;  prismatic (w = 0): R = I,
// p = v q.  The branch is decided from the (double) model twist only.
M4 exp_twist(const V6& S, double q) {
  V3 w = {S[3], S[4], S[5]};
  V3 v = {S[0], S[1], S[2]};
  double wn = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  M4 g = eye4();
  if (wn < 0.5) {  // prismatic: |w| = 0, |v| = 1
    for (int i = 0; i < 3; ++i) g[i][3] = v[i] * q;
    return g;
  }
  M3 W = skew(w), W2 = mul3(W, W);
  double s = std::sin(q), c = std::cos(q);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      g[i][j] = (i == j ? 1.0 : 0.0) + s * W[i][j] + (1.0 - c) * W2[i][j];
  for (int i = 0; i < 3; ++i) {
    double t = 0;
    for (int j = 0; j < 3; ++j) {
      double G = (i == j ? q : 0.0) + (1.0 - c) * W[i][j] + (q - s) * W2[i][j];
      t += G * v[j];
    }
    g[i][3] = t;
  }
  return g;
}

struct Chain {
  int n;
  std::vector<M4> M;
  std::vector<V6> S;
  std::vector<M6> J;
};

Chain make_chain(int n, const double* M, const double* S, const double* J) {
  Chain c;
  c.n = n;
  for (int i = 0; i < n; ++i) {
    c.M.push_back(load4(M + 16 * i));
    c.S.push_back(loadv(S + 6 * i));
    c.J.push_back(load6(J + 36 * i));
  }
  return c;
}

// f_{i-1,i} = M_i e^{[S_i] q_i} for i = 1..n (Alg. 1 CalcTransform P:408).
// f[k] holds f_{k,k+1} (0-based link k = link k+1 of the paper).
std::vector<M4> calc_transform(const Chain& c, const double* q) {
  std::vector<M4> f(c.n);
  for (int i = 0; i < c.n; ++i) f[i] = mul4(c.M[i], exp_twist(c.S[i], q[i]));
  return f;
}

// ------------------------------------------------ RNEA, Eq. (1)-(2)
struct IdOut {
  std::vector<double> tau;
  std::vector<V6> V, Vd, F, Fhat;
};

// tau = ID(q, qd, qdd, V_0, Vdot_0, F_{n+1})   (Eq. 3).
IdOut rnea(const Chain& c, const double* q, const double* qd, const double* qdd,
           const V6& V0, const V6& Vd0, const V6& Ftip) {
  const int n = c.n;
  IdOut o;
  o.tau.assign(n, 0.0); o.V.assign(n, zv6()); o.Vd.assign(n, zv6());
  o.F.assign(n, zv6()); o.Fhat.assign(n, zv6());
  std::vector<M4> f = calc_transform(c, q);
  // Forward recursion, Eq. (1), i = 1..n.
  V6 Vp = V0, Vdp = Vd0;
  for (int i = 0; i < n; ++i) {
    M6 A = Ad(inv4(f[i]));                       // Ad_{f_{i-1,i}^{-1}}
    V6 Sqd = scalev(c.S[i], qd[i]);
    V6 AV = mv6(A, Vp);
    o.V[i] = addv(AV, Sqd);                      // V_i = Ad V_{i-1} + S_i qd_i
    o.Vd[i] = subv(addv(scalev(c.S[i], qdd[i]), mv6(A, Vdp)),
                   mv6(ad(Sqd), AV));            // Vdot_i = S qdd + Ad Vdot - ad_{S qd} Ad V
    Vp = o.V[i]; Vdp = o.Vd[i];
  }
  // Backward recursion, Eq. (2), i = n..1.
  V6 Fn = Ftip;
  for (int i = n - 1; i >= 0; --i) {
    M6 AT = (i == n - 1) ? eye6() : tr6(Ad(inv4(f[i + 1])));   // Ad^T_{f_{i,i+1}^{-1}}; f_{n,n+1} := I
    V6 JV = mv6(c.J[i], o.V[i]);
    o.Fhat[i] = subv(mv6(c.J[i], o.Vd[i]), mv6(tr6(ad(o.V[i])), JV));  // J Vdot - ad^T_V (J V)
    o.F[i] = addv(mv6(AT, Fn), o.Fhat[i]);
    o.tau[i] = dot6(c.S[i], o.F[i]);             // tau_i = S_i^T F_i
    Fn = o.F[i];
  }
  return o;
}

// ------------------------------------------------ scans, Eq. (9)-(11)
// combine(earlier, later) is the semigroup product with the later operand on the
// LEFT (reading A4: P_i = a_i (+) P_{i-1}), so both orders below compute the
// same inclusive prefixes x_i = a_i (+) ... (+) a_0 with different association.
template <class E>
std::vector<E> scan_sequential(const std::vector<E>& a, const std::function<E(const E&, const E&)>& combine) {
  std::vector<E> x(a.size());
  if (a.empty()) return x;
  x[0] = a[0];
  for (size_t i = 1; i < a.size(); ++i) x[i] = combine(x[i - 1], a[i]);
  return x;
}
// Kogge-Stone (Hillis-Steele) tree order: log2(n) rounds, round d combines
// x_{i-d} with x_i (the association a GPU warp scan uses).
template <class E>
std::vector<E> scan_kogge_stone(const std::vector<E>& a, const std::function<E(const E&, const E&)>& combine) {
  std::vector<E> x = a;
  for (size_t d = 1; d < a.size(); d <<= 1) {
    std::vector<E> y = x;
    for (size_t i = d; i < a.size(); ++i) y[i] = combine(x[i - d], x[i]);
    x = y;
  }
  return x;
}
template <class E>
std::vector<E> run_scan(int order, const std::vector<E>& a, const std::function<E(const E&, const E&)>& combine) {
  return order == 0 ? scan_sequential<E>(a, combine) : scan_kogge_stone<E>(a, combine);
}

// Element of SE(3) x se(3)^2 with the operation of Eq. (13):
// (g, xi1, xi2) (+) (g', xi1', xi2') = (g g', Ad_g xi1' + xi1 - ad_{xi2} Ad_g xi2', Ad_g xi2' + xi2).
struct VelAcc { M4 g; V6 xi1, xi2; };
VelAcc velacc_oplus(const VelAcc& a, const VelAcc& b) {
  M6 A = Ad(a.g);
  V6 Ax1 = mv6(A, b.xi1), Ax2 = mv6(A, b.xi2);
  VelAcc r;
  r.g = mul4(a.g, b.g);
  r.xi1 = subv(addv(Ax1, a.xi1), mv6(ad(a.xi2), Ax2));
  r.xi2 = addv(Ax2, a.xi2);
  return r;
}
// Inverse, Eq. (14): (g^{-1}, -Ad_{g^{-1}} xi1, -Ad_{g^{-1}} xi2).
VelAcc velacc_inverse(const VelAcc& a) {
  VelAcc r;
  r.g = inv4(a.g);
  M6 A = Ad(r.g);
  r.xi1 = scalev(mv6(A, a.xi1), -1.0);
  r.xi2 = scalev(mv6(A, a.xi2), -1.0);
  return r;
}
// 13x13 lift Phi of Eq. (12): [[Ad_g, -ad_{xi2} Ad_g, xi1], [0, Ad_g, xi2], [0, 0, 1]].
void velacc_lift13(const VelAcc& a, double* out /*13x13*/) {
  std::memset(out, 0, 169 * sizeof(double));
  M6 A = Ad(a.g);
  M6 B = scale6(mul6(ad(a.xi2), A), -1.0);
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      out[13 * i + j] = A[i][j];
      out[13 * i + 6 + j] = B[i][j];
      out[13 * (6 + i) + 6 + j] = A[i][j];
    }
  for (int i = 0; i < 6; ++i) { out[13 * i + 12] = a.xi1[i]; out[13 * (6 + i) + 12] = a.xi2[i]; }
  out[13 * 12 + 12] = 1.0;
}

// Ad-affine element (g, xi) with (g, xi) (+) (g', xi') = (g g', Ad_g xi' + xi):
// the sub-semigroup of Eq. (13) dropping xi1, used by the split scans of Alg. 1.
struct AdAff { M4 g; V6 xi; };
AdAff adaff_oplus(const AdAff& a, const AdAff& b) {
  AdAff r;
  r.g = mul4(a.g, b.g);
  r.xi = addv(mv6(Ad(a.g), b.xi), a.xi);
  return r;
}

// Affine map F -> L F + b (the backward operand of Eq. (16), without
// the lagged torque row, reading A5).  Composition B_k o B_{k+1}.
struct Aff6 { M6 L; V6 b; };
Aff6 aff_compose(const Aff6& later_left, const Aff6& earlier_right) {
  Aff6 r;
  r.L = mul6(later_left.L, earlier_right.L);
  r.b = addv(mv6(later_left.L, earlier_right.b), later_left.b);
  return r;
}

// Bias wrench Fhat = J Vdot - ad^T_V (J V).
V6 bias_force(const M6& J, const V6& V, const V6& Vd) {
  return subv(mv6(J, Vd), mv6(tr6(ad(V)), mv6(J, V)));
}

// Alg. 1 lines 4-5: backward force scan over k = n+1, n, ..., 1 with operands
// B_k = (Ad^T_{f_{k,k+1}^{-1}}, Fhat_k) (Eq. 2 / Eq. 16 without the lagged torque
// row, A5), seed F_{n+1}; then CalcTorque tau_k = S_k^T F_k.
void force_scan_and_torque(const Chain& c, const std::vector<M4>& f, const V6& Ftip, int order, IdOut& o) {
  const int n = c.n;
  std::vector<Aff6> b(n + 1);
  b[0] = {zero6(), Ftip};           // constant map to F_{n+1}
  for (int k = n - 1; k >= 0; --k) {
    M6 L = (k == n - 1) ? eye6() : tr6(Ad(inv4(f[k + 1])));   // f_{n,n+1} := I
    b[n - k] = {L, o.Fhat[k]};
  }
  std::function<Aff6(const Aff6&, const Aff6&)> combF =
      [](const Aff6& earlier, const Aff6& later) { return aff_compose(later, earlier); };
  std::vector<Aff6> Q = run_scan<Aff6>(order, b, combF);
  for (int k = 0; k < n; ++k) {
    o.F[k] = Q[n - k].b;            // F_k = (B_k o ... o B_n)(F_{n+1})
    o.tau[k] = dot6(c.S[k], o.F[k]);
  }
}

// Parallel ID of Alg. 1 with structured operands:
// CalcTransform -> InclusiveVelScan -> InclusiveAccScan -> bias forces
// -> InclusiveForceScan (backward) -> CalcTorque.
IdOut rnea_scan_split(const Chain& c, const double* q, const double* qd, const double* qdd,
                      const V6& V0, const V6& Vd0, const V6& Ftip, int order) {
  const int n = c.n;
  IdOut o;
  o.tau.assign(n, 0.0); o.V.assign(n, zv6()); o.Vd.assign(n, zv6());
  o.F.assign(n, zv6()); o.Fhat.assign(n, zv6());
  std::vector<M4> f = calc_transform(c, q);                       // line 1
  std::function<AdAff(const AdAff&, const AdAff&)> comb =
      [](const AdAff& earlier, const AdAff& later) { return adaff_oplus(later, earlier); };
  // line 2: velocity scan, operands (f^{-1}, S qd), seed a_0 = (I, V_0).
  std::vector<AdAff> a(n + 1);
  a[0] = {eye4(), V0};
  for (int i = 0; i < n; ++i) a[i + 1] = {inv4(f[i]), scalev(c.S[i], qd[i])};
  std::vector<AdAff> P = run_scan<AdAff>(order, a, comb);
  for (int i = 0; i < n; ++i) o.V[i] = P[i + 1].xi;
  // line 3: acceleration scan, operands (f^{-1}, S qdd + ad_{V_i}(S qd)), seed (I, Vdot_0).
  // (-ad_{S qd} Ad V_{i-1} = -ad_{S qd}(V_i - S qd) = ad_{V_i}(S qd), Eq. (1).)
  a[0] = {eye4(), Vd0};
  for (int i = 0; i < n; ++i)
    a[i + 1] = {inv4(f[i]), addv(scalev(c.S[i], qdd[i]), mv6(ad(o.V[i]), scalev(c.S[i], qd[i])))};
  P = run_scan<AdAff>(order, a, comb);
  for (int i = 0; i < n; ++i) o.Vd[i] = P[i + 1].xi;
  // bias forces in parallel.
  for (int i = 0; i < n; ++i) o.Fhat[i] = bias_force(c.J[i], o.V[i], o.Vd[i]);
  force_scan_and_torque(c, f, Ftip, order, o);    // lines 4-5
  return o;
}

// Fused variant: ONE forward scan of the Eq. (13) operands (f^{-1}, S qdd, S qd)
// with seed A_0 = (I, Vdot_0, V_0) (Eq. 12; isomorphism remark P:213),
// then bias forces, the backward scan and the torque map as above.
IdOut rnea_scan_fused(const Chain& c, const double* q, const double* qd, const double* qdd,
                      const V6& V0, const V6& Vd0, const V6& Ftip, int order) {
  const int n = c.n;
  IdOut o;
  o.tau.assign(n, 0.0); o.V.assign(n, zv6()); o.Vd.assign(n, zv6());
  o.F.assign(n, zv6()); o.Fhat.assign(n, zv6());
  std::vector<M4> f = calc_transform(c, q);
  std::vector<VelAcc> a(n + 1);
  a[0] = {eye4(), Vd0, V0};
  for (int i = 0; i < n; ++i) a[i + 1] = {inv4(f[i]), scalev(c.S[i], qdd[i]), scalev(c.S[i], qd[i])};
  std::function<VelAcc(const VelAcc&, const VelAcc&)> comb =
      [](const VelAcc& earlier, const VelAcc& later) { return velacc_oplus(later, earlier); };
  std::vector<VelAcc> P = run_scan<VelAcc>(order, a, comb);
  for (int i = 0; i < n; ++i) { o.V[i] = P[i + 1].xi2; o.Vd[i] = P[i + 1].xi1; }
  for (int i = 0; i < n; ++i) o.Fhat[i] = bias_force(c.J[i], o.V[i], o.Vd[i]);
  force_scan_and_torque(c, f, Ftip, order, o);
  return o;
}

// Dense-lift variant: the literal 13x13 matrices of Eq. (12) multiplied in
// sequence, and the literal 8x8 matrices of Eq. (16) (state (F_i, tau_{i+1}, 1))
// with the boundary read as F_{n+1} = tip wrench, S_{n+1} := 0, f_{n,n+1} := I (A5).
typedef std::vector<double> Dense;
Dense dmul(const Dense& A, const Dense& B, int d) {
  Dense C(d * d, 0.0);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double s = 0;
      for (int k = 0; k < d; ++k) s += A[d * i + k] * B[d * k + j];
      C[d * i + j] = s;
    }
  return C;
}
IdOut rnea_scan_lift(const Chain& c, const double* q, const double* qd, const double* qdd,
                     const V6& V0, const V6& Vd0, const V6& Ftip) {
  const int n = c.n;
  IdOut o;
  o.tau.assign(n, 0.0); o.V.assign(n, zv6()); o.Vd.assign(n, zv6());
  o.F.assign(n, zv6()); o.Fhat.assign(n, zv6());
  std::vector<M4> f = calc_transform(c, q);
  Dense A0(169, 0.0);
  for (int i = 0; i < 13; ++i) A0[14 * i] = 1.0;
  for (int i = 0; i < 6; ++i) { A0[13 * i + 12] = Vd0[i]; A0[13 * (6 + i) + 12] = V0[i]; }
  Dense P = A0;
  for (int i = 0; i < n; ++i) {
    Dense Ai(169);
    velacc_lift13({inv4(f[i]), scalev(c.S[i], qdd[i]), scalev(c.S[i], qd[i])}, Ai.data());
    P = dmul(Ai, P, 13);                          // x_i = A_i x_{i-1}
    for (int k = 0; k < 6; ++k) { o.Vd[i][k] = P[13 * k + 12]; o.V[i][k] = P[13 * (6 + k) + 12]; }
  }
  for (int i = 0; i < n; ++i) o.Fhat[i] = bias_force(c.J[i], o.V[i], o.Vd[i]);
  // Eq. (16): (F_i, tau_{i+1}, 1) = A_i (F_{i+1}, tau_{i+2}, 1), i = n..1.
  Dense Q(64, 0.0);
  for (int k = 0; k < 8; ++k) Q[9 * k] = 1.0;
  for (int k = 0; k < 6; ++k) Q[8 * k + 7] = Ftip[k];           // seed (F_{n+1}, tau_{n+2}=0, 1)
  std::vector<double> tau_lag(n + 2, 0.0);
  for (int i = n - 1; i >= 0; --i) {
    Dense Ai(64, 0.0);
    M6 L = (i == n - 1) ? eye6() : tr6(Ad(inv4(f[i + 1])));
    for (int r = 0; r < 6; ++r) {
      for (int s = 0; s < 6; ++s) Ai[8 * r + s] = L[r][s];
      Ai[8 * r + 7] = o.Fhat[i][r];
    }
    if (i < n - 1) for (int s = 0; s < 6; ++s) Ai[8 * 6 + s] = c.S[i + 1][s];   // S_{i+1}^T row
    Ai[63] = 1.0;
    Q = dmul(Ai, Q, 8);
    for (int k = 0; k < 6; ++k) o.F[i][k] = Q[8 * k + 7];
    tau_lag[i + 1] = Q[8 * 6 + 7];                                  // tau_{i+1} (paper index i+2)
  }
  // The lagged row yields tau_2..tau_n; tau_1 = S_1^T F_1 closes the scan (A5).
  for (int i = 1; i < n; ++i) o.tau[i] = tau_lag[i];
  o.tau[0] = dot6(c.S[0], o.F[0]);
  return o;
}

// Synchronous forward scan of Eq. (15): x_i = A_i x_{i-1} on the
// 28-vector x = (Vdot, Q, V, Fhat, 1), Q = (w x v, w1^2, w1w2, w1w3, w2^2, w2w3, w3^2)
// (P:218).  The paper prints only the block pattern; the starred blocks (reading
// A6) follow from Eq. (1) and P:217 for f = f_{i-1,i} = (R, p), s = S_i qd_i,
// a = S_i qdd_i, X = Ad_{f^-1}:
//   V'    = X V + s
//   Vdot' = X Vdot + a + ad_{V'} s = X Vdot - ad_s X V + a            (ad_s s = 0)
//   w' = R^T w + s_w,  v' = R^T (v + w x p) + s_v, so
//   w' x v' = R^T (w x v) + R^T (w x (w x p)) + [s_w] R^T v
//             + (-[s_v] R^T - [s_w] R^T [p]) w + s_w x s_v
//   w'_a w'_b = (R^T w)_a (R^T w)_b + (R^T w)_a s_w,b + s_w,a (R^T w)_b + s_w,a s_w,b
//   Fhat' = J Vdot' - ad^T_{V'} J V' = J Vdot' + H Q(V'),
//   H Q = (m (w x v) + w x (w x h),  h x (w x v) + w x (I_o w))   (J = [[m, -[h]], [[h], I_o]])
// (the 9-of-21 claim of P:218).  Every quadratic term is a fixed linear map of
// the ww entries, so A_i is affine with the printed zero blocks (pinned against a
// least-squares fit and against the recursion in tests/).  F_0 = 0 is
// read as: the Fhat entry of the seed is unused (no row reads it).
namespace eq15 {
constexpr int Vd = 0, Q = 6, V = 15, F = 21, ONE = 27, D = 28;
int widx(int j, int k) {                    // position of w_j w_k among (11, 12, 13, 22, 23, 33)
  if (j > k) std::swap(j, k);
  static const int tab[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
  return tab[j][k];
}
// coefficients of w x (w x x) on the ww entries: w (w.x) - x |w|^2
void G(const V3& x, double out[3][6]) {
  for (int k = 0; k < 3; ++k) for (int e = 0; e < 6; ++e) out[k][e] = 0;
  for (int k = 0; k < 3; ++k)
    for (int j = 0; j < 3; ++j) {
      out[k][widx(k, j)] += x[j];
      out[k][widx(j, j)] -= x[k];
    }
}
double eps(int a, int b, int c) { return (double)((a - b) * (b - c) * (c - a)) / 2.0; }   // Levi-Civita
}  // namespace eq15

Dense eq15_operator(const M4& f, const V6& s, const V6& a, const M6& J) {
  using namespace eq15;
  Dense A(D * D, 0.0);
  const M6 X = Ad(inv4(f));
  M3 Rt{}, P{};
  V3 p{}, sv{}, sw{};
  for (int i = 0; i < 3; ++i) {
    p[i] = f[i][3];
    sv[i] = s[i];
    sw[i] = s[3 + i];
    for (int j = 0; j < 3; ++j) Rt[i][j] = f[j][i];
  }
  P = skew(p);
  const M3 Ssv = skew(sv), Ssw = skew(sw);
  // V' = X V + s
  for (int r = 0; r < 6; ++r) {
    for (int c = 0; c < 6; ++c) A[D * (V + r) + V + c] = X[r][c];
    A[D * (V + r) + ONE] = s[r];
  }
  // Vdot' = X Vdot - ad_s X V + a
  const M6 adsX = mul6(ad(s), X);
  for (int r = 0; r < 6; ++r) {
    for (int c = 0; c < 6; ++c) {
      A[D * (Vd + r) + Vd + c] = X[r][c];
      A[D * (Vd + r) + V + c] = -adsX[r][c];
    }
    A[D * (Vd + r) + ONE] = a[r];
  }
  // Q'[0:3] = w' x v'
  double Gp[3][6];
  G(p, Gp);
  const M3 SswRt = mul3(Ssw, Rt), SsvRt = mul3(Ssv, Rt), SswRtP = mul3(SswRt, P);
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) A[D * (Q + r) + Q + c] = Rt[r][c];                 // R^T (w x v)
    for (int e = 0; e < 6; ++e) {                                                   // R^T (w x (w x p))
      double acc = 0;
      for (int k = 0; k < 3; ++k) acc += Rt[r][k] * Gp[k][e];
      A[D * (Q + r) + Q + 3 + e] = acc;
    }
    for (int c = 0; c < 3; ++c) {
      A[D * (Q + r) + V + c] = SswRt[r][c];                                         // [s_w] R^T v
      A[D * (Q + r) + V + 3 + c] = -SsvRt[r][c] - SswRtP[r][c];                     // (-[s_v]R^T - [s_w]R^T[p]) w
    }
  }
  const V3 swxsv = {sw[1] * sv[2] - sw[2] * sv[1], sw[2] * sv[0] - sw[0] * sv[2], sw[0] * sv[1] - sw[1] * sv[0]};
  for (int r = 0; r < 3; ++r) A[D * (Q + r) + ONE] = swxsv[r];
  // Q'[3:9] = w'_a w'_b
  for (int a_ = 0; a_ < 3; ++a_)
    for (int b_ = a_; b_ < 3; ++b_) {
      const int row = Q + 3 + widx(a_, b_);
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) A[D * row + Q + 3 + widx(j, k)] += Rt[a_][j] * Rt[b_][k];
      for (int j = 0; j < 3; ++j) A[D * row + V + 3 + j] = Rt[a_][j] * sw[b_] + sw[a_] * Rt[b_][j];
      A[D * row + ONE] = sw[a_] * sw[b_];
    }
  // H: Q -> -ad^T_V J V
  const double m = J[0][0];
  const V3 h = {J[5][1], J[3][2], J[4][0]};
  M3 Io{};
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) Io[i][j] = J[3 + i][3 + j];
  double H[6][9] = {};
  double Gh[3][6];
  G(h, Gh);
  const M3 Sh = skew(h);
  for (int k = 0; k < 3; ++k) {
    H[k][k] = m;
    for (int e = 0; e < 6; ++e) H[k][3 + e] = Gh[k][e];
    for (int c = 0; c < 3; ++c) H[3 + k][c] = Sh[k][c];
    for (int a_ = 0; a_ < 3; ++a_)
      for (int b_ = 0; b_ < 3; ++b_)
        for (int c = 0; c < 3; ++c) H[3 + k][3 + widx(a_, c)] += eps(k, a_, b_) * Io[b_][c];
  }
  // Fhat' = J (Vdot' row) + H (Q' row)
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < D; ++c) {
      double acc = 0;
      for (int k = 0; k < 6; ++k) acc += J[r][k] * A[D * (Vd + k) + c];
      for (int k = 0; k < 9; ++k) acc += H[r][k] * A[D * (Q + k) + c];
      A[D * (F + r) + c] = acc;
    }
  A[D * ONE + ONE] = 1.0;
  return A;
}

IdOut rnea_scan_sync15(const Chain& c, const double* q, const double* qd, const double* qdd,
                       const V6& V0, const V6& Vd0, const V6& Ftip, int order) {
  using namespace eq15;
  const int n = c.n;
  IdOut o;
  o.tau.assign(n, 0.0); o.V.assign(n, zv6()); o.Vd.assign(n, zv6());
  o.F.assign(n, zv6()); o.Fhat.assign(n, zv6());
  std::vector<M4> f = calc_transform(c, q);
  // seed: constant map to x_0 = (Vdot_0, Q(V_0), V_0, 0, 1)
  Dense seed(D * D, 0.0);
  {
    double x0[D] = {};
    for (int k = 0; k < 6; ++k) { x0[Vd + k] = Vd0[k]; x0[V + k] = V0[k]; }
    const double v[3] = {V0[0], V0[1], V0[2]}, w[3] = {V0[3], V0[4], V0[5]};
    x0[Q + 0] = w[1] * v[2] - w[2] * v[1];
    x0[Q + 1] = w[2] * v[0] - w[0] * v[2];
    x0[Q + 2] = w[0] * v[1] - w[1] * v[0];
    for (int a_ = 0; a_ < 3; ++a_)
      for (int b_ = a_; b_ < 3; ++b_) x0[Q + 3 + widx(a_, b_)] = w[a_] * w[b_];
    x0[ONE] = 1.0;
    for (int r = 0; r < D; ++r) seed[D * r + ONE] = x0[r];
  }
  std::vector<Dense> a;
  a.push_back(seed);
  for (int i = 0; i < n; ++i) a.push_back(eq15_operator(f[i], scalev(c.S[i], qd[i]), scalev(c.S[i], qdd[i]), c.J[i]));
  std::function<Dense(const Dense&, const Dense&)> comb =
      [](const Dense& earlier, const Dense& later) { return dmul(later, earlier, D); };
  std::vector<Dense> P = run_scan<Dense>(order, a, comb);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < 6; ++k) {
      o.Vd[i][k] = P[i + 1][D * (Vd + k) + ONE];
      o.V[i][k] = P[i + 1][D * (V + k) + ONE];
      o.Fhat[i][k] = P[i + 1][D * (F + k) + ONE];
    }
  force_scan_and_torque(c, f, Ftip, order, o);
  return o;
}

// --------------------------------------------- forward dynamics, Eq. (4)-(8)
V6 gravity_vd0(const double* g) { V6 a = zv6(); a[0] = -g[0]; a[1] = -g[1]; a[2] = -g[2]; return a; }

// Joint-space inertia column by column, Eq. (17):
// M_{.,j} = ID(q, 0, delta_{.,j}, 0, 0, 0).
std::vector<double> jsi(const Chain& c, const double* q) {
  const int n = c.n;
  std::vector<double> M(n * n, 0.0), zero(n, 0.0), e(n, 0.0);
  for (int j = 0; j < n; ++j) {
    std::fill(e.begin(), e.end(), 0.0);
    e[j] = 1.0;
    IdOut o = rnea(c, q, zero.data(), e.data(), zv6(), zv6(), zv6());
    for (int i = 0; i < n; ++i) M[n * i + j] = o.tau[i];
  }
  return M;
}

// Textbook Cholesky M = L L^T and two triangular solves (the SPD solve the
// paper points to; no explicit inverse).  Throws if not SPD.
std::vector<double> chol_solve(std::vector<double> M, const std::vector<double>& rhs, int n) {
  std::vector<double> L(n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = M[n * j + j];
    for (int k = 0; k < j; ++k) d -= L[n * j + k] * L[n * j + k];
    if (!(d > 0.0)) throw std::runtime_error("jsiia: M(q) not positive definite at pivot " + std::to_string(j));
    L[n * j + j] = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double s = M[n * i + j];
      for (int k = 0; k < j; ++k) s -= L[n * i + k] * L[n * j + k];
      L[n * i + j] = s / L[n * j + j];
    }
  }
  std::vector<double> y(n), x(n);
  for (int i = 0; i < n; ++i) {
    double s = rhs[i];
    for (int k = 0; k < i; ++k) s -= L[n * i + k] * y[k];
    y[i] = s / L[n * i + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < n; ++k) s -= L[n * k + i] * x[k];
    x[i] = s / L[n * i + i];
  }
  return x;
}

// JSIIA, Alg. 2: tau_bias (Eq. 5), M by Eq. (17), qdd = M^{-1}(tau - tau_bias) (Eq. 6).
std::vector<double> fd_jsiia(const Chain& c, const double* q, const double* qd, const double* tau,
                             const V6& V0, const V6& Vd0, const V6& Ftip) {
  const int n = c.n;
  std::vector<double> zero(n, 0.0);
  IdOut bias = rnea(c, q, qd, zero.data(), V0, Vd0, Ftip);
  std::vector<double> M = jsi(c, q), rhs(n);
  for (int i = 0; i < n; ++i) rhs[i] = tau[i] - bias.tau[i];
  return chol_solve(M, rhs, n);
}

// ABI recursion, Eq. (7), i = n..1, with Jhat_n = J_n (A9) and
// explicit re-symmetrisation (A10).  Omega_{i+1} <= eps throws (A11).
std::vector<M6> abi(const Chain& c, const std::vector<M4>& f) {
  const int n = c.n;
  std::vector<M6> Jh(n);
  Jh[n - 1] = c.J[n - 1];
  for (int i = n - 2; i >= 0; --i) {
    M6 X = Ad(inv4(f[i + 1]));                  // Ad_{f_{i,i+1}^{-1}}
    M6 XT = tr6(X);
    V6 JS = mv6(Jh[i + 1], c.S[i + 1]);
    double Om = dot6(c.S[i + 1], JS);
    if (!(Om > 1e-12)) throw std::runtime_error("abi: Omega not positive at link " + std::to_string(i + 2));
    M6 T1 = mul6(mul6(XT, Jh[i + 1]), X);
    M6 T2 = scale6(mul6(mul6(XT, outer6(JS, JS)), X), 1.0 / Om);
    M6 R = sub6(add6(c.J[i], T1), T2);
    Jh[i] = scale6(add6(R, tr6(R)), 0.5);
  }
  return Jh;
}

// Hybrid ABIA, Alg. 3 in the recursive form of Eq. (8):
// tau_hat = tau - tau_bias; ABI; Omega, Pi, Y; backward zhat/c/chat; forward lambda/qdd.
// Boundaries: zhat_{n+1} = 0 with Y_{n,n+1} = Pi_{n,n+1} = 0; lambda_0 = 0 (A9).
std::vector<double> fd_aba(const Chain& c, const double* q, const double* qd, const double* tau,
                           const V6& V0, const V6& Vd0, const V6& Ftip, std::vector<M6>* Jhat_out) {
  const int n = c.n;
  std::vector<double> zero(n, 0.0);
  IdOut bias = rnea(c, q, qd, zero.data(), V0, Vd0, Ftip);            // line 1
  std::vector<double> th(n);
  for (int i = 0; i < n; ++i) th[i] = tau[i] - bias.tau[i];           // line 2
  std::vector<M4> f = calc_transform(c, q);
  std::vector<M6> Jh = abi(c, f);                                      // line 3
  if (Jhat_out) *Jhat_out = Jh;
  // line 4: Omega_i = S_i^T Jhat_i S_i; Y_{i-1,i}, Pi_{i-1,i} stored at index i (link i).
  std::vector<double> Om(n);
  std::vector<M6> Y(n);
  std::vector<V6> Pi(n);
  for (int i = 0; i < n; ++i) {
    V6 JS = mv6(Jh[i], c.S[i]);
    Om[i] = dot6(c.S[i], JS);
    if (!(Om[i] > 1e-12)) throw std::runtime_error("aba: Omega not positive at link " + std::to_string(i + 1));
    M6 XT = tr6(Ad(inv4(f[i])));                 // Ad^T_{f_{i-1,i}^{-1}}
    Y[i] = mul6(XT, sub6(eye6(), scale6(outer6(JS, c.S[i]), 1.0 / Om[i])));
    Pi[i] = scalev(mv6(XT, JS), 1.0 / Om[i]);
  }
  // lines 5-6: backward zhat_i = Y_{i,i+1} zhat_{i+1} + Pi_{i,i+1} tau_hat_{i+1}; chat.
  std::vector<V6> zh(n);
  std::vector<double> ch(n);
  V6 znext = zv6();
  for (int i = n - 1; i >= 0; --i) {
    if (i == n - 1) zh[i] = zv6();
    else zh[i] = addv(mv6(Y[i + 1], znext), scalev(Pi[i + 1], th[i + 1]));
    double ci = th[i] - dot6(c.S[i], zh[i]);
    ch[i] = ci / Om[i];
    znext = zh[i];
  }
  // lines 7-8: forward lambda_i = Y^T_{i-1,i} lambda_{i-1} + S_i chat_i; qdd_i = chat_i - Pi^T lambda_{i-1}.
  std::vector<double> qdd(n);
  V6 lam = zv6();
  for (int i = 0; i < n; ++i) {
    qdd[i] = ch[i] - dot6(Pi[i], lam);
    lam = addv(mv6(tr6(Y[i]), lam), scalev(c.S[i], ch[i]));
  }
  return qdd;
}

// ABIA with the two linear phases as scans of the 8x8 operands of Eq. (18)
// (with the Omega^{-1} reading A7) and Eq. (19).
std::vector<double> fd_aba_scan(const Chain& c, const double* q, const double* qd, const double* tau,
                                const V6& V0, const V6& Vd0, const V6& Ftip, int order) {
  const int n = c.n;
  std::vector<double> zero(n, 0.0);
  IdOut bias = rnea(c, q, qd, zero.data(), V0, Vd0, Ftip);
  std::vector<double> th(n);
  for (int i = 0; i < n; ++i) th[i] = tau[i] - bias.tau[i];
  std::vector<M4> f = calc_transform(c, q);
  std::vector<M6> Jh = abi(c, f);
  std::vector<double> Om(n);
  std::vector<M6> Y(n);
  std::vector<V6> Pi(n);
  for (int i = 0; i < n; ++i) {
    V6 JS = mv6(Jh[i], c.S[i]);
    Om[i] = dot6(c.S[i], JS);
    M6 XT = tr6(Ad(inv4(f[i])));
    Y[i] = mul6(XT, sub6(eye6(), scale6(outer6(JS, c.S[i]), 1.0 / Om[i])));
    Pi[i] = scalev(mv6(XT, JS), 1.0 / Om[i]);
  }
  std::function<Dense(const Dense&, const Dense&)> comb =
      [](const Dense& earlier, const Dense& later) { return dmul(later, earlier, 8); };
  // Eq. (18): (zhat_i, chat_{i+1}, 1) = A_i (zhat_{i+1}, chat_{i+2}, 1), i = n..0,
  // A_i = [[Y_{i,i+1}, 0, Pi_{i,i+1} th_{i+1}], [-S_{i+1}^T/Omega_{i+1}, 0, th_{i+1}/Omega_{i+1}], [0,0,1]],
  // out-of-range (i = n) entries zero; seed zhat_{n+1} = chat_{n+1} = chat_{n+2} = 0.
  std::vector<Dense> a;
  {
    Dense seed(64, 0.0); seed[63] = 1.0;       // constant map to (0, 0, 1)
    a.push_back(seed);
  }
  for (int i = n; i >= 0; --i) {                // paper index i; link i+1 is 0-based index i
    Dense A(64, 0.0);
    if (i < n) {
      for (int r = 0; r < 6; ++r) {
        for (int s = 0; s < 6; ++s) A[8 * r + s] = Y[i][r][s];
        A[8 * r + 7] = Pi[i][r] * th[i];
      }
      for (int s = 0; s < 6; ++s) A[8 * 6 + s] = -c.S[i][s] / Om[i];
      A[8 * 6 + 7] = th[i] / Om[i];
    }
    A[63] = 1.0;
    a.push_back(A);
  }
  std::vector<Dense> P = run_scan<Dense>(order, a, comb);
  std::vector<double> ch(n);
  for (int i = 0; i < n; ++i) ch[i] = P[1 + (n - i)][8 * 6 + 7];   // chat_{i+1} from A_i's output
  // Eq. (19): (lambda_i, qdd_i, 1) = [[Y^T_{i-1,i}, 0, S_i chat_i], [-Pi^T_{i-1,i}, 0, chat_i], [0,0,1]] (...), lambda_0 = qdd_0 = 0.
  std::vector<Dense> b;
  {
    Dense seed(64, 0.0); seed[63] = 1.0;
    b.push_back(seed);
  }
  for (int i = 0; i < n; ++i) {
    Dense A(64, 0.0);
    for (int r = 0; r < 6; ++r) {
      for (int s = 0; s < 6; ++s) A[8 * r + s] = Y[i][s][r];
      A[8 * r + 7] = c.S[i][r] * ch[i];
    }
    for (int s = 0; s < 6; ++s) A[8 * 6 + s] = -Pi[i][s];
    A[8 * 6 + 7] = ch[i];
    A[63] = 1.0;
    b.push_back(A);
  }
  std::vector<Dense> Q = run_scan<Dense>(order, b, comb);
  std::vector<double> qdd(n);
  for (int i = 0; i < n; ++i) qdd[i] = Q[i + 1][8 * 6 + 7];
  return qdd;
}

// ABIA with the MERGED backward scan of Eq. (20): one scan of the
// 15x15 operators acting on x_i = (F_{i-1}, tau_hat_i, zhat_i, chat_{i+1}, 1),
//   A_i = [[Ad^T_{f_{i-1,i}^{-1}}, 0, 0, 0, Fhat_{i-1}],
//          [-S_i^T, 0, 0, 0, tau_in_i],
//          [0, Pi_{i,i+1}, Y_{i,i+1}, 0, 0],
//          [0, Omega_{i+1}^{-1}, -Omega_{i+1}^{-1} S_{i+1}^T, 0, 0],     (A7: Omega^{-1})
//          [0, 0, 0, 0, 1]],
// where F / Fhat are the bias-force recursion of tau_bias (qdd = 0, Eq. 5), so
// tau_hat_i = tau_in_i - S_i^T F_i.  Seed (A8): (F_n, 0, 0, 0, 1) with
// F_n = Fhat_n + F_{n+1}; operators for paper index i = n..0 with out-of-range
// S, Omega^{-1}, Pi, Y, Fhat := 0 (and f_{-1,0} := I).  chat_{i+1} is read from
// x_i; then the Eq. (19) forward scan gives qdd.
std::vector<double> fd_aba_merged(const Chain& c, const double* q, const double* qd, const double* tau,
                                  const V6& V0, const V6& Vd0, const V6& Ftip, int order) {
  const int n = c.n;
  std::vector<double> zero(n, 0.0);
  IdOut bias = rnea(c, q, qd, zero.data(), V0, Vd0, Ftip);      // Fhat of the qdd = 0 recursion
  std::vector<M4> f = calc_transform(c, q);
  std::vector<M6> Jh = abi(c, f);
  std::vector<double> Om(n);
  std::vector<M6> Y(n);
  std::vector<V6> Pi(n);
  for (int i = 0; i < n; ++i) {
    V6 JS = mv6(Jh[i], c.S[i]);
    Om[i] = dot6(c.S[i], JS);
    M6 XT = tr6(Ad(inv4(f[i])));
    Y[i] = mul6(XT, sub6(eye6(), scale6(outer6(JS, c.S[i]), 1.0 / Om[i])));
    Pi[i] = scalev(mv6(XT, JS), 1.0 / Om[i]);
  }
  const int D = 15;
  std::function<Dense(const Dense&, const Dense&)> comb =
      [](const Dense& earlier, const Dense& later) { return dmul(later, earlier, 15); };
  std::vector<Dense> a;
  {
    Dense seed(D * D, 0.0);
    V6 Fn = addv(bias.Fhat[n - 1], Ftip);
    for (int r = 0; r < 6; ++r) seed[D * r + 14] = Fn[r];
    seed[D * 14 + 14] = 1.0;                        // constant map to (F_n, 0, 0, 0, 1)
    a.push_back(seed);
  }
  // paper index i = n..0; 0-based link of paper i is i-1.
  for (int i = n; i >= 0; --i) {
    Dense A(D * D, 0.0);
    const int li = i - 1;                           // link i (0-based), valid if 0 <= li < n
    const int ln = i;                               // link i+1 (0-based), valid if < n
    // row block F_{i-1} = Ad^T_{f_{i-1,i}^{-1}} F_i + Fhat_{i-1}
    if (li >= 0) {
      M6 L = tr6(Ad(inv4(f[li])));
      for (int r = 0; r < 6; ++r)
        for (int s2 = 0; s2 < 6; ++s2) A[D * r + s2] = L[r][s2];
    } else {
      for (int r = 0; r < 6; ++r) A[D * r + r] = 1.0;            // f_{-1,0} := I (row unused)
    }
    if (li - 1 >= 0) for (int r = 0; r < 6; ++r) A[D * r + 14] = bias.Fhat[li - 1][r];
    // row tau_hat_i = tau_in_i - S_i^T F_i
    if (li >= 0) {
      for (int s2 = 0; s2 < 6; ++s2) A[D * 6 + s2] = -c.S[li][s2];
      A[D * 6 + 14] = tau[li];
    }
    // row block zhat_i = Pi_{i,i+1} tau_hat_{i+1} + Y_{i,i+1} zhat_{i+1}; row chat_{i+1}
    if (ln < n) {
      for (int r = 0; r < 6; ++r) {
        A[D * (7 + r) + 6] = Pi[ln][r];
        for (int s2 = 0; s2 < 6; ++s2) A[D * (7 + r) + 7 + s2] = Y[ln][r][s2];
      }
      A[D * 13 + 6] = 1.0 / Om[ln];
      for (int s2 = 0; s2 < 6; ++s2) A[D * 13 + 7 + s2] = -c.S[ln][s2] / Om[ln];
    }
    A[D * 14 + 14] = 1.0;
    a.push_back(A);
  }
  std::vector<Dense> P = run_scan<Dense>(order, a, comb);
  std::vector<double> ch(n);
  for (int i = 0; i <= n - 1; ++i) ch[i] = P[1 + (n - i)][D * 13 + 14];   // x_i holds chat_{i+1} (0-based link i)
  // Eq. (19) forward scan, as in fd_aba_scan
  std::function<Dense(const Dense&, const Dense&)> comb8 =
      [](const Dense& earlier, const Dense& later) { return dmul(later, earlier, 8); };
  std::vector<Dense> b;
  {
    Dense seed(64, 0.0); seed[63] = 1.0;
    b.push_back(seed);
  }
  for (int i = 0; i < n; ++i) {
    Dense A(64, 0.0);
    for (int r = 0; r < 6; ++r) {
      for (int s2 = 0; s2 < 6; ++s2) A[8 * r + s2] = Y[i][s2][r];
      A[8 * r + 7] = c.S[i][r] * ch[i];
    }
    for (int s2 = 0; s2 < 6; ++s2) A[8 * 6 + s2] = -Pi[i][s2];
    A[8 * 6 + 7] = ch[i];
    A[63] = 1.0;
    b.push_back(A);
  }
  std::vector<Dense> Q = run_scan<Dense>(order, b, comb8);
  std::vector<double> qdd(n);
  for (int i = 0; i < n; ++i) qdd[i] = Q[i + 1][8 * 6 + 7];
  return qdd;
}

thread_local std::string g_err;

template <class Fn>
int guarded(Fn fn) {
  try { fn(); return 0; }
  catch (const std::exception& e) { g_err = e.what(); return 1; }
}

void parallel_for(int64_t B, int nthreads, const std::function<void(int64_t, int64_t)>& body) {
  if (nthreads <= 1 || B < 2) { body(0, B); return; }
  std::vector<std::thread> th;
  int64_t chunk = (B + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    int64_t b0 = t * chunk, b1 = std::min<int64_t>(B, b0 + chunk);
    if (b0 >= b1) break;
    th.emplace_back(body, b0, b1);
  }
  for (auto& x : th) x.join();
}

}  // namespace

// =============================================================== C entry points
extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

void orc_exp_twist(const double* S, double q, double* g) { store4(exp_twist(loadv(S), q), g); }
void orc_Ad(const double* g, double* out) { store6(Ad(load4(g)), out); }
void orc_ad(const double* xi, double* out) { store6(ad(loadv(xi)), out); }
void orc_inv(const double* g, double* out) { store4(inv4(load4(g)), out); }

// VelAcc element layout: g[16] (row-major 4x4), xi1[6], xi2[6] -> 28 doubles.
static VelAcc load_va(const double* p) { return {load4(p), loadv(p + 16), loadv(p + 22)}; }
static void store_va(const VelAcc& a, double* p) { store4(a.g, p); storev(a.xi1, p + 16); storev(a.xi2, p + 22); }
void orc_velacc_oplus(const double* a, const double* b, double* out) { store_va(velacc_oplus(load_va(a), load_va(b)), out); }
void orc_velacc_inverse(const double* a, double* out) { store_va(velacc_inverse(load_va(a)), out); }
void orc_velacc_lift13(const double* a, double* out) { velacc_lift13(load_va(a), out); }

// Single-state RNEA (Eq. 1-2) with the full signature of Eq. (3).
// variant: 0 serial recursion; 1 Alg. 1 split scans; 2 fused Eq. (13) scan;
// 3 dense lifts Eq. (12)/(16); 4 synchronous Eq. (15) scan.  order: 0 sequential fold, 1 Kogge-Stone.
// Optional outputs (may be NULL): V, Vd, F, Fhat as [n][6].
int orc_rnea(int n, const double* M, const double* S, const double* J,
             const double* q, const double* qd, const double* qdd,
             const double* V0, const double* Vd0, const double* Ftip,
             int variant, int order,
             double* tau, double* V, double* Vd, double* F, double* Fhat) {
  return guarded([&] {
    if (n < 1) throw std::runtime_error("n < 1");
    Chain c = make_chain(n, M, S, J);
    V6 v0 = loadv(V0), vd0 = loadv(Vd0), ft = loadv(Ftip);
    IdOut o;
    if (variant == 0) o = rnea(c, q, qd, qdd, v0, vd0, ft);
    else if (variant == 1) o = rnea_scan_split(c, q, qd, qdd, v0, vd0, ft, order);
    else if (variant == 2) o = rnea_scan_fused(c, q, qd, qdd, v0, vd0, ft, order);
    else if (variant == 3) o = rnea_scan_lift(c, q, qd, qdd, v0, vd0, ft);
    else if (variant == 4) o = rnea_scan_sync15(c, q, qd, qdd, v0, vd0, ft, order);
    else throw std::runtime_error("unknown variant");
    for (int i = 0; i < n; ++i) {
      tau[i] = o.tau[i];
      if (V) storev(o.V[i], V + 6 * i);
      if (Vd) storev(o.Vd[i], Vd + 6 * i);
      if (F) storev(o.F[i], F + 6 * i);
      if (Fhat) storev(o.Fhat[i], Fhat + 6 * i);
    }
  });
}

// The 28x28 operator A_i of Eq. (15) for ONE link (n = 1 chain) at (q, qd, qdd).
int orc_eq15_operator(const double* M, const double* S, const double* J, double q, double qd, double qdd,
                      double* out) {
  return guarded([&] {
    Chain c = make_chain(1, M, S, J);
    std::vector<M4> f = calc_transform(c, &q);
    Dense A = eq15_operator(f[0], scalev(c.S[0], qd), scalev(c.S[0], qdd), c.J[0]);
    for (int i = 0; i < 28 * 28; ++i) out[i] = A[i];
  });
}

// Joint-space inertia M(q) by Eq. (17), row-major n x n.
int orc_jsi(int n, const double* M, const double* S, const double* J, const double* q, double* Mq) {
  return guarded([&] {
    Chain c = make_chain(n, M, S, J);
    std::vector<double> m = jsi(c, q);
    std::memcpy(Mq, m.data(), sizeof(double) * n * n);
  });
}

// Forward dynamics qdd = FD(q, qd, tau, V_0, Vdot_0, F_{n+1}) (Eq. 4).
// algo: 0 ABIA recursive Eq. (7)-(8); 1 JSIIA Alg. 2; 2 ABIA with Eq. (18)/(19) scans;
// 3 ABIA with the merged Eq. (20) backward scan + Eq. (19).
// Jhat (optional, [n][6][6]) receives the ABI of Eq. (7) for algo 0.
int orc_fd(int n, const double* M, const double* S, const double* J,
           const double* q, const double* qd, const double* tau,
           const double* V0, const double* Vd0, const double* Ftip,
           int algo, int order, double* qdd, double* Jhat) {
  return guarded([&] {
    if (n < 1) throw std::runtime_error("n < 1");
    Chain c = make_chain(n, M, S, J);
    V6 v0 = loadv(V0), vd0 = loadv(Vd0), ft = loadv(Ftip);
    std::vector<double> r;
    std::vector<M6> Jh;
    if (algo == 0) r = fd_aba(c, q, qd, tau, v0, vd0, ft, &Jh);
    else if (algo == 1) r = fd_jsiia(c, q, qd, tau, v0, vd0, ft);
    else if (algo == 2) r = fd_aba_scan(c, q, qd, tau, v0, vd0, ft, order);
    else if (algo == 3) r = fd_aba_merged(c, q, qd, tau, v0, vd0, ft, order);
    else throw std::runtime_error("unknown algo");
    std::memcpy(qdd, r.data(), sizeof(double) * n);
    if (Jhat && algo == 0) for (int i = 0; i < n; ++i) store6(Jh[i], Jhat + 36 * i);
  });
}

// Batched ID over B independent states ("one thread per independent
// dynamics computation" -> here a pool of nthreads host threads over a static
// partition).  Gravity form: V_0 = 0, Vdot_0 = (-g, 0), F_{n+1} = 0 (A3).
// q/qd/qdd/tau are link-major [n][B].
int orc_rnea_batch(int n, const double* M, const double* S, const double* J, const double* g,
                   int64_t B, const double* q, const double* qd, const double* qdd,
                   double* tau, int nthreads) {
  return guarded([&] {
    Chain c = make_chain(n, M, S, J);
    V6 vd0 = gravity_vd0(g);
    parallel_for(B, nthreads, [&](int64_t b0, int64_t b1) {
      std::vector<double> xq(n), xd(n), xa(n);
      for (int64_t b = b0; b < b1; ++b) {
        for (int i = 0; i < n; ++i) { xq[i] = q[i * B + b]; xd[i] = qd[i * B + b]; xa[i] = qdd[i * B + b]; }
        IdOut o = rnea(c, xq.data(), xd.data(), xa.data(), zv6(), vd0, zv6());
        for (int i = 0; i < n; ++i) tau[i * B + b] = o.tau[i];
      }
    });
  });
}

// Batched FD (gravity form), algo as in orc_fd.  A state whose ABI/Cholesky
// fails gets NaN outputs (mirrors the product's per-state NaN policy, A11).
int orc_fd_batch(int n, const double* M, const double* S, const double* J, const double* g,
                 int64_t B, const double* q, const double* qd, const double* tau,
                 double* qdd, int algo, int nthreads) {
  return guarded([&] {
    Chain c = make_chain(n, M, S, J);
    V6 vd0 = gravity_vd0(g);
    parallel_for(B, nthreads, [&](int64_t b0, int64_t b1) {
      std::vector<double> xq(n), xd(n), xt(n), r;
      for (int64_t b = b0; b < b1; ++b) {
        for (int i = 0; i < n; ++i) { xq[i] = q[i * B + b]; xd[i] = qd[i * B + b]; xt[i] = tau[i * B + b]; }
        try {
          if (algo == 1) r = fd_jsiia(c, xq.data(), xd.data(), xt.data(), zv6(), vd0, zv6());
          else r = fd_aba(c, xq.data(), xd.data(), xt.data(), zv6(), vd0, zv6(), nullptr);
        } catch (const std::exception&) {
          r.assign(n, NAN);
        }
        for (int i = 0; i < n; ++i) qdd[i * B + b] = r[i];
      }
    });
  });
}

}  // extern "C"
