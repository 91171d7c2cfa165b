"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every test here checks oracle/ against something other than itself: closed
forms, textbook definitions, an independent Lagrangian model (energy_ref.py),
library routines (scipy expm), semigroup laws and cross-algorithm identities.
No GPU needed (-m "not gpu").
"""
import os

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth
from energy_ref import (euler_lagrange_tau, power, kinetic, tip_body_velocity, hat, vee,
                        mass_matrix)

G = 9.81
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rand_twist(rng, kind="revolute"):
    w = rng.standard_normal(3)
    w /= np.linalg.norm(w)
    if kind == "prismatic":
        return np.concatenate([w, np.zeros(3)])
    r = rng.uniform(-1, 1, 3)
    v = np.cross(r, w)
    if kind == "screw":
        v = v + 0.3 * w
    return np.concatenate([v, w])


def rand_g(rng):
    g = np.eye(4)
    g[:3, :3] = synth.random_rotation(rng)
    g[:3, 3] = rng.uniform(-1, 1, 3)
    return g


def rand_va(rng):
    return rand_g(rng), rng.standard_normal(6), rng.standard_normal(6)


# ------------------------------------------------------------------ SE(3) pins
def test_exp_twist_golden_cases():
    # rotation about z by pi/2 (golden/exp_twist.txt), S:62 -- pure translation.
    data = np.loadtxt(os.path.join(GOLDEN, "exp_twist.txt"))
    for row in data:
        S, th, g = row[:6], row[6], row[7:].reshape(4, 4)
        np.testing.assert_allclose(oracle.exp_twist(S, th), g, atol=1e-15)


@pytest.mark.parametrize("kind", ["revolute", "prismatic", "screw"])
def test_exp_twist_matches_library_expm(rng, kind):
    # The closed form of P:63 must equal the matrix exponential (scipy Pade).
    for _ in range(50):
        S = rand_twist(rng, kind)
        th = rng.uniform(-4, 4)
        np.testing.assert_allclose(oracle.exp_twist(S, th), scipy.linalg.expm(hat(S) * th),
                                   atol=1e-12, rtol=0)


def test_exp_twist_one_parameter_group(rng):
    for _ in range(50):
        S = rand_twist(rng, "screw")
        a, b = rng.uniform(-3, 3, 2)
        np.testing.assert_allclose(oracle.exp_twist(S, a) @ oracle.exp_twist(S, b),
                                   oracle.exp_twist(S, a + b), atol=1e-14)


def test_Ad_is_conjugation(rng):
    # Definition of the Adjoint: hat(Ad_g xi) = g hat(xi) g^{-1} (fixes the (v, w) block layout, A1).
    for _ in range(100):
        g = rand_g(rng)
        xi = rng.standard_normal(6)
        lhs = oracle.Ad(g) @ xi
        rhs = vee(g @ hat(xi) @ np.linalg.inv(g))
        np.testing.assert_allclose(lhs, rhs, atol=1e-13)
        np.testing.assert_allclose(oracle.inv(g), np.linalg.inv(g), atol=1e-14)


def test_ad_is_matrix_bracket(rng):
    # Definition of ad: hat(ad_xi eta) = [hat(xi), hat(eta)].
    for _ in range(100):
        xi, eta = rng.standard_normal((2, 6))
        lhs = oracle.ad(xi) @ eta
        rhs = vee(hat(xi) @ hat(eta) - hat(eta) @ hat(xi))
        np.testing.assert_allclose(lhs, rhs, atol=1e-13)


def test_Ad_homomorphism_and_dual_pairing(rng):
    for _ in range(100):
        g, h = rand_g(rng), rand_g(rng)
        np.testing.assert_allclose(oracle.Ad(g @ h), oracle.Ad(g) @ oracle.Ad(h), atol=1e-13)
        F, V = rng.standard_normal((2, 6))
        assert abs((oracle.Ad(g).T @ F) @ V - F @ (oracle.Ad(g) @ V)) < 1e-12


# ------------------------------------------------------- semigroup (Eq. 12-14)
def va_close(a, b, tol):
    for x, y in zip(a, b):
        np.testing.assert_allclose(x, y, atol=tol * max(1.0, np.abs(y).max()))


def test_velacc_associativity(rng):
    for _ in range(1000):
        a, b, c = rand_va(rng), rand_va(rng), rand_va(rng)
        va_close(oracle.velacc_oplus(oracle.velacc_oplus(a, b), c),
                 oracle.velacc_oplus(a, oracle.velacc_oplus(b, c)), 1e-12)


def test_velacc_identity_and_inverse(rng):
    e = (np.eye(4), np.zeros(6), np.zeros(6))
    for _ in range(200):
        a = rand_va(rng)
        va_close(oracle.velacc_oplus(a, e), a, 1e-15)
        va_close(oracle.velacc_oplus(e, a), a, 1e-15)
        ai = oracle.velacc_inverse(a)                       # Eq. (14)
        va_close(oracle.velacc_oplus(a, ai), e, 1e-12)
        va_close(oracle.velacc_oplus(ai, a), e, 1e-12)


def test_velacc_lift_homomorphism(rng):
    # Phi(a (+) b) = Phi(a) Phi(b) for the 13x13 lift of Eq. (12) (A4).
    for _ in range(1000):
        a, b = rand_va(rng), rand_va(rng)
        lhs = oracle.velacc_lift13(oracle.velacc_oplus(a, b))
        rhs = oracle.velacc_lift13(a) @ oracle.velacc_lift13(b)
        np.testing.assert_allclose(lhs, rhs, atol=1e-12 * np.abs(rhs).max())


def test_velacc_is_not_commutative(rng):
    # The scans must preserve operand order; (+) is genuinely non-commutative.
    a, b = rand_va(rng), rand_va(rng)
    ab, ba = oracle.velacc_oplus(a, b), oracle.velacc_oplus(b, a)
    assert np.abs(ab[0] - ba[0]).max() > 1e-3


def test_lift_recursion_matches_eq1_rows(rng):
    # The lifted operand applied to (Vdot_{i-1}, V_{i-1}, 1) reproduces Eq. (1) rows,
    # computed here from hat/vee definitions (Ad_{f^-1} = conjugation).
    for _ in range(100):
        f = rand_g(rng)
        S = rand_twist(rng)
        qd, qdd = rng.standard_normal(2)
        Vp, Vdp = rng.standard_normal((2, 6))
        fi = np.linalg.inv(f)
        AdV = vee(fi @ hat(Vp) @ f)
        AdVd = vee(fi @ hat(Vdp) @ f)
        Sq = S * qd
        V = AdV + Sq
        Vd = S * qdd + AdVd - vee(hat(Sq) @ hat(AdV) - hat(AdV) @ hat(Sq))
        x = oracle.velacc_lift13((fi, S * qdd, Sq)) @ np.concatenate([Vdp, Vp, [1.0]])
        np.testing.assert_allclose(x[:6], Vd, atol=1e-12)
        np.testing.assert_allclose(x[6:12], V, atol=1e-12)


# ----------------------------------------------------------- RNEA closed forms
def test_zero_motion_zero_gravity_gives_zero():
    r = synth.random_chain(12, 5, prismatic_fraction=0.5)
    z = np.zeros(12)
    q = np.linspace(-2, 2, 12)
    assert np.all(oracle.rnea(r, q, z, z, g=[0, 0, 0]) == 0.0)


def test_pendulum_closed_form_golden():
    # tau = m l^2 qdd + m g l cos q  (point mass, axis z, gravity -y).
    data = np.loadtxt(os.path.join(GOLDEN, "pendulum.txt"))
    for m, l, q, qd, qdd, tau in data:
        r = synth.pendulum(m, l)
        t = oracle.rnea(r, [q], [qd], [qdd], g=[0, -G, 0])
        np.testing.assert_allclose(t, [tau], rtol=1e-14, atol=1e-14)


def test_pendulum_closed_form_random(rng):
    for _ in range(200):
        m, l, Izz = rng.uniform(0.5, 3), rng.uniform(0.2, 2), rng.uniform(0, 0.3)
        q, qd, qdd = rng.uniform(-4, 4, 3)
        t = oracle.rnea(synth.pendulum(m, l, Izz), [q], [qd], [qdd], g=[0, -G, 0])[0]
        ref = (m * l * l + Izz) * qdd + m * G * l * np.cos(q)
        assert abs(t - ref) <= 1e-13 * max(1, abs(ref))


def planar2_closed_form(q, qd, qdd, l1=1.1, r1=0.45, r2=0.6, m1=1.3, m2=0.9, I1=0.12, I2=0.07, g=G):
    """Textbook 2-link planar arm: tau = M qdd + C + G."""
    c2 = np.cos(q[1])
    M11 = I1 + I2 + m1 * r1 ** 2 + m2 * (l1 ** 2 + r2 ** 2 + 2 * l1 * r2 * c2)
    M12 = I2 + m2 * (r2 ** 2 + l1 * r2 * c2)
    M22 = I2 + m2 * r2 ** 2
    h = m2 * l1 * r2 * np.sin(q[1])
    C = np.array([-h * qd[1] * (2 * qd[0] + qd[1]), h * qd[0] ** 2])
    Gv = np.array([(m1 * r1 + m2 * l1) * g * np.cos(q[0]) + m2 * r2 * g * np.cos(q[0] + q[1]),
                   m2 * r2 * g * np.cos(q[0] + q[1])])
    return np.array([[M11, M12], [M12, M22]]) @ qdd + C + Gv


def test_planar2_closed_form_config_C1():
    # Config C1 (1000 states, the C1 state recipe) against the textbook closed form.
    cfg = synth.CONFIGS["C1"]
    q, qd, qdd = synth.states(cfg["seed"], 2, 0, 1000, cfg["ranges"])
    tau = oracle.rnea_batch(synth.planar2(), cfg["gravity"], q, qd, qdd)
    ref = np.stack([planar2_closed_form(q[:, b], qd[:, b], qdd[:, b]) for b in range(1000)], axis=1)
    err = np.abs(tau - ref).max(axis=0) / np.abs(ref).max(axis=0)
    assert err.max() < 1e-13


@pytest.mark.parametrize("n,seed,pf", [(1, 1, 0.0), (2, 2, 0.5), (3, 3, 0.0), (4, 4, 0.5), (6, 6, 0.3)])
def test_rnea_equals_euler_lagrange_brute_force(n, seed, pf, rng):
    # Textbook reduction: RNEA torques equal d/dt dL/dqd - dL/dq from an independent
    # energy model, every derivative by complex step (exact to rounding).
    r = synth.random_chain(n, seed, prismatic_fraction=pf)
    g = np.array([0.3, -1.2, -9.81])
    for _ in range(3):
        q, qd, qdd = rng.uniform(-np.pi, np.pi, n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        tau = oracle.rnea(r, q, qd, qdd, g=g)
        ref = euler_lagrange_tau(r, q, qd, qdd, g)
        assert np.abs(tau - ref).max() <= 1e-12 * np.abs(ref).max()


def test_power_identity(rng):
    # tau . qd = dE/dt with E = T + PE from the independent energy model (north_star pin).
    for n, pf in [(5, 0.0), (9, 0.4)]:
        r = synth.random_chain(n, 40 + n, prismatic_fraction=pf)
        g = np.array([0, 0, -9.81])
        for _ in range(5):
            q, qd, qdd = rng.uniform(-np.pi, np.pi, n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
            tau = oracle.rnea(r, q, qd, qdd, g=g)
            P = power(r, q, qd, qdd, g)
            assert abs(tau @ qd - P) <= 1e-12 * max(1.0, np.abs(tau).max() * np.abs(qd).sum())


def test_telescoping_power_identity(rng):
    # tau . qd = sum_i V_i . Fhat_i (discrete Newton-Euler power balance, zero boundary).
    r = synth.random_chain(20, 7)
    q, qd, qdd = rng.uniform(-3, 3, 20), rng.uniform(-1, 1, 20), rng.uniform(-1, 1, 20)
    tau, o = oracle.rnea(r, q, qd, qdd, g=[0, 0, 0], full=True)
    lhs = tau @ qd
    rhs = sum(o["V"][i] @ o["Fhat"][i] for i in range(20))
    assert abs(lhs - rhs) < 1e-11 * max(1, abs(lhs))


def test_tip_wrench_is_virtual_work(rng):
    # F_{n+1} (Eq. 3): tau(F) - tau(0) paired with qd equals the power V_tip . F_{n+1}
    # (f_{n,n+1} = I, reading A5), V_tip from the independent FK model.
    r = synth.random_chain(6, 8, prismatic_fraction=0.3)
    for _ in range(10):
        q, qd, qdd = rng.uniform(-3, 3, 6), rng.uniform(-1, 1, 6), rng.uniform(-1, 1, 6)
        F = rng.standard_normal(6)
        t1 = oracle.rnea(r, q, qd, qdd, Ftip=F)
        t0 = oracle.rnea(r, q, qd, qdd)
        Vt = tip_body_velocity(r, q, qd)
        assert abs((t1 - t0) @ qd - Vt @ F) < 1e-12 * max(1, np.abs(t1).max())


def test_base_acceleration_equals_gravity():
    # Reading A3: gravity g is the base acceleration Vdot_0 = (-g, 0); the explicit
    # Vdot_0 argument and the g= shorthand agree, and the EL pins above fix its sign.
    r = synth.random_chain(5, 9)
    q, qd, qdd = np.ones(5), np.zeros(5), np.zeros(5)
    g = np.array([1.0, 2.0, -9.0])
    np.testing.assert_array_equal(oracle.rnea(r, q, qd, qdd, g=g),
                                  oracle.rnea(r, q, qd, qdd, Vd0=np.concatenate([-g, np.zeros(3)])))


# ------------------------------------------------------------- scans (Alg. 1)
@pytest.mark.parametrize("variant", ["split", "fused", "lift", "sync15"])
@pytest.mark.parametrize("order", ["sequential", "kogge_stone"])
def test_scan_equals_recursion_tiny_chains(variant, order, rng):
    for n in range(1, 9):
        for pf in (0.0, 0.5):
            r = synth.random_chain(n, 100 + n, prismatic_fraction=pf)
            q, qd, qdd = rng.uniform(-3, 3, n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
            V0, Vd0, Ft = rng.standard_normal((3, 6))
            t0, o0 = oracle.rnea(r, q, qd, qdd, V0, Vd0, Ft, full=True)
            t1, o1 = oracle.rnea(r, q, qd, qdd, V0, Vd0, Ft, variant=variant, order=order, full=True)
            s = np.abs(t0).max()
            assert np.abs(t1 - t0).max() <= 1e-13 * s
            for k in ("V", "Vd", "F"):
                np.testing.assert_allclose(o1[k], o0[k], atol=1e-12 * max(1, np.abs(o0[k]).max()))


@pytest.mark.parametrize("n", [30, 64, 100])
def test_scan_equals_recursion_long_chains(n, rng):
    r = synth.random_chain(n, n)
    q, qd, qdd = rng.uniform(-3, 3, n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    t0 = oracle.rnea(r, q, qd, qdd, g=[0, 0, -9.81])
    for variant in ("split", "fused", "sync15"):
        t1 = oracle.rnea(r, q, qd, qdd, g=[0, 0, -9.81], variant=variant, order="kogge_stone")
        assert np.abs(t1 - t0).max() <= (1e-13 if variant != "sync15" else 1e-11) * np.abs(t0).max()


def test_bias_force_nine_of_21_quadratic_terms(rng):
    # Fhat depends on V = (v, w) only through w w^T and w x v.  With Vdot = 0,
    # changing v by alpha*w leaves w x v (and w w^T) unchanged, so Fhat is invariant.
    r = synth.random_chain(1, 11)
    for _ in range(20):
        V0 = rng.standard_normal(6)
        V1 = V0.copy()
        V1[:3] += rng.uniform(-2, 2) * V0[3:]
        # single link, q = qd = qdd = 0, f = M_1; choose V_0 so that V_1 = Ad_{M^-1} V_0 takes each value
        Mi = np.linalg.inv(r["M"][0])
        Ad_m = oracle.Ad(r["M"][0])
        z = np.zeros(1)
        _, oa = oracle.rnea(r, z, z, z, V0=Ad_m @ V0, full=True)
        _, ob = oracle.rnea(r, z, z, z, V0=Ad_m @ V1, full=True)
        np.testing.assert_allclose(oa["V"][0], V0, atol=1e-13)
        np.testing.assert_allclose(oa["Fhat"][0], ob["Fhat"][0], atol=1e-12)
        del Mi


# -------------------------------------------------------- JSI and FD (Eq. 5-8)
def test_jsi_symmetric_spd_and_linearity(rng):
    r = synth.random_chain(15, 12, prismatic_fraction=0.3)
    g = np.array([0, 0, -9.81])
    for _ in range(5):
        q, qd, qdd = rng.uniform(-3, 3, 15), rng.uniform(-1, 1, 15), rng.uniform(-1, 1, 15)
        M = oracle.jsi(r, q)
        assert np.abs(M - M.T).max() < 1e-13 * np.abs(M).max()
        np.linalg.cholesky(M)                                      # SPD
        bias = oracle.rnea(r, q, qd, np.zeros(15), g=g)            # Eq. (5)
        tau = oracle.rnea(r, q, qd, qdd, g=g)
        np.testing.assert_allclose(tau - bias, M @ qdd, atol=1e-12 * np.abs(tau).max())
        # kinetic energy 1/2 qd^T M qd from the independent energy model
        assert abs(0.5 * qd @ M @ qd - kinetic(r, q, qd)) < 1e-12 * max(1, abs(kinetic(r, q, qd)))


def test_jsi_matches_energy_model_mass_matrix(rng):
    r = synth.random_chain(5, 13, prismatic_fraction=0.4)
    q = rng.uniform(-3, 3, 5)
    np.testing.assert_allclose(oracle.jsi(r, q), mass_matrix(r, q), atol=1e-12)


def test_pendulum_fd_closed_form(rng):
    # point-mass pendulum, tau = 0 -> qdd = -(g/l) cos q.
    for algo in ("aba", "jsiia", "aba_scan"):
        for _ in range(20):
            m, l, q, qd = rng.uniform(0.5, 3), rng.uniform(0.2, 2), rng.uniform(-4, 4), rng.uniform(-2, 2)
            qdd = oracle.fd(synth.pendulum(m, l), [q], [qd], [0.0], g=[0, -G, 0], algo=algo)[0]
            assert abs(qdd + G / l * np.cos(q)) < 1e-13 * max(1, G / l)


@pytest.mark.parametrize("n", [1, 2, 7, 30, 100])
def test_fd_round_trip_and_cross_algorithm(n, rng):
    r = synth.random_chain(n, 200 + n, prismatic_fraction=0.2 if n < 30 else 0.0)
    g = np.array([0, 0, -9.81])
    for _ in range(3):
        q, qd, qdd = rng.uniform(-3, 3, n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        tau = oracle.rnea(r, q, qd, qdd, g=g)
        a = oracle.fd(r, q, qd, tau, g=g, algo="aba")
        j = oracle.fd(r, q, qd, tau, g=g, algo="jsiia")
        s = oracle.fd(r, q, qd, tau, g=g, algo="aba_scan", order="kogge_stone")
        # backward error (A14): RNEA(q, qd, qdd_fd) reproduces tau
        for x in (a, j, s):
            back = oracle.rnea(r, q, qd, x, g=g)
            assert np.abs(back - tau).max() <= 1e-11 * np.abs(tau).max()
        # forward error bounded by cond(M)
        cond = np.linalg.cond(oracle.jsi(r, q))
        tol = 1e-14 * max(10.0, cond) * 10
        assert np.abs(a - qdd).max() <= tol * max(1, np.abs(qdd).max())
        assert np.abs(a - j).max() <= tol * max(1, np.abs(qdd).max())
        assert np.abs(a - s).max() <= tol * max(1, np.abs(a).max())


def test_abi_boundary_and_psd(rng):
    r = synth.random_chain(10, 14, prismatic_fraction=0.3)
    q, qd = rng.uniform(-3, 3, 10), rng.uniform(-1, 1, 10)
    _, Jh = oracle.fd(r, q, qd, np.zeros(10), g=[0, 0, -9.81], return_abi=True)
    np.testing.assert_array_equal(Jh[-1], r["J"][-1])                   # Jhat_n = J_n (A9)
    for i in range(10):
        assert np.linalg.eigvalsh(Jh[i] - r["J"][i]).min() > -1e-10      # articulation adds inertia
        assert np.linalg.eigvalsh(Jh[i]).min() > 0


def test_fd_affine_in_tau(rng):
    r = synth.random_chain(8, 15)
    q, qd = rng.uniform(-3, 3, 8), rng.uniform(-1, 1, 8)
    t1, t2 = rng.standard_normal((2, 8)) * 5
    f1 = oracle.fd(r, q, qd, t1, g=[0, 0, -9.81])
    f2 = oracle.fd(r, q, qd, t2, g=[0, 0, -9.81])
    fa = oracle.fd(r, q, qd, t1 + 0.3 * (t2 - t1), g=[0, 0, -9.81])
    np.testing.assert_allclose(fa, f1 + 0.3 * (f2 - f1), atol=1e-10)


def test_batch_equals_single_calls(rng):
    r = synth.random_chain(7, 16)
    q, qd, qdd = synth.states(9, 7, 0, 50)
    g = np.array([0, 0, -9.81])
    tb = oracle.rnea_batch(r, g, q, qd, qdd, nthreads=3)
    for b in range(50):
        np.testing.assert_array_equal(tb[:, b], oracle.rnea(r, q[:, b], qd[:, b], qdd[:, b], g=g))
    fb = oracle.fd_batch(r, g, q, qd, tb, nthreads=2)
    for b in (0, 17, 49):
        np.testing.assert_array_equal(fb[:, b], oracle.fd(r, q[:, b], qd[:, b], tb[:, b], g=g))
    # empty batch
    assert oracle.rnea_batch(r, g, q[:, :0], qd[:, :0], qdd[:, :0]).shape == (7, 0)


@pytest.mark.parametrize("order", ["sequential", "kogge_stone"])
def test_merged_eq20_scan_equals_aba(order, rng):
    # Eq. (20) with the Omega^{-1} reading (A7) and the seeding of A8:
    # the merged 15x15 backward scan reproduces the ABA accelerations.
    for n in (1, 2, 3, 5, 8, 30):
        r = synth.random_chain(n, 300 + n, prismatic_fraction=0.3 if n < 30 else 0.0)
        V0, Vd0, Ft = rng.standard_normal((3, 6))
        q, qd, tau = rng.uniform(-3, 3, n), rng.uniform(-1, 1, n), rng.standard_normal(n) * 5
        a = oracle.fd(r, q, qd, tau, V0, Vd0, Ft, algo="aba")
        m = oracle.fd(r, q, qd, tau, V0, Vd0, Ft, algo="aba_merged", order=order)
        cond = np.linalg.cond(oracle.jsi(r, q))
        assert np.abs(m - a).max() <= 1e-14 * max(10.0, cond) * 10 * max(1, np.abs(a).max())


def _Q(V):
    # Q = (w x v, w1^2, w1 w2, w1 w3, w2^2, w2 w3, w3^2)
    v, w = V[:3], V[3:]
    return np.concatenate([np.cross(w, v), [w[0] * w[0], w[0] * w[1], w[0] * w[2], w[1] * w[1], w[1] * w[2],
                                            w[2] * w[2]]])


def test_eq15_synchronous_scan_operator_exists_with_block_pattern(rng):
    # Eq. (15) claims a LINEAR 28-dim recursion on (Vdot, Q, V, Fhat, 1) with the
    # block pattern of P:233-241 (starred blocks unspecified, A6).  For one link with fixed
    # (q, qd, qdd), sample previous states (Vdot_{i-1}, V_{i-1}) as the base twist of a 1-link
    # chain, fit the operator by least squares, and check: exact fit (the map is affine in the
    # lifted coordinates) and zeros where the paper prints 0.
    for seed in range(3):
        r = synth.random_chain(1, 900 + seed, prismatic_fraction=0.5 * seed)
        q, qd, qdd = rng.uniform(-3, 3, 3)
        X, Yv = [], []
        for _ in range(300):
            V0, Vd0 = rng.standard_normal((2, 6))
            Fprev = rng.standard_normal(6)
            _, o = oracle.rnea(r, [q], [qd], [qdd], V0=V0, Vd0=Vd0, full=True)
            X.append(np.concatenate([Vd0, _Q(V0), V0, Fprev, [1.0]]))
            Yv.append(np.concatenate([o["Vd"][0], _Q(o["V"][0]), o["V"][0], o["Fhat"][0], [1.0]]))
        X, Yv = np.array(X), np.array(Yv)
        A, *_ = np.linalg.lstsq(X, Yv, rcond=None)
        A = A.T                                               # x_i = A x_{i-1}
        assert np.abs(X @ A.T - Yv).max() < 1e-9 * np.abs(Yv).max()
        rows = {"Vdot": slice(0, 6), "Q": slice(6, 15), "V": slice(15, 21), "Fhat": slice(21, 27)}
        cols = {"Vdot": slice(0, 6), "Q": slice(6, 15), "V": slice(15, 21), "Fhat": slice(21, 27)}
        zero = [("Vdot", "Q"), ("Vdot", "Fhat"), ("Q", "Vdot"), ("Q", "Fhat"), ("V", "Vdot"), ("V", "Q"),
                ("V", "Fhat"), ("Fhat", "Fhat")]                   # the 0 entries of P:233-239
        for rr, cc in zero:
            assert np.abs(A[rows[rr], cols[cc]]).max() < 1e-8, (rr, cc)
        np.testing.assert_allclose(A[27], np.eye(28)[27], atol=1e-9)   # last row (0 ... 0 1)
        # the oracle's closed-form starred blocks (A6) are exactly this fitted operator
        A_closed = oracle.eq15_operator(r, q, qd, qdd)
        np.testing.assert_allclose(A_closed, A, atol=1e-8 * max(1.0, np.abs(A).max()))
