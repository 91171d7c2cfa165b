"""Independent Lagrangian model of a serial chain, used ONLY to pin the oracle.

Written from textbook rigid-body mechanics, not from the paper's recursions and
sharing no code with oracle/ or the CUDA path:

* forward kinematics g_{0,i}(q) = prod_k M_k exp([S_k] q_k), with exp computed by
  scaling-and-squaring of a truncated Taylor series of the 4x4 matrix (analytic
  in q, so complex-step differentiation is exact to rounding);
* link body velocity V_i = vee(g^{-1} dg/dt), dg/dt = sum_k (dg/dq_k) qd_k with
  dg/dq_k by the product rule d/dq exp([S]q) = [S] exp([S]q);
* kinetic energy T = 1/2 sum_i V_i^T J_i V_i, potential PE = -sum_i m_i g . c_i^0;
* Euler-Lagrange torques tau = M qdd + Mdot qd - dT/dq + dPE/dq, with M by
  polarisation of T (exact for a quadratic form) and every derivative by
  complex step (h = 1e-30).

Twist layout (v, w), hat(xi) = [[w^, v], [0, 0]] (A1).
"""
from __future__ import annotations

import numpy as np

H = 1e-30


def hat(xi):
    v, w = xi[:3], xi[3:]
    X = np.zeros((4, 4), dtype=np.result_type(xi, np.float64))
    X[0, 1], X[0, 2], X[1, 2] = -w[2], w[1], -w[0]
    X[1, 0], X[2, 0], X[2, 1] = w[2], -w[1], w[0]
    X[:3, 3] = v
    return X


def vee(X):
    return np.array([X[0, 3], X[1, 3], X[2, 3], X[2, 1], X[0, 2], X[1, 0]])


def expm4(A, terms: int = 18):
    """exp(A) of a 4x4 (real or complex) matrix: scale by 2^-s, Taylor, square s times."""
    nrm = np.abs(A.real).sum(axis=1).max() + 1e-300
    s = max(0, int(np.ceil(np.log2(nrm))) + 1)
    B = A / (2.0 ** s)
    E = np.eye(4, dtype=A.dtype)
    term = np.eye(4, dtype=A.dtype)
    for k in range(1, terms + 1):
        term = term @ B / k
        E = E + term
    for _ in range(s):
        E = E @ E
    return E


def rigid_inv(g):
    R, p = g[:3, :3], g[:3, 3]
    h = np.eye(4, dtype=g.dtype)
    h[:3, :3] = R.T
    h[:3, 3] = -R.T @ p
    return h


def fk(robot, q):
    """[g_{0,1}, ..., g_{0,n}] and the per-joint factors."""
    n = len(q)
    dt = np.result_type(q, np.float64)
    g = np.eye(4, dtype=dt)
    gs, Es = [], []
    for i in range(n):
        E = expm4(hat(robot["S"][i].astype(dt)) * q[i])
        Es.append(E)
        g = g @ robot["M"][i].astype(dt) @ E
        gs.append(g)
    return gs, Es


def body_velocities(robot, q, qd):
    """V_i = vee(g_{0,i}^{-1} d/dt g_{0,i}) along qd."""
    n = len(q)
    dt = np.result_type(q, qd, np.float64)
    gs, Es = fk(robot, q)
    Vs = []
    for i in range(n):
        gdot = np.zeros((4, 4), dtype=dt)
        for k in range(i + 1):
            # d g_{0,i} / d q_k = g_{0,k-1} M_k [S_k] e^{[S_k]q_k} (M_{k+1} e_{k+1}) ... (M_i e_i)
            left = np.eye(4, dtype=dt) if k == 0 else gs[k - 1]
            D = left @ robot["M"][k] @ hat(robot["S"][k]) @ Es[k]
            for j in range(k + 1, i + 1):
                D = D @ robot["M"][j] @ Es[j]
            gdot = gdot + D * qd[k]
        Vs.append(vee(rigid_inv(gs[i]) @ gdot))
    return Vs, gs


def mass_and_com(J):
    m = J[0, 0]
    C = J[3:, :3] / m                      # m[c] block
    return m, np.array([C[2, 1], C[0, 2], C[1, 0]])


def kinetic(robot, q, qd):
    Vs, _ = body_velocities(robot, q, qd)
    return 0.5 * sum(V @ robot["J"][i] @ V for i, V in enumerate(Vs))


def potential(robot, q, g):
    gs, _ = fk(robot, q)
    pe = 0.0
    for i, gi in enumerate(gs):
        m, c = mass_and_com(robot["J"][i])
        pc = gi[:3, :3] @ c + gi[:3, 3]
        pe = pe - m * (np.asarray(g) @ pc)
    return pe


def energy(robot, q, qd, g):
    return kinetic(robot, q, qd) + potential(robot, q, g)


def mass_matrix(robot, q):
    n = len(q)
    dt = np.result_type(q, np.float64)
    T1 = []
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        T1.append(kinetic(robot, q, e))
    M = np.zeros((n, n), dtype=dt)
    for j in range(n):
        M[j, j] = 2.0 * T1[j]
        for k in range(j + 1, n):
            e = np.zeros(n)
            e[j] = e[k] = 1.0
            M[j, k] = M[k, j] = kinetic(robot, q, e) - T1[j] - T1[k]
    return M


def euler_lagrange_tau(robot, q, qd, qdd, g):
    """tau = M qdd + Mdot qd - dT/dq + dPE/dq, all derivatives by complex step."""
    q, qd, qdd = (np.asarray(x, dtype=np.float64) for x in (q, qd, qdd))
    n = len(q)
    M = mass_matrix(robot, q)
    Mdot = mass_matrix(robot, q + 1j * H * qd).imag / H
    dT = np.zeros(n)
    dP = np.zeros(n)
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        dT[j] = kinetic(robot, q + 1j * H * e, qd).imag / H
        dP[j] = potential(robot, q + 1j * H * e, g).imag / H
    return M @ qdd + Mdot @ qd - dT + dP


def power(robot, q, qd, qdd, g):
    """dE/dt along (qd, qdd) by one complex step of E(q + ih qd, qd + ih qdd)."""
    q, qd, qdd = (np.asarray(x, dtype=np.float64) for x in (q, qd, qdd))
    return energy(robot, q + 1j * H * qd, qd + 1j * H * qdd, g).imag / H


def tip_body_velocity(robot, q, qd):
    Vs, _ = body_velocities(robot, q, qd)
    return Vs[-1]
