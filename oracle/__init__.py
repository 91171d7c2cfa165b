"""ctypes wrapper of the C++ oracle (oracle/oracle.cpp) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this package.  The product package
paper_1609_04493_b200 never imports it and shares no code with it.

Every function takes the robot as numpy arrays M [n,4,4], S [n,6], J [n,6,6]
(see synth/) and works in float64.  Citations are to PAPER.md lines (P:n) in
oracle.cpp.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

# Plain -O2, no -ffast-math, no explicit SIMD (SURVEY §8(d) CPU baseline).
CXXFLAGS = ["-O2", "-std=c++17", "-shared", "-fPIC", "-Wall"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++) if missing or older than oracle.cpp."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *CXXFLAGS, "-o", tmp, _SRC, "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d = ctypes.POINTER(ctypes.c_double)
        i32, i64 = ctypes.c_int, ctypes.c_int64
        L.orc_last_error.restype = ctypes.c_char_p
        for name, args in {
            "orc_exp_twist": [d, ctypes.c_double, d],
            "orc_Ad": [d, d], "orc_ad": [d, d], "orc_inv": [d, d],
            "orc_velacc_oplus": [d, d, d], "orc_velacc_inverse": [d, d], "orc_velacc_lift13": [d, d],
        }.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = None
        L.orc_rnea.argtypes = [i32, d, d, d, d, d, d, d, d, d, i32, i32, d, d, d, d, d]
        L.orc_jsi.argtypes = [i32, d, d, d, d, d]
        L.orc_eq15_operator.argtypes = [d, d, d, ctypes.c_double, ctypes.c_double, ctypes.c_double, d]
        L.orc_fd.argtypes = [i32, d, d, d, d, d, d, d, d, d, i32, i32, d, d]
        L.orc_rnea_batch.argtypes = [i32, d, d, d, d, i64, d, d, d, d, i32]
        L.orc_fd_batch.argtypes = [i32, d, d, d, d, i64, d, d, d, d, i32, i32]
        for name in ("orc_rnea", "orc_jsi", "orc_fd", "orc_rnea_batch", "orc_fd_batch", "orc_eq15_operator"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def _check(rc):
    if rc != 0:
        raise RuntimeError("oracle: " + lib().orc_last_error().decode())


def _robot(robot):
    M, S, J = (_f64(robot[k]) for k in ("M", "S", "J"))
    n = S.shape[0]
    assert M.shape == (n, 4, 4) and J.shape == (n, 6, 6)
    return n, M, S, J


def gravity_boundary(g):
    """(V_0, Vdot_0, F_{n+1}) for gravity g: (0, (-g, 0), 0) (reading A3)."""
    vd0 = np.zeros(6)
    vd0[:3] = -np.asarray(g, dtype=np.float64)
    return np.zeros(6), vd0, np.zeros(6)


# ------------------------------------------------------------------ SE(3) helpers
def exp_twist(S, q):
    g = np.zeros((4, 4))
    lib().orc_exp_twist(_p(_f64(S)), float(q), _p(g))
    return g


def Ad(g):
    out = np.zeros((6, 6))
    lib().orc_Ad(_p(_f64(g)), _p(out))
    return out


def ad(xi):
    out = np.zeros((6, 6))
    lib().orc_ad(_p(_f64(xi)), _p(out))
    return out


def inv(g):
    out = np.zeros((4, 4))
    lib().orc_inv(_p(_f64(g)), _p(out))
    return out


def _va(a):
    g, x1, x2 = a
    return np.concatenate([_f64(g).ravel(), _f64(x1), _f64(x2)])


def _unva(v):
    return v[:16].reshape(4, 4).copy(), v[16:22].copy(), v[22:28].copy()


def velacc_oplus(a, b):
    """Eq. (13): (g,xi1,xi2) (+) (g',xi1',xi2')."""
    out = np.zeros(28)
    lib().orc_velacc_oplus(_p(_va(a)), _p(_va(b)), _p(out))
    return _unva(out)


def velacc_inverse(a):
    """Eq. (14)."""
    out = np.zeros(28)
    lib().orc_velacc_inverse(_p(_va(a)), _p(out))
    return _unva(out)


def velacc_lift13(a):
    """13x13 lift of Eq. (12)."""
    out = np.zeros((13, 13))
    lib().orc_velacc_lift13(_p(_va(a)), _p(out))
    return out


# ------------------------------------------------------------------ dynamics
RNEA_VARIANTS = {"recursive": 0, "split": 1, "fused": 2, "lift": 3, "sync15": 4}
SCAN_ORDERS = {"sequential": 0, "kogge_stone": 1}


def rnea(robot, q, qd, qdd, V0=None, Vd0=None, Ftip=None, g=None,
         variant="recursive", order="sequential", full=False):
    """tau = ID(q, qd, qdd, V_0, Vdot_0, F_{n+1}) (Eq. 3) for ONE state.

    Give either g (gravity, reading A3) or explicit V0/Vd0/Ftip (defaults 0).
    full=True also returns dict(V, Vd, F, Fhat) as [n, 6] arrays.
    """
    n, M, S, J = _robot(robot)
    if g is not None:
        V0, Vd0, Ftip = gravity_boundary(g)
    V0 = np.zeros(6) if V0 is None else _f64(V0)
    Vd0 = np.zeros(6) if Vd0 is None else _f64(Vd0)
    Ftip = np.zeros(6) if Ftip is None else _f64(Ftip)
    q, qd, qdd = (_f64(x, (n,)) for x in (q, qd, qdd))
    tau = np.zeros(n)
    V, Vd, F, Fh = (np.zeros((n, 6)) for _ in range(4))
    _check(lib().orc_rnea(n, _p(M), _p(S), _p(J), _p(q), _p(qd), _p(qdd), _p(V0), _p(Vd0), _p(Ftip),
                          RNEA_VARIANTS[variant], SCAN_ORDERS[order], _p(tau), _p(V), _p(Vd), _p(F), _p(Fh)))
    if full:
        return tau, dict(V=V, Vd=Vd, F=F, Fhat=Fh)
    return tau


def eq15_operator(robot1, q, qd, qdd):
    """The 28x28 operator A_i of Eq. (15) (x = (Vdot, Q, V, Fhat, 1)) of a 1-link robot."""
    n, M, S, J = _robot(robot1)
    assert n == 1
    out = np.zeros((28, 28))
    _check(lib().orc_eq15_operator(_p(M), _p(S), _p(J), float(q), float(qd), float(qdd), _p(out)))
    return out


def jsi(robot, q):
    """Joint-space inertia M(q) by Eq. (17)."""
    n, M, S, J = _robot(robot)
    out = np.zeros((n, n))
    _check(lib().orc_jsi(n, _p(M), _p(S), _p(J), _p(_f64(q, (n,))), _p(out)))
    return out


FD_ALGOS = {"aba": 0, "jsiia": 1, "aba_scan": 2, "aba_merged": 3}


def fd(robot, q, qd, tau, V0=None, Vd0=None, Ftip=None, g=None, algo="aba",
       order="sequential", return_abi=False):
    """qdd = FD(q, qd, tau, V_0, Vdot_0, F_{n+1}) (Eq. 4) for ONE state."""
    n, M, S, J = _robot(robot)
    if g is not None:
        V0, Vd0, Ftip = gravity_boundary(g)
    V0 = np.zeros(6) if V0 is None else _f64(V0)
    Vd0 = np.zeros(6) if Vd0 is None else _f64(Vd0)
    Ftip = np.zeros(6) if Ftip is None else _f64(Ftip)
    q, qd, tau = (_f64(x, (n,)) for x in (q, qd, tau))
    qdd = np.zeros(n)
    Jh = np.zeros((n, 6, 6))
    _check(lib().orc_fd(n, _p(M), _p(S), _p(J), _p(q), _p(qd), _p(tau), _p(V0), _p(Vd0), _p(Ftip),
                        FD_ALGOS[algo], SCAN_ORDERS[order], _p(qdd), _p(Jh)))
    return (qdd, Jh) if return_abi else qdd


def _nthreads(nthreads):
    return int(nthreads) if nthreads else (os.cpu_count() or 1)


def rnea_batch(robot, g, q, qd, qdd, nthreads=None):
    """Batched ID, link-major [n, B] arrays, gravity boundary (A3)."""
    n, M, S, J = _robot(robot)
    q, qd, qdd = (_f64(x) for x in (q, qd, qdd))
    B = q.shape[1]
    tau = np.zeros((n, B))
    _check(lib().orc_rnea_batch(n, _p(M), _p(S), _p(J), _p(_f64(g)), B, _p(q), _p(qd), _p(qdd),
                                _p(tau), _nthreads(nthreads)))
    return tau


def fd_batch(robot, g, q, qd, tau, algo="aba", nthreads=None):
    """Batched FD, link-major [n, B] arrays, gravity boundary (A3)."""
    n, M, S, J = _robot(robot)
    q, qd, tau = (_f64(x) for x in (q, qd, tau))
    B = q.shape[1]
    qdd = np.zeros((n, B))
    _check(lib().orc_fd_batch(n, _p(M), _p(S), _p(J), _p(_f64(g)), B, _p(q), _p(qd), _p(tau),
                              _p(qdd), FD_ALGOS[algo], _nthreads(nthreads)))
    return qdd
