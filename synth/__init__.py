"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no transforms, no recursion, no
dynamics).  It only draws robot parameters and joint states from seeded random
distributions, so both sides of every parity check see the same numbers:

* robots:   M_i (home transform, frame i -> frame i-1), S_i (joint twist,
            (v, w) ordering) and J_i (6x6 spatial inertia),
            drawn per DESIGN.md "Input recipe" (SURVEY §8(d), S:207 ranges);
* presets:  the single pendulum, the 2-link planar arm (config C1) and the
            synthetic 7-DoF `arm7` (config C2);
* states:   q, qd, qdd (and tau) as a pure function of
            (seed, stream, link, GLOBAL state index) through a counter-based
            splitmix64 hash, so any shard of the batch regenerates its slice
            bit-identically (SURVEY §8(d) "States", §8(e)).

Arrays are structure-of-arrays, link-major: x[i, b] (C order), i.e. the
device layout x[i*B + b] of include/rd.h.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "splitmix64", "uniform01", "uniform_states", "states",
    "random_chain", "pendulum", "planar2", "arm7", "spatial_inertia",
    "random_rotation", "CONFIGS",
]

_MASK = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vigna's splitmix64 finaliser on uint64 arrays (wrap-around arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, stream: int, link: int, idx: np.ndarray) -> np.ndarray:
    """U[0,1) doubles, a pure function of (seed, stream, link, global index)."""
    with np.errstate(over="ignore"):
        key = splitmix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
        key = splitmix64(key ^ np.uint64((stream & 0xFFFF) << 48 | (link & 0xFFFFFFFF)))
        z = splitmix64(key ^ (np.asarray(idx, dtype=np.uint64) * _GOLD))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def uniform_states(seed: int, stream: int, n: int, b0: int, b1: int,
                   lo: float, hi: float) -> np.ndarray:
    """[n, b1-b0] array of U[lo, hi) draws for global state indices b0..b1-1."""
    idx = np.arange(b0, b1, dtype=np.uint64)
    out = np.empty((n, b1 - b0), dtype=np.float64)
    for i in range(n):
        out[i] = lo + (hi - lo) * uniform01(seed, stream, i, idx)
    return out


# Per-config state ranges (SURVEY §8(d) "States"): q~U[-pi,pi], qd,qdd~U[-1,1];
# C1 uses qd~U[-2,2], qdd~U[-5,5]; FD torques come from the oracle (round trip).
_RANGES = {
    "default": ((-np.pi, np.pi), (-1.0, 1.0), (-1.0, 1.0)),
    "C1": ((-np.pi, np.pi), (-2.0, 2.0), (-5.0, 5.0)),
}


def states(seed: int, n: int, b0: int, b1: int, ranges: str = "default"):
    """(q, qd, qdd), each [n, b1-b0] float64, for global states b0..b1-1.

    Streams 0/1/2 are q/qd/qdd; the state seed is the config id.
    """
    (ql, qh), (dl, dh), (al, ah) = _RANGES[ranges]
    q = uniform_states(seed, 0, n, b0, b1, ql, qh)
    qd = uniform_states(seed, 1, n, b0, b1, dl, dh)
    qdd = uniform_states(seed, 2, n, b0, b1, al, ah)
    return q, qd, qdd


# ---------------------------------------------------------------------------
# Robot parameters
# ---------------------------------------------------------------------------

def _skew(c):
    return np.array([[0.0, -c[2], c[1]], [c[2], 0.0, -c[0]], [-c[1], c[0], 0.0]])


def spatial_inertia(m: float, com, I_c) -> np.ndarray:
    """6x6 spatial inertia about the link-frame origin, (v, w) ordering.

    Assembled from mass m, centre of mass c and the rotational inertia I_c about
    the centre of mass: [[m I, -m[c]], [m[c], I_c - m[c][c]]]  (A1).
    This is the parameterisation of the model input, not a dynamics step.
    """
    c = np.asarray(com, dtype=np.float64)
    C = _skew(c)
    J = np.zeros((6, 6))
    J[:3, :3] = m * np.eye(3)
    J[:3, 3:] = -m * C
    J[3:, :3] = m * C
    J[3:, 3:] = np.asarray(I_c, dtype=np.float64) - m * C @ C
    return 0.5 * (J + J.T)


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    """Uniform random rotation: QR of a Gaussian with sign fix, det +1."""
    A = rng.standard_normal((3, 3))
    Q, R = np.linalg.qr(A)
    Q = Q * np.sign(np.diag(R))
    if np.linalg.det(Q) < 0:
        Q[:, 0] = -Q[:, 0]
    return Q


def _unit(rng):
    v = rng.standard_normal(3)
    return v / np.linalg.norm(v)


def random_chain(n: int, seed: int, prismatic_fraction: float = 0.0):
    """Random n-link serial chain (SURVEY §8(d) "Robots"; S:207 ranges).

    Returns dict(M=[n,4,4], S=[n,6], J=[n,6,6]).  Per link:
    * M_i: uniform random rotation; translation direction uniform on S^2, length
      U[0.1, 1.0] m;
    * joint: revolute about a unit axis w through a point r ~ U[-0.2,0.2]^3,
      S = (r x w, w); or (with probability prismatic_fraction) prismatic along
      a unit direction, S = (v, 0);
    * inertia: mass U[0.5, 5] kg; CoM U[-0.2, 0.2]^3 m; I_c = R diag(l) R^T with
      l ~ U[0.01, 0.2] kg m^2.
    """
    if n < 1:
        raise ValueError("random_chain: n must be >= 1")
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), int(n), 1609_04493]))
    M = np.zeros((n, 4, 4))
    S = np.zeros((n, 6))
    J = np.zeros((n, 6, 6))
    for i in range(n):
        M[i, :3, :3] = random_rotation(rng)
        M[i, :3, 3] = _unit(rng) * rng.uniform(0.1, 1.0)
        M[i, 3, 3] = 1.0
        prismatic = rng.uniform() < prismatic_fraction
        w = _unit(rng)
        r = rng.uniform(-0.2, 0.2, 3)
        if prismatic:
            S[i, :3] = w
        else:
            S[i, :3] = np.cross(r, w)
            S[i, 3:] = w
        m = rng.uniform(0.5, 5.0)
        com = rng.uniform(-0.2, 0.2, 3)
        Rc = random_rotation(rng)
        lam = rng.uniform(0.01, 0.2, 3)
        J[i] = spatial_inertia(m, com, Rc @ np.diag(lam) @ Rc.T)
    return {"M": M, "S": S, "J": J}


def _trans(x, y, z):
    T = np.eye(4)
    T[:3, 3] = (x, y, z)
    return T


def _rotx(a):
    T = np.eye(4)
    c, s = np.cos(a), np.sin(a)
    T[1:3, 1:3] = [[c, -s], [s, c]]
    return T


def _roty(a):
    T = np.eye(4)
    c, s = np.cos(a), np.sin(a)
    T[0, 0], T[0, 2], T[2, 0], T[2, 2] = c, s, -s, c
    return T


def tilted_planar(n: int, eps: float, seed: int):
    """A planar n-link arm (all joint axes parallel to z) whose every joint axis is
    tilted by ~eps rad (a calibrated, nominally planar arm): consecutive axes are
    NEARLY parallel, so their common normal lies ~offset/eps away from the links."""
    rng = np.random.default_rng(seed)
    M, S, J = [], [], []
    for i in range(n):
        tilt = _rotx(eps * rng.choice([-1, 1]) * (0.5 + rng.random())) @ _roty(eps * rng.standard_normal())
        M.append((_trans(0.4 + 0.2 * rng.random(), 0, 0.05 * rng.standard_normal()) if i else np.eye(4)) @ tilt)
        S.append([0, 0, 0, 0, 0, 1.0])
        J.append(spatial_inertia(1.0 + rng.random(), (0.2, 0.01, 0.0), np.diag([0.01, 0.02, 0.02])))
    return {"M": np.array(M), "S": np.array(S), "J": np.array(J)}


def pendulum(m: float = 1.7, l: float = 0.8, Izz: float = 0.0):
    """Single revolute link about z, mass m at (l, 0, 0), gravity -y.

    Izz = 0 is the point mass of S:272 (J is then PSD, rank 4: fine for the
    oracle).  Izz > 0 gives I_c = Izz*I (SPD, accepted by rd_model_create); the
    closed form becomes tau = (m l^2 + Izz) qdd + m g l cos q.
    """
    M = np.eye(4)[None]
    S = np.array([[0, 0, 0, 0, 0, 1.0]])
    J = spatial_inertia(m, (l, 0, 0), Izz * np.eye(3))[None]
    return {"M": M, "S": S, "J": J}


def planar2(l1=1.1, r1=0.45, r2=0.6, m1=1.3, m2=0.9, I1=0.12, I2=0.07):
    """Config C1: 2-link planar arm; gravity (0, -g, 0).

    M_1 = I, M_2 = Trans(l1, 0, 0), S_1 = S_2 = (0,0,0, 0,0,1); link i has mass
    m_i, CoM (r_i, 0, 0) and I_c = diag(I_i, I_i, I_i) (only the z entry acts).
    """
    M = np.stack([np.eye(4), _trans(l1, 0, 0)])
    S = np.array([[0, 0, 0, 0, 0, 1.0]] * 2)
    J = np.stack([spatial_inertia(m1, (r1, 0, 0), I1 * np.eye(3)),
                  spatial_inertia(m2, (r2, 0, 0), I2 * np.eye(3))])
    return {"M": M, "S": S, "J": J}


def arm7():
    """Config C2: synthetic anthropomorphic 7-DoF arm; not a real robot.

    Every joint revolute about its local z; M_i = Trans(0,0,d_i) Rot_x(alpha_i);
    CoM (0, 0, 0.1); I_c = m_i diag(0.01, 0.01, 0.005).
    """
    d = (0.34, 0.0, 0.40, 0.0, 0.40, 0.0, 0.126)
    alpha = (0.0, -np.pi / 2, np.pi / 2, np.pi / 2, -np.pi / 2, -np.pi / 2, np.pi / 2)
    mass = (4.0, 4.0, 3.0, 2.7, 1.7, 1.8, 0.3)
    M = np.stack([_trans(0, 0, d[i]) @ _rotx(alpha[i]) for i in range(7)])
    S = np.array([[0, 0, 0, 0, 0, 1.0]] * 7)
    J = np.stack([spatial_inertia(mass[i], (0, 0, 0.1), mass[i] * np.diag([0.01, 0.01, 0.005]))
                  for i in range(7)])
    return {"M": M, "S": S, "J": J}


GRAVITY_Z = np.array([0.0, 0.0, -9.81])
GRAVITY_Y = np.array([0.0, -9.81, 0.0])

# BASELINE.json configs (C1..C5): robot, state seed/ranges, batch, dtype.
CONFIGS = {
    "C1": dict(robot="planar2", n=2, batch=1000, seed=1, ranges="C1", gravity=GRAVITY_Y),
    "C2": dict(robot="arm7", n=7, batch=100_000, seed=2, ranges="default", gravity=GRAVITY_Z),
    "C3": dict(robot="random", n=30, batch=1_000_000, seed=3, ranges="default", gravity=GRAVITY_Z),
    "C4": dict(robot="random", n=100, batch=100_000, seed=4, ranges="default", gravity=GRAVITY_Z),
    "C5": dict(robot="random", n=30, batch=10_000_000, seed=5, ranges="default", gravity=GRAVITY_Z),
}


def robot_for(cfg: dict):
    """The robot of a CONFIGS entry (random chains use robot seed 1000 + n)."""
    if cfg["robot"] == "planar2":
        return planar2()
    if cfg["robot"] == "arm7":
        return arm7()
    return random_chain(cfg["n"], 1000 + cfg["n"])


# ---------------------------------------------------------------------------
# The same state generator on the GPU (synth/gen.cu -> synth/libsynth.so):
# each rank generates its shard in device memory from the GLOBAL state indices.
# ---------------------------------------------------------------------------

import ctypes as _ctypes  # noqa: E402
import os as _os  # noqa: E402
import subprocess as _subprocess  # noqa: E402

_HERE = _os.path.dirname(_os.path.abspath(__file__))
_GEN_SRC = _os.path.join(_HERE, "gen.cu")
_GEN_LIB = _os.path.join(_HERE, "libsynth.so")
_gen = None


def build_device_generator(force: bool = False) -> str:
    """nvcc -> synth/libsynth.so (sm_100a), if missing or older than gen.cu."""
    if force or not _os.path.exists(_GEN_LIB) or _os.path.getmtime(_GEN_LIB) < _os.path.getmtime(_GEN_SRC):
        nvcc = "/usr/local/cuda/bin/nvcc" if _os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc"
        tmp = _GEN_LIB + f".tmp{_os.getpid()}"
        _subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                                "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-o", tmp, _GEN_SRC])
        _os.replace(tmp, _GEN_LIB)
    return _GEN_LIB


def _gen_lib():
    global _gen
    if _gen is None:
        build_device_generator()
        L = _ctypes.CDLL(_GEN_LIB)
        u64, i32, i64, dbl, vp = (_ctypes.c_uint64, _ctypes.c_int, _ctypes.c_int64, _ctypes.c_double,
                                  _ctypes.c_void_p)
        for name in ("synth_uniform_states_f64", "synth_uniform_states_f32"):
            getattr(L, name).argtypes = [u64, i32, i32, i64, i64, dbl, dbl, vp, i64, vp]
            getattr(L, name).restype = i32
        _gen = L
    return _gen


def states_device(seed: int, n: int, b0: int, b1: int, ranges: str = "default", dtype=None, device=None):
    """`states` generated on the GPU: (q, qd, qdd) torch tensors [n, b1-b0] of
    `dtype` (float64 default; float32 = the float64 draw rounded to nearest)
    on `device`, bit-identical to torch.from_numpy(states(...)).to(dtype)."""
    import torch
    dtype = torch.float64 if dtype is None else dtype
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    L = _gen_lib()
    fn = L.synth_uniform_states_f64 if dtype == torch.float64 else L.synth_uniform_states_f32
    out = []
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream(device).cuda_stream
        for k, (lo, hi) in enumerate(_RANGES[ranges]):
            t = torch.empty((n, b1 - b0), dtype=dtype, device=device)
            rc = fn(seed & 0xFFFFFFFFFFFFFFFF, k, n, b0, b1, float(lo), float(hi), t.data_ptr(), b1 - b0, stream)
            if rc:
                raise RuntimeError(f"synth device generator failed (status {rc})")
            out.append(t)
    return tuple(out)
