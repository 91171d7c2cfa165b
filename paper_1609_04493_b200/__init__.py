"""paper_1609_04493_b200 -- batched robot dynamics on B200 (arXiv 1609.04493).

Thin Python binding of librd.so (include/rd.h): argument marshalling only.
Every step of the dynamics runs in the library's sm_100a kernels; PyTorch is
used for device memory and streams.  There is no CPU fallback: if librd.so is
missing or no CUDA device is present, calls raise.

    import paper_1609_04493_b200 as rd
    model = rd.Model(M, S, J, gravity=(0, 0, -9.81))   # numpy arrays, see include/rd.h
    tau = rd.inverse_dynamics(model, q, qd, qdd)        # torch CUDA tensors [n, B]
    qdd = rd.forward_dynamics(model, q, qd, tau)

Names follow the paper: ID(q, qd, qdd) = tau (Eq. 3), FD(q, qd, tau) = qdd (Eq. 4).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["Model", "inverse_dynamics", "forward_dynamics", "inverse_dynamics_host", "forward_dynamics_host", "lib",
           "RdError", "STRATEGIES", "last_launch_count", "LIB_PATH"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "librd.so")

STRATEGIES = {"auto": 0, "thread": 1, "warp_scan": 2, "generic": 3, "reverse": 4, "block_scan": 5,
              "warp_scan_eq13": 6, "warp_scan_eq15": 7, "chunk": 8}
_STRAT_NAMES = {v: k for k, v in STRATEGIES.items()}
FD_ALGOS = {"aba": 0, "jsiia": 1, "aba_scan": 2, "aba_merged": 3}

# Symbols declared in include/rd.h (checked by tests/test_capi.py).
EXPORTS = [
    "rd_version", "rd_last_error", "rd_model_create", "rd_model_destroy", "rd_model_n", "rd_model_device",
    "rd_model_set_strategy", "rd_model_resolve_strategy", "rd_model_set_boundary",
    "rd_inverse_dynamics_f64", "rd_inverse_dynamics_f32", "rd_forward_dynamics_f64",
    "rd_forward_dynamics_f32", "rd_model_set_fd_algo", "rd_inverse_dynamics_host_f64",
    "rd_last_launch_count", "rd_forward_dynamics_ex_f64", "rd_forward_dynamics_ex_f32",
    "rd_inverse_dynamics_bnd_f64", "rd_inverse_dynamics_bnd_f32", "rd_forward_dynamics_bnd_f64",
    "rd_forward_dynamics_bnd_f32", "rd_forward_dynamics_host_f64",
]


class RdError(RuntimeError):
    pass


_lib = None


def lib():
    """Load librd.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RdError(f"librd.so not found at {LIB_PATH}: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        dp = ctypes.POINTER(ctypes.c_double)
        L.rd_version.restype = ctypes.c_char_p
        L.rd_last_error.restype = ctypes.c_char_p
        L.rd_model_create.argtypes = [i32, dp, dp, dp, dp, ctypes.POINTER(vp)]
        L.rd_model_destroy.argtypes = [vp]
        L.rd_model_n.argtypes = [vp]
        L.rd_model_n.restype = i32
        L.rd_model_device.argtypes = [vp]
        L.rd_model_device.restype = i32
        L.rd_model_set_strategy.argtypes = [vp, ctypes.c_int, i32]
        L.rd_model_resolve_strategy.argtypes = [vp, i64, i32]
        L.rd_model_resolve_strategy.restype = ctypes.c_int
        L.rd_model_set_boundary.argtypes = [vp, dp, dp, dp]
        L.rd_model_set_fd_algo.argtypes = [vp, ctypes.c_int]
        for name in ("rd_inverse_dynamics_f64", "rd_inverse_dynamics_f32",
                     "rd_forward_dynamics_f64", "rd_forward_dynamics_f32"):
            getattr(L, name).argtypes = [vp, i64, vp, vp, vp, vp, vp]
        for name in ("rd_forward_dynamics_ex_f64", "rd_forward_dynamics_ex_f32"):
            getattr(L, name).argtypes = [vp, i64, vp, vp, vp, vp, vp, vp]
        for name in ("rd_inverse_dynamics_bnd_f64", "rd_inverse_dynamics_bnd_f32"):
            getattr(L, name).argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp, vp]
        for name in ("rd_forward_dynamics_bnd_f64", "rd_forward_dynamics_bnd_f32"):
            getattr(L, name).argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.rd_inverse_dynamics_host_f64.argtypes = [vp, i64, vp, vp, vp, vp]
        L.rd_forward_dynamics_host_f64.argtypes = [vp, i64, vp, vp, vp, vp]
        L.rd_last_launch_count.restype = i32
        for name in EXPORTS:
            if name not in ("rd_version", "rd_last_error", "rd_model_n", "rd_model_device",
                            "rd_model_resolve_strategy", "rd_last_launch_count"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        raise RdError(f"{what}: status {rc}: {lib().rd_last_error().decode()}")


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def last_launch_count() -> int:
    """Kernels the last rd_* compute call on this thread enqueued."""
    return int(lib().rd_last_launch_count())


class Model:
    """A robot: M [n,4,4], S [n,6], J [n,6,6] (host float64), gravity (3,).

    Created on the current CUDA device (rd_model_create, include/rd.h).
    """

    def __init__(self, M, S, J, gravity=(0.0, 0.0, -9.81)):
        M, S, J = (np.ascontiguousarray(x, dtype=np.float64) for x in (M, S, J))
        n = S.shape[0]
        if M.shape != (n, 4, 4) or S.shape != (n, 6) or J.shape != (n, 6, 6):
            raise ValueError("Model expects M [n,4,4], S [n,6], J [n,6,6]")
        g = np.ascontiguousarray(gravity, dtype=np.float64).reshape(3)
        h = ctypes.c_void_p()
        _check(lib().rd_model_create(n, _dptr(M), _dptr(S), _dptr(J), _dptr(g), ctypes.byref(h)),
               "rd_model_create")
        self._h = h
        self.n = n
        self.device = int(lib().rd_model_device(h))     # CUDA ordinal the constants live on

    @classmethod
    def from_robot(cls, robot: dict, gravity=(0.0, 0.0, -9.81)):
        return cls(robot["M"], robot["S"], robot["J"], gravity)

    @property
    def handle(self):
        return self._h

    def set_strategy(self, name: str, lanes_per_state: int = 0):
        """Inverse-dynamics strategy by name (STRATEGIES); "chunk" takes lanes_per_state
        (0 = from n), also spelled "chunk:L" (e.g. "chunk:8")."""
        if name.startswith("chunk:"):
            name, lanes_per_state = "chunk", int(name.split(":", 1)[1])
        _check(lib().rd_model_set_strategy(self._h, STRATEGIES[name], int(lanes_per_state)),
               "rd_model_set_strategy")

    def resolve_strategy(self, batch: int, fp64: bool = True) -> str:
        return _STRAT_NAMES[lib().rd_model_resolve_strategy(self._h, int(batch), int(fp64))]

    def set_fd_algo(self, name: str):
        _check(lib().rd_model_set_fd_algo(self._h, FD_ALGOS[name]), "rd_model_set_fd_algo")

    def set_boundary(self, V0=None, Vdot0=None, Ftip=None):
        """Full Eq. (3) boundary: base twist, base acceleration, tip wrench (frame n)."""
        arrs = [None if x is None else np.ascontiguousarray(x, dtype=np.float64).reshape(6)
                for x in (V0, Vdot0, Ftip)]
        ptrs = [None if a is None else _dptr(a) for a in arrs]
        _check(lib().rd_model_set_boundary(self._h, *ptrs), "rd_model_set_boundary")

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().rd_model_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stream_ptr(stream, device_index=None):
    import torch
    if stream is not None:
        return stream.cuda_stream
    # the current stream's raw handle without constructing a torch.cuda.Stream
    # object (the binding's own cost dominated small-batch calls, tools/host_overhead.py)
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None and device_index is not None:
        return raw(device_index)
    return torch.cuda.current_stream().cuda_stream


def _check_tensors(model: Model, *ts):
    """Marshalling checks only: CUDA, fp64/fp32, one device, contiguous [n, B]."""
    import torch
    t0 = ts[0]
    dt = t0.dtype
    if not t0.is_cuda:
        raise RdError("inputs must be CUDA tensors (use inverse_dynamics_host for host arrays)")
    if dt is not torch.float64 and dt is not torch.float32:
        raise RdError("dtype must be float64 or float32")
    dev = t0.get_device()
    if dev != model.device:
        raise RdError(f"tensors are on cuda:{dev} but the model was created on cuda:{model.device}")
    shape = t0.shape
    if len(shape) != 2 or shape[0] != model.n:
        raise RdError("tensors must be contiguous [n, B] with one dtype/device")
    for t in ts:
        if t.dtype is not dt or t.get_device() != dev or t.shape != shape or not t.is_contiguous():
            raise RdError("tensors must be contiguous [n, B] with one dtype/device")
    return dt


def _boundary_ptrs(boundary, ref):
    """(V0, Vdot0, Ftip) per-state arrays [6, B] (None entries allowed) -> pointers."""
    ptrs = []
    for t in boundary:
        if t is None:
            ptrs.append(None)
            continue
        if t.dtype != ref.dtype or t.device != ref.device or tuple(t.shape) != (6, ref.shape[1]) \
                or not t.is_contiguous():
            raise RdError("boundary arrays must be contiguous [6, B] tensors with the inputs' dtype/device")
        ptrs.append(t.data_ptr())
    if len(ptrs) != 3:
        raise RdError("boundary = (V0, Vdot0, Ftip)")
    return ptrs


def inverse_dynamics(model: Model, q, qd, qdd, out=None, stream=None, boundary=None):
    """tau = ID(q, qd, qdd) (Eq. 1-3) for B states; torch CUDA tensors [n, B].

    boundary: optional per-state (V0, Vdot0, Ftip), each a [6, B] tensor or None
    (rd_inverse_dynamics_bnd_*); None = the model's boundary."""
    import torch
    dt = _check_tensors(model, q, qd, qdd)
    if out is None:
        out = torch.empty_like(q)
    _check_tensors(model, q, out)
    if boundary is not None:
        v0, vd0, ft = _boundary_ptrs(boundary, q)
        f = lib().rd_inverse_dynamics_bnd_f64 if dt == torch.float64 else lib().rd_inverse_dynamics_bnd_f32
        _check(f(model.handle, q.shape[1], q.data_ptr(), qd.data_ptr(), qdd.data_ptr(), v0, vd0, ft,
                 out.data_ptr(), _stream_ptr(stream)), "rd_inverse_dynamics_bnd")
        return out
    L = lib()
    f = L.rd_inverse_dynamics_f64 if dt is torch.float64 else L.rd_inverse_dynamics_f32
    rc = f(model.handle, q.shape[1], q.data_ptr(), qd.data_ptr(), qdd.data_ptr(), out.data_ptr(),
           _stream_ptr(stream, q.get_device()))
    if rc:
        _check(rc, "rd_inverse_dynamics")
    return out


def forward_dynamics(model: Model, q, qd, tau, out=None, stream=None, status=None, boundary=None):
    """qdd = FD(q, qd, tau) (Eq. 4, ABA Eq. 7-8) for B states; torch CUDA tensors [n, B].

    status: optional int32 CUDA tensor [B] (rd_forward_dynamics_ex_*): 0, or the
    1-based link of the failing pivot of that state (its qdd is NaN).
    boundary: optional per-state (V0, Vdot0, Ftip) as in inverse_dynamics (ABA only)."""
    import torch
    dt = _check_tensors(model, q, qd, tau)
    if out is None:
        out = torch.empty_like(q)
    _check_tensors(model, q, out)
    if status is not None and (status.dtype != torch.int32 or status.device != q.device
                               or status.shape != (q.shape[1],) or not status.is_contiguous()):
        raise RdError("status must be a contiguous int32 [B] tensor on the inputs' device")
    if boundary is not None:
        v0, vd0, ft = _boundary_ptrs(boundary, q)
        f = lib().rd_forward_dynamics_bnd_f64 if dt == torch.float64 else lib().rd_forward_dynamics_bnd_f32
        _check(f(model.handle, q.shape[1], q.data_ptr(), qd.data_ptr(), tau.data_ptr(), v0, vd0, ft,
                 out.data_ptr(), status.data_ptr() if status is not None else None, _stream_ptr(stream)),
               "rd_forward_dynamics_bnd")
        return out
    if status is None:
        f = lib().rd_forward_dynamics_f64 if dt == torch.float64 else lib().rd_forward_dynamics_f32
        _check(f(model.handle, q.shape[1], q.data_ptr(), qd.data_ptr(), tau.data_ptr(), out.data_ptr(),
                 _stream_ptr(stream, q.get_device())), "rd_forward_dynamics")
        return out
    if status.dtype != torch.int32 or status.device != q.device or status.shape != (q.shape[1],) \
            or not status.is_contiguous():
        raise RdError("status must be a contiguous int32 [B] tensor on the inputs' device")
    f = lib().rd_forward_dynamics_ex_f64 if dt == torch.float64 else lib().rd_forward_dynamics_ex_f32
    _check(f(model.handle, q.shape[1], q.data_ptr(), qd.data_ptr(), tau.data_ptr(), out.data_ptr(),
             status.data_ptr(), _stream_ptr(stream)), "rd_forward_dynamics_ex")
    return out


def _host_ptr(x):
    if isinstance(x, np.ndarray):
        if x.dtype != np.float64 or not x.flags.c_contiguous:
            raise RdError("host arrays must be C-contiguous float64")
        return x.ctypes.data
    if x.dtype.__str__() != "torch.float64" or x.is_cuda or not x.is_contiguous():
        raise RdError("host tensors must be contiguous CPU float64")
    return x.data_ptr()


def _host_call(fn, name, model, a, b, c, out):
    """Marshalling checks of the host-buffer API: four C-contiguous float64 host
    arrays of one shape [n, B] (the library reads/writes n*B doubles of each)."""
    if len(a.shape) != 2 or a.shape[0] != model.n:
        raise RdError(f"host arrays must be [n, B] with n = {model.n}, got {tuple(a.shape)}")
    if out is None:
        out = np.empty_like(np.asarray(a)) if isinstance(a, np.ndarray) else a.new_empty(a.shape)
    for x in (b, c, out):
        if tuple(x.shape) != tuple(a.shape):
            raise RdError(f"host arrays must share one shape {tuple(a.shape)}, got {tuple(x.shape)}")
    B = a.shape[1]
    _check(fn(model.handle, B, _host_ptr(a), _host_ptr(b), _host_ptr(c), _host_ptr(out)), name)
    return out


def inverse_dynamics_host(model: Model, q, qd, qdd, out=None):
    """End-to-end ID on HOST float64 arrays [n, B] (numpy or CPU torch, pinned preferred).

    The library pipelines H2D copies, kernels and D2H copies on its own streams
    and returns when tau is in host memory (rd_inverse_dynamics_host_f64).
    """
    return _host_call(lib().rd_inverse_dynamics_host_f64, "rd_inverse_dynamics_host_f64", model, q, qd, qdd, out)


def forward_dynamics_host(model: Model, q, qd, tau, out=None):
    """End-to-end FD on HOST float64 arrays [n, B] (rd_forward_dynamics_host_f64)."""
    return _host_call(lib().rd_forward_dynamics_host_f64, "rd_forward_dynamics_host_f64", model, q, qd, tau, out)
