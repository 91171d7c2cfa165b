"""C-ABI contract checks that need no GPU: the library loads, exports every
symbol include/rd.h declares, and rejects bad models/arguments before touching
CUDA (RD_E_MODEL / RD_E_ARG with messages naming the link)."""
import ctypes
import os
import re

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rd():
    import paper_1609_04493_b200 as rd
    if not os.path.exists(rd.LIB_PATH):
        from paper_1609_04493_b200 import _build
        _build.build()
    return rd


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "rd.h")).read()
    return sorted(set(re.findall(r"\b(rd_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported(rd):
    syms = header_symbols()
    assert len(syms) >= 14
    L = rd.lib()
    for s in syms:
        assert hasattr(L, s), f"librd.so does not export {s}"
    assert sorted(rd.EXPORTS) == syms


def test_version_and_error_strings(rd):
    assert b"sm_100a" in rd.lib().rd_version()
    assert isinstance(rd.lib().rd_last_error(), bytes)


def _create(rd, M, S, J, g=(0, 0, -9.81)):
    L = rd.lib()
    h = ctypes.c_void_p()
    M, S, J = (np.ascontiguousarray(x, dtype=np.float64) for x in (M, S, J))
    g = np.asarray(g, dtype=np.float64)
    rc = L.rd_model_create(S.shape[0], rd._dptr(M), rd._dptr(S), rd._dptr(J), rd._dptr(g), ctypes.byref(h))
    return rc, L.rd_last_error().decode(), h


def test_invalid_models_rejected_naming_links(rd):
    r = synth.random_chain(4, 3)
    M, S, J = r["M"].copy(), r["S"].copy(), r["J"].copy()
    S[1, 3:] *= 0.5                                # angular norm 0.5
    J[2, 3:, 3:] -= 10.0 * np.eye(3)               # negative eigenvalue
    M[3, :3, :3] *= 1.1                            # non-orthonormal rotation
    rc, msg, _ = _create(rd, M, S, J)
    assert rc == 2, msg                            # RD_E_MODEL
    assert "link 2" in msg and "angular norm" in msg
    assert "link 3" in msg and "positive definite" in msg
    assert "link 4" in msg and "orthonormal" in msg


def test_non_rigid_inertia_rejected(rd):
    r = synth.random_chain(2, 4)
    J = r["J"].copy()
    J[0, 0, 1] = J[0, 1, 0] = 0.3                  # upper-left block not m*I
    rc, msg, _ = _create(rd, r["M"], r["S"], J)
    assert rc == 2 and "link 1" in msg and "rigid" in msg


def test_argument_errors(rd):
    L = rd.lib()
    h = ctypes.c_void_p()
    g = np.zeros(3)
    assert L.rd_model_create(0, None, None, None, rd._dptr(g), ctypes.byref(h)) == 1   # n < 1
    assert L.rd_inverse_dynamics_f64(None, 10, None, None, None, None, None) == 1      # null model
    assert L.rd_model_destroy(None) == 0


def test_oracle_and_product_share_no_code():
    # The oracle is test infrastructure: the product package never imports it and
    # no source under paper_1609_04493_b200/ includes oracle/ files (and vice versa).
    pkg = os.path.join(ROOT, "paper_1609_04493_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "oracle.cpp" not in txt and "liboracle" not in txt, f
    otxt = open(os.path.join(ROOT, "oracle", "oracle.cpp")).read()
    assert "rd_internal" not in otxt and "rd_math" not in otxt and "rd.h" not in otxt


# ----------------------------------------------------------- the ABI from plain C
def _build_c_example(rd, tmp_path):
    """gcc the plain-C99 example (no CUDA headers, no Python) against include/rd.h and librd.so."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    exe = str(tmp_path / "planar2_c")
    libdir = os.path.dirname(rd.LIB_PATH)
    cmd = [cc, "-O2", "-std=c99", "-Wall", "-Wextra", "-Werror", f"-I{os.path.join(ROOT, 'include')}",
           os.path.join(ROOT, "examples", "planar2_c.c"), f"-L{libdir}", "-lrd", f"-Wl,-rpath,{libdir}", "-lm",
           "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_builds_against_the_header(rd, tmp_path):
    # include/rd.h is plain C (C99, no torch / CUDA types) and librd.so links from C
    _build_c_example(rd, tmp_path)


@pytest.mark.gpu
def test_c_example_runs(rd, tmp_path):
    # examples/planar2_c.c: C1's robot through rd_model_create and the host-buffer ID / FD
    # calls, checked in C against the textbook closed form and the FD round trip (1e-10)
    import subprocess
    exe = _build_c_example(rd, tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "planar2_c: ok" in r.stdout
