"""Robot model files (host-side I/O, no dynamics): the JSON text format of the
paper's reference program spec (SPEC.md "External Interfaces"):

    {"version": 1, "links": [{"home_rotation": [9, row-major], "home_translation": [3],
      "joint_twist": [6, linear then angular], "mass": m, "com": [3],
      "rot_inertia": [9, row-major, about the centre of mass]}, ...]}

Link i's home transform M_i = f_{i-1,i}(q_i = 0) (frame i -> frame i-1)
and twist S_i are in link i's frame; the spatial inertia about the link origin
is assembled as J = [[m I, -m[c]], [m[c], I_c - m[c][c]]] ((v, w) ordering,
DESIGN.md A1).  Numbers are written as shortest round-trip decimals (at most 17
significant digits), so the link records survive a save/load bit-exactly.  Returns / accepts the dict(M, S, J) that
`Model.from_robot` takes; validation happens in rd_model_create.
"""
from __future__ import annotations

import json

import numpy as np

__all__ = ["load_model", "save_model", "robot_from_links"]


def _skew(c):
    return np.array([[0.0, -c[2], c[1]], [c[2], 0.0, -c[0]], [-c[1], c[0], 0.0]])


def robot_from_links(links) -> dict:
    """dict(M [n,4,4], S [n,6], J [n,6,6]) from a list of link records."""
    n = len(links)
    if n < 1:
        raise ValueError("model has no links")
    M = np.zeros((n, 4, 4))
    S = np.zeros((n, 6))
    J = np.zeros((n, 6, 6))
    for i, L in enumerate(links):
        R = np.asarray(L["home_rotation"], dtype=np.float64).reshape(3, 3)
        M[i, :3, :3] = R
        M[i, :3, 3] = np.asarray(L["home_translation"], dtype=np.float64)
        M[i, 3, 3] = 1.0
        S[i] = np.asarray(L["joint_twist"], dtype=np.float64)
        m = float(L["mass"])
        c = np.asarray(L["com"], dtype=np.float64)
        Ic = np.asarray(L["rot_inertia"], dtype=np.float64).reshape(3, 3)
        C = _skew(c)
        J[i, :3, :3] = m * np.eye(3)
        J[i, :3, 3:] = -m * C
        J[i, 3:, :3] = m * C
        J[i, 3:, 3:] = Ic - m * C @ C
    return {"M": M, "S": S, "J": J}


def load_model(path: str) -> dict:
    with open(path) as f:
        doc = json.load(f)
    if doc.get("version") != 1:
        raise ValueError(f"{path}: unsupported model version {doc.get('version')!r}")
    return robot_from_links(doc["links"])


def _links_from_robot(robot: dict):
    M, S, J = (np.asarray(robot[k], dtype=np.float64) for k in ("M", "S", "J"))
    links = []
    for i in range(S.shape[0]):
        m = J[i, 0, 0]
        # [m c] is the lower-left block; I_c = I_o + m[c][c]
        mc = np.array([J[i, 5, 1], J[i, 3, 2], J[i, 4, 0]])
        c = mc / m
        C = _skew(c)
        Ic = J[i, 3:, 3:] + m * C @ C
        links.append({"home_rotation": M[i, :3, :3].ravel().tolist(),
                      "home_translation": M[i, :3, 3].tolist(),
                      "joint_twist": S[i].tolist(), "mass": float(m), "com": c.tolist(),
                      "rot_inertia": Ic.ravel().tolist()})
    return links


def save_model(robot: dict, path: str) -> None:
    """Write dict(M, S, J) as a model file.  Python's float repr is the shortest
    string that round-trips, i.e. at most 17 significant digits, so the link
    records reload bit-exactly (J is re-assembled from m, c, I_c: equal to the
    input to rounding)."""
    doc = {"version": 1, "links": _links_from_robot(robot)}
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
