"""Stretch of the modified-DH frames the library builds for a chain (numpy replica of
capi.cu build_dh): max_i max(|a_i|, |d_i|, |c_i|) over the largest joint-frame link offset.
Nearly parallel consecutive joint axes put the common normal (and so the DH origin) far
from the links.  usage: python tools/dh_conditioning.py  (development aid)"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def joint_frames(robot):
    """G_i with z_i = joint axis (as capi: joint frames from (M, S))."""
    M, S = robot["M"], robot["S"]
    n = len(M)
    G, acc = [], np.eye(4)
    for i in range(n):
        acc = acc @ M[i]
        v, w = S[i, :3], S[i, 3:]
        if np.linalg.norm(w) > 0.5:        # revolute: axis w through point r = w x v (zero pitch)
            z, r = w / np.linalg.norm(w), np.cross(w, v)
        else:                              # prismatic: direction v through the origin
            z, r = v / np.linalg.norm(v), np.zeros(3)
        x = np.cross([0, 1, 0], z) if abs(z[1]) < 0.9 else np.cross([1, 0, 0], z)
        x /= np.linalg.norm(x)
        J = np.eye(4); J[:3, 0] = x; J[:3, 1] = np.cross(z, x); J[:3, 2] = z; J[:3, 3] = r
        G.append(acc @ J)
    return G


def stretch(robot):
    G = joint_frames(robot)
    n = len(G)
    worst = 0.0
    for i in range(n - 1):
        z, o, z2, o2 = G[i][:3, 2], G[i][:3, 3], G[i + 1][:3, 2], G[i + 1][:3, 3]
        cz = np.cross(z, z2); cn = np.linalg.norm(cz); w0 = o - o2
        if cn > 1e-9:
            b, dd, e = z @ z2, z @ w0, z2 @ w0
            den = 1 - b * b
            s1 = (b * e - dd) / den
            P = o + s1 * z
            worst = max(worst, abs(s1), np.linalg.norm(P - o2))
    L = max(np.linalg.norm(m[:3, 3]) for m in robot["M"])
    return worst / L


if __name__ == "__main__":
    for n, seed in ((30, 1030), (100, 1100), (100, 1800), (200, 1900), (400, 2100), (1000, 1700), (1000, 2700)):
        r = synth.random_chain(n, seed, prismatic_fraction=0.05 if seed in (1700, 1800, 1900, 2100, 2700) else 0.0)
        print(n, seed, f"stretch {stretch(r):.3g}")
