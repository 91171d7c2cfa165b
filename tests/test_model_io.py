"""Model files (paper_1609_04493_b200.model_io): the SPEC JSON format (CPU only)."""
import json
import os

import numpy as np

import synth
from paper_1609_04493_b200 import model_io


def test_round_trip_and_inertia_assembly(tmp_path):
    r = synth.random_chain(9, 123, prismatic_fraction=0.4)
    p = os.path.join(tmp_path, "robot.json")
    model_io.save_model(r, p)
    doc = json.load(open(p))
    assert doc["version"] == 1 and len(doc["links"]) == 9
    r2 = model_io.load_model(p)
    np.testing.assert_array_equal(r2["M"], r["M"])
    np.testing.assert_array_equal(r2["S"], r["S"])
    np.testing.assert_allclose(r2["J"], r["J"], rtol=0, atol=1e-14)
    # saving the reloaded model reproduces the file exactly (link records are bit-exact)
    p2 = os.path.join(tmp_path, "robot2.json")
    model_io.save_model(r2, p2)
    assert json.load(open(p2))["links"][3]["joint_twist"] == doc["links"][3]["joint_twist"]


def test_inertia_matches_spatial_inertia_definition():
    m, c, Ic = 2.5, [0.1, -0.2, 0.05], np.diag([0.03, 0.04, 0.05])
    link = {"home_rotation": np.eye(3).ravel().tolist(), "home_translation": [0.3, 0, 0],
            "joint_twist": [0, 0, 0, 0, 0, 1], "mass": m, "com": c, "rot_inertia": Ic.ravel().tolist()}
    r = model_io.robot_from_links([link])
    np.testing.assert_allclose(r["J"][0], synth.spatial_inertia(m, c, Ic), atol=1e-15)
    # the parallel-axis term: I_o = I_c + m (|c|^2 I - c c^T)
    cc = np.asarray(c)
    np.testing.assert_allclose(r["J"][0][3:, 3:], Ic + m * (cc @ cc * np.eye(3) - np.outer(cc, cc)), atol=1e-15)


def test_bad_version_rejected(tmp_path):
    p = os.path.join(tmp_path, "bad.json")
    json.dump({"version": 2, "links": []}, open(p, "w"))
    try:
        model_io.load_model(p)
    except ValueError:
        return
    raise AssertionError("version 2 accepted")
