"""Shared test helpers: golden fixtures, hashing, case construction."""

import hashlib
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")

FIELDS = ("x", "v", "rho", "p", "m", "Vol", "drho", "dvdt", "rho_scratch",
          "id", "wall", "nnb", "oflow")

TRAJ = {
    # tag: (case factory kwargs, precision)
    "dambreak2d_f32": dict(kind="2d", dp=0.025, precision="f32"),
    "dambreak2d_f64": dict(kind="2d", dp=0.025, precision="f64"),
    "dambreak2d_coarse_f32": dict(kind="2d", dp=0.05, precision="f32"),
    "kleefsman3d_f32": dict(kind="3d", dp=0.04, precision="f32"),
}


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def by_id(arr, ids):
    return arr[np.argsort(ids, kind="stable")]


def case(tag):
    from paper_2603_11868_b200 import cases
    spec = TRAJ[tag]
    if spec["kind"] == "2d":
        cfg = cases.CaseConfig(case="dambreak2d", dp=spec["dp"],
                               precision=spec["precision"])
    else:
        cfg = cases.kleefsman_config(dp=spec["dp"], precision=spec["precision"])
    return cases.build_case(cfg)


def mismatched(get, z, step, physical_get=None):
    """Fields whose by-id (and optionally physical) hash differs at step."""
    bad = [f for f in FIELDS if sha(get(f)) != z["hid_" + f][step]]
    if physical_get is not None:
        bad += [f + "@phys" for f in FIELDS
                if sha(physical_get(f)) != z["hph_" + f][step]]
    return bad
