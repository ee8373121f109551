"""report.py file formats against the reference's own files (CPU): a registry
rebuilt from a reference snapshot writes that snapshot back byte for byte;
the probe series and report rows keep the reference's layout."""

import csv
import os

import numpy as np

from golden.make_run_goldens import HERE, TIMING
from paper_2603_11868_b200 import report
from paper_2603_11868_b200.physics import setup_state_variables
from paper_2603_11868_b200.variables import VariableRegistry


def _snapshot_registry(path):
    with open(path) as fh:
        head = fh.readline().strip().split(",")
        data = np.array([ln.strip().split(",") for ln in fh if ln.strip()])
    d = sum(1 for h in head if h.startswith("x"))
    n = data.shape[0]
    reg = VariableRegistry(n, d, dtype=np.float32)
    setup_state_variables(reg)
    # scramble the physical order: the writer sorts by id
    perm = np.random.default_rng(1).permutation(n)
    col = {h: data[perm, k] for k, h in enumerate(head)}
    reg.raw_view("id")[:] = col["id"].astype(np.uint32)
    for k in range(d):
        reg.raw_view("x")[:, k] = col[f"x{k}"].astype(np.float64).astype(np.float32)
        reg.raw_view("v")[:, k] = col[f"v{k}"].astype(np.float64).astype(np.float32)
    reg.raw_view("rho")[:] = col["rho"].astype(np.float64).astype(np.float32)
    reg.raw_view("p")[:] = col["p"].astype(np.float64).astype(np.float32)
    return reg


def test_snapshot_writer_reproduces_reference_files(tmp_path):
    for run in ("run_dambreak2d", "run_kleefsman"):
        gold = os.path.join(HERE, run, "snapshot_0000.csv")
        reg = _snapshot_registry(gold)
        out = tmp_path / f"{run}.csv"
        report.write_snapshot(reg, str(out))
        assert out.read_bytes() == open(gold, "rb").read(), run


def test_probe_series_layout(tmp_path):
    gold = os.path.join(HERE, "run_hydrostatic", "probes.csv")
    with open(gold) as fh:
        fh.readline()
        rows = [[float(v) for v in ln.split(",")] for ln in fh]
    probes = ((0.5, 0.75), (0.5, 0.5), (0.5, 0.25))
    out = tmp_path / "probes.csv"
    report.write_probe_series(rows, probes, str(out))
    assert out.read_bytes() == open(gold, "rb").read()


def test_report_row_schema(tmp_path):
    rep = report.RunReport(case="hydrostatic", policy="cuda", workers=4, precision="f32",
                           particle_count=3028, fluid_count=2500, step_count=30,
                           end_time=0.03, simulated_time=0.03, interaction_count=9101500,
                           wall_seconds=2.0, substep_count=60)
    rep.gpips = report.compute_gpips(rep.interaction_count, rep.wall_seconds)

    class Cfg:
        out_dir = str(tmp_path)
    report.write_report(rep, Cfg)
    rows = report.read_report_csv(str(tmp_path / "report.csv"))
    with open(os.path.join(HERE, "run_hydrostatic", "report.csv")) as fh:
        fh.readline()
        ref = next(csv.DictReader(fh))
    assert list(rows[0])[:len(ref)] == list(ref)     # the reference's columns, in order
    for k, v in ref.items():
        if k not in TIMING and k != "policy":
            assert rows[0][k] == v, k
    assert float(rows[0]["particle_updates_per_s"]) == 3028 * 30 / 2.0
    assert (tmp_path / "report.txt").read_text().startswith("case:            hydrostatic")


def test_binary_snapshot_holds_the_csv_values_by_id(tmp_path):
    """write_snapshot_npy (host-authoritative path) writes row = id,
    x*, v*, rho, p: the values the reference-format CSV prints."""
    from paper_2603_11868_b200.neighborhood import UniformGrid
    from paper_2603_11868_b200.physics import Simulation
    from paper_2603_11868_b200 import ExecutionPolicy
    gold = os.path.join(HERE, "run_kleefsman", "snapshot_0000.csv")
    reg = _snapshot_registry(gold)
    sim = Simulation(reg, UniformGrid.from_bounds((0, 0, 0), (1, 1, 1), 0.1),
                     ExecutionPolicy.sequenced())
    out = tmp_path / "s.npy"
    report.write_snapshot_npy(sim, str(out))
    rows = np.load(out)
    with open(gold) as fh:
        fh.readline()
        txt = np.loadtxt(fh, delimiter=",", dtype=np.float64, ndmin=2)
    assert rows.dtype == np.float32 and rows.shape == (txt.shape[0], txt.shape[1] - 1)
    assert np.array_equal(rows.astype(np.float64), txt[np.argsort(txt[:, 0]), 1:])
