"""The run driver (report.py / cli.py) on the device engine
vs the reference's own run driver: report.csv (all but the machine-dependent
timing columns and the policy name), probes.csv and every snapshot file
byte for byte (tests/golden/make_run_goldens.py)."""

import csv
import os

import pytest

from golden.make_run_goldens import HERE, RUNS, TIMING
from paper_2603_11868_b200 import cases, report

pytestmark = pytest.mark.gpu


def _config(name, out_dir):
    kw = dict(RUNS[name])
    cfg = cases.kleefsman_config(**kw) if name == "kleefsman" else cases.CaseConfig(**kw)
    cfg.policy = "cuda"
    cfg.out_dir = str(out_dir)
    return cfg


def _rows(path):
    with open(path) as fh:
        fh.readline()
        return list(csv.DictReader(fh))


@pytest.mark.parametrize("name", sorted(RUNS))
def test_run_driver_outputs_match_reference(name, tmp_path):
    rep = report.run_simulation(_config(name, tmp_path))
    gold = os.path.join(HERE, f"run_{name}")
    assert sorted(f for f in os.listdir(tmp_path) if f.endswith(".csv")) == \
        sorted(os.listdir(gold))
    ours, ref = _rows(tmp_path / "report.csv")[0], _rows(os.path.join(gold, "report.csv"))[0]
    for k, v in ref.items():
        if k in TIMING or k == "policy":
            continue
        assert ours[k] == v, k
    assert float(ours["particle_updates_per_s"]) > 0
    for f in os.listdir(gold):
        if f != "report.csv":
            assert (tmp_path / f).read_bytes() == open(os.path.join(gold, f), "rb").read(), f
    assert rep.step_count > 0 and not rep.aborted


def test_cli_runs_a_case(tmp_path, capsys):
    from paper_2603_11868_b200.cli import main
    rc = main(["hydrostatic", "--policy", "cuda", "--end-time", "0.005", "--out",
               str(tmp_path), "--report", "csv", "--snapshots", "1"])
    assert rc == 0
    line = capsys.readouterr().out.strip().splitlines()[-1].split(",")
    assert line[0] == "hydrostatic" and line[1] == "cuda"
    assert (tmp_path / "report.txt").exists() and (tmp_path / "snapshot_0000.csv").exists()


@pytest.mark.parametrize("name", sorted(RUNS))
def test_binary_snapshots_equal_the_csv_snapshots(name, tmp_path):
    """snapshot_format="npy" (device gather by id, one D2H copy) holds the
    bits the reference-format CSV snapshots print: rows by id, x*, v*, rho, p."""
    import numpy as np
    csv_dir, npy_dir = tmp_path / "csv", tmp_path / "npy"
    report.run_simulation(_config(name, csv_dir))
    cfg = _config(name, npy_dir)
    cfg.snapshot_format = "npy"
    report.run_simulation(cfg)
    snaps = sorted(f for f in os.listdir(csv_dir) if f.startswith("snapshot_"))
    assert snaps
    assert sorted(f for f in os.listdir(npy_dir) if f.startswith("snapshot_")) == \
        [f[:-4] + ".npy" for f in snaps]
    for f in snaps:
        rows = np.load(npy_dir / (f[:-4] + ".npy"))
        with open(csv_dir / f) as fh:
            head = fh.readline().strip().split(",")
            txt = np.loadtxt(fh, delimiter=",", dtype=np.float64, ndmin=2)
        assert head[0] == "id" and rows.shape == (txt.shape[0], len(head) - 1)
        assert np.array_equal(txt[:, 0], np.arange(rows.shape[0]))
        # %.17g round-trips binary64 exactly; the run dtype widens exactly
        assert np.array_equal(rows.astype(np.float64), txt[:, 1:])
