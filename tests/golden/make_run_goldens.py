"""Golden outputs of the reference's run driver (minisph report.py:117-178)
for tests/test_gpu_report.py.  Run in the build container with the reference
importable (it is not needed afterwards):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_run_goldens.py

Each run writes report.csv, probes.csv and snapshot_*.csv; the timing
columns of report.csv (wall_seconds, gpips, time_*) are machine dependent and
are blanked here.  Files land in tests/golden/run_<name>/.
"""

import csv
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
TIMING = ("wall_seconds", "gpips", "time_cll", "time_interactions", "time_integration",
          "time_sorting", "time_output")

RUNS = {
    "hydrostatic": dict(case="hydrostatic", tank=(1.0, 1.2), column=(1.0, 1.0), dp=0.02,
                        hydrostatic_init=True, probes=((0.5, 0.75), (0.5, 0.5), (0.5, 0.25)),
                        end_time=0.03, snapshots=2, precision="f32"),
    "dambreak2d": dict(case="dambreak2d", dp=0.025, end_time=0.02, snapshots=2,
                       probes=((1.0, 0.2), (0.3, 0.5)), precision="f32"),
    "kleefsman": dict(dp=0.08, end_time=0.006, snapshots=1, precision="f32"),
}


def main():
    from minisph import cases, report
    for name, kw in RUNS.items():
        if name == "kleefsman":
            import importlib.resources
            text = (importlib.resources.files("minisph") / "data" / "kleefsman.cfg").read_text()
            fields = cases.parse_config_text(text)
            fields.update(kw)
            cfg = cases.CaseConfig(**fields)
        else:
            cfg = cases.CaseConfig(**kw)
        cfg.policy = "seq"
        tmp = tempfile.mkdtemp()
        cfg.out_dir = tmp
        report.run_simulation(cfg)
        out = os.path.join(HERE, f"run_{name}")
        shutil.rmtree(out, ignore_errors=True)
        os.makedirs(out)
        for f in sorted(os.listdir(tmp)):
            if f == "report.csv":
                with open(os.path.join(tmp, f)) as fh:
                    note = fh.readline()
                    rows = list(csv.DictReader(fh))
                for r in rows:
                    for k in TIMING:
                        r[k] = ""
                with open(os.path.join(out, f), "w", newline="\n") as fh:
                    fh.write(note)
                    w = csv.DictWriter(fh, fieldnames=list(rows[0]), lineterminator="\n")
                    w.writeheader()
                    w.writerows(rows)
            elif f.endswith(".csv"):
                shutil.copy(os.path.join(tmp, f), os.path.join(out, f))
        shutil.rmtree(tmp)
        print(name, sorted(os.listdir(out)))


if __name__ == "__main__":
    sys.exit(main())
