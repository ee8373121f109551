"""bench.py's contract pieces that run without a GPU: the reference arm's
JSON line (CPU oracle port on the reference's own 2D case), the byte model,
and the clock sampler's filtering of rows to the timed window."""

import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_arm_prints_one_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "2dref", "--steps", "2", "--warmup", "3",
                          "--cpu-budget", "20"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_under_gpus_2_respawns_one_rank_line():
    """`bench.py --gpus 2` without a launcher re-executes under
    torch.distributed.run; only rank 0 runs the reference arm and prints."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--config", "2dref", "--steps", "1", "--warmup", "3",
                          "--cpu-budget", "10"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    assert d["config"] == bench.config_of("2dref", 2, 5153, 3200, 1953, 7656)


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_roofline_bytes_follow_survey_8d():
    # momentum: nf (20d + 20); 2D 1M: 963,966 x 60 = 57.8 MB (VERDICT r1 recompute)
    assert bench.kernel_bytes("momentum_kick", 2, 997518, 963966, 33552) == 963966 * 60
    assert bench.kernel_bytes("continuity_du", 3, 10, 7, 3) == 7 * 48
    assert bench.kernel_bytes("wall_pressure", 3, 10, 7, 3) == 3 * 28
    # neighbour-list bytes are reported separately, never as algorithmic
    assert bench.list_bytes("momentum_kick", 100, 0, 0, 0) == 400


def test_step_byte_model_matches_survey_table():
    # config 1 B_sub = 109.1, B_step = 103.9 (d = 2, w = 0.379)
    n, nw = 5153, 1953
    b1 = bench.step_bytes_model(2, n, n - nw, nw, 1, 7656, 2)
    b3 = bench.step_bytes_model(2, n, n - nw, nw, 3, 7656, 2)
    assert abs((b3 - b1) / 2 - 109.1) < 0.2
    assert abs(b1 - 109.1 - 103.9) < 0.5


class _FakeProc:
    def __init__(self, lines):
        self.stdout = iter(lines)

    def terminate(self):
        pass

    def wait(self, timeout=None):
        return 0


def test_clock_sampler_keeps_rows_of_the_timed_window():
    s = bench.ClockSampler(0)
    s.proc = _FakeProc([])
    s.thread = threading.Thread(target=lambda: None)
    s.thread.start()
    now = time.perf_counter()
    s.rows = [(now - 1.0, ["900", "1965", "Not Active", "Not Active", "Not Active", "Active"]),
              (now + 0.01, ["1965", "1965", "Not Active", "Not Active", "Not Active",
                            "Not Active"]),
              (now + 5.0, ["100", "1965", "Active", "Not Active", "Not Active", "Not Active"])]
    s.t0, s.t1 = now, now + 0.02
    c = s.stop()
    assert c["samples"] == 1 and c["sm_mhz"] == 1965.0 and c["reasons"] == []
