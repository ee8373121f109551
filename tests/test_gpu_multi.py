"""Real multi-GPU runs (NCCL between distinct GPUs): `bench.py --gpus N`
over N >= 2 visible B200s must reproduce the one-GPU run bit for bit (same
nsub list, interaction count and by-id state hash after the timed window),
for the bounded dam break and the periodic ring.  The pool's boxes have one
GPU, so these are skipped there; the gloo / shared-GPU variants
(tests/test_gpu_bench_slab.py, tests/test_gpu_distributed.py) cover the same
code paths host-staged."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:   # pragma: no cover
        return 0


def _bench(*extra):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT", "SPH_BENCH_BACKEND"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3",
                          "--warmup", "3", "--digest", "--no-cpu-baseline", "--no-e2e", *extra],
                         capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs (NCCL between devices)")
@pytest.mark.parametrize("config", ["2dref", "3d4m"])
def test_nccl_slabs_equal_one_gpu(config):
    world = min(_ngpu(), 4)
    one = _bench("--config", config, "--slab")
    many = _bench("--config", config, "--gpus", str(world))
    assert many["n_gpus"] == world
    assert many["nsub_per_step"] == one["nsub_per_step"]
    assert many["interactions_total"] == one["interactions_total"]
    assert many["state_sha256"] == one["state_sha256"]


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs (NCCL between devices)")
def test_nccl_periodic_ring_runs():
    """Config 5's weak-scaled Taylor-Green ring (the box grows with N, so
    only the run itself is checked here; the ring's bitwise equality with
    one rank is tests/test_gpu_distributed.py's tg cases)."""
    world = min(_ngpu(), 4)
    many = _bench("--config", "tg8m", "--gpus", str(world))
    assert many["n_gpus"] == world and many["value"] > 0
