"""bench.py --gpus N runs N ranks (re-executing itself under
torch.distributed.run) and the slab arm reproduces the 1-rank run bit for
bit: same nsub list, interaction count and by-id state hash after the timed
window.  Ranks share the box's one GPU and exchange host-staged over gloo
(SPH_BENCH_BACKEND=gloo: no rank's kernel waits on another's) -- the
correctness configuration of the multi-GPU bench path."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _bench(*extra, env_extra=None):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT"):
        env.pop(k, None)
    env.update(env_extra or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "2dref",
                          "--steps", "3", "--warmup", "3", "--digest", "--no-cpu-baseline",
                          *extra], capture_output=True, text=True, timeout=900, cwd=ROOT,
                         env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("world", [2, 3])
def test_bench_gpus_n_runs_n_ranks_bitwise_equal_to_one(world):
    one = _bench()
    many = _bench("--gpus", str(world), env_extra={"SPH_BENCH_BACKEND": "gloo"})
    assert one["n_gpus"] == 1 and many["n_gpus"] == world
    assert many["nsub_per_step"] == one["nsub_per_step"]
    assert many["interactions_total"] == one["interactions_total"]
    assert many["state_sha256"] == one["state_sha256"]
    assert len(many["slab_cuts"]) == world + 1
    assert many["e2e"]["nsub_per_step"] == one["nsub_per_step"]
    assert one["e2e"]["nsub_per_step"] == one["nsub_per_step"]
    assert many["config"]["particles"] == one["config"]["particles"]
