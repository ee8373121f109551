"""Wall-clock breakdown of slab-orchestrated steps on one rank (NCCL,
no peers) by phase, synchronising between phases (diagnostic for the slab
overhead): python tools/slab_phases.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29546"), ("RANK", "0"),
             ("WORLD_SIZE", "1")):
    os.environ.setdefault(k, v)
import torch  # noqa: E402

torch.cuda.set_device(0)
torch.distributed.init_process_group("nccl")
from paper_2603_11868_b200 import cases, distributed as D  # noqa: E402
from paper_2603_11868_b200.physics import force_scalars  # noqa: E402
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "3d4m"
reg, grid, owned = cases.build_slab_case(bench.case_config(cfg), 0, 1, torch.device("cuda", 0))
sing = {k: reg.singular(k) for k in ("rho0", "c0", "h", "g")}
comm = D.Comm("cuda:0")
be = D.EngineBackend(force_scalars(reg, grid), sing, grid, "cuda:0")
sim = D.DistributedSimulation(comm, be, grid, owned, sing)
acc = {}


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
        return r
    return w


for name in ("_migrate_rows",):
    pass
sim._load_step = timed("load (classify, exchange, assemble, push, halo plan)", sim._load_step)
be.norms = timed("norms", be.norms)
be.prepare = timed("skin build", be.prepare)
be.substeps = timed("sub-steps", be.substeps)
be.counters = timed("counters", be.counters)
be.export_owned = timed("export (pull)", be.export_owned)
be.stability = timed("stability", be.stability)
sim.initialize()
for _ in range(3):
    sim.advance()
acc.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
K = 5
for _ in range(K):
    sim.advance()
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / K
print(f"{cfg}: {1e3 * tot:.2f} ms per step (synchronised phases)")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {1e3 * v / K:8.3f} ms  {k}")
torch.distributed.destroy_process_group()
