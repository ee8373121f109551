import os, time, sys
sys.path.insert(0, os.getcwd())
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29544")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import torch, numpy as np
torch.cuda.set_device(0)
torch.distributed.init_process_group("nccl")
from bench import build_case
from paper_2603_11868_b200 import distributed as D
from paper_2603_11868_b200.physics import force_scalars
cfg = sys.argv[1] if len(sys.argv) > 1 else "2d1m"
reg, grid = build_case(cfg)
owned = {f: reg.raw_view(f) for f in D.FIELDS}
sing = {k: reg.singular(k) for k in ("rho0", "c0", "h", "g")}
comm = D.Comm("cuda:0")
be = D.EngineBackend(force_scalars(reg, grid), sing, grid, "cuda:0")
sim = D.DistributedSimulation(comm, be, grid, owned, sing)
sim.initialize()
for _ in range(2): sim.advance()
# instrument
T = {}
def wrap(obj, name):
    f = getattr(obj, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); T[name] = T.get(name, 0) + time.perf_counter() - t0
        return r
    setattr(obj, name, g)
for n in ("_rebalance", "_migrate", "_build_local", "_finish_counts"):
    wrap(sim, n)
for n in ("load", "set_halo", "norms", "prepare", "substeps", "counters", "stability", "export_owned", "planes"):
    wrap(be, n)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(3): sim.advance()
torch.cuda.synchronize(); tot = time.perf_counter() - t0
print(cfg, "per step ms", 1e3 * tot / 3)
for k, v in sorted(T.items(), key=lambda x: -x[1]): print(f"  {k:15s} {1e3*v/3:8.2f} ms")
