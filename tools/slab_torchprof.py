"""Kernel-level breakdown of one slab-orchestrated step on one rank
(torch.profiler; diagnostic for the slab overhead)."""
import os, sys
sys.path.insert(0, os.getcwd())
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29545")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import torch
torch.cuda.set_device(0)
torch.distributed.init_process_group("nccl")
from bench import build_case
from paper_2603_11868_b200 import distributed as D
from paper_2603_11868_b200.physics import force_scalars
cfg = sys.argv[1] if len(sys.argv) > 1 else "3d4m"
reg, grid = build_case(cfg)
owned = {f: reg.raw_view(f) for f in D.FIELDS}
sing = {k: reg.singular(k) for k in ("rho0", "c0", "h", "g")}
comm = D.Comm("cuda:0")
be = D.EngineBackend(force_scalars(reg, grid), sing, grid, "cuda:0")
sim = D.DistributedSimulation(comm, be, grid, owned, sing)
sim.initialize()
for _ in range(2):
    sim.advance()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    sim._load_step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
