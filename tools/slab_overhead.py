"""Where a slab-path step (distributed.DistributedSimulation, one rank) spends
its time beyond the single-GPU engine step: wall-clock per phase with a
device synchronisation after each (diagnostic)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist
    for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_ADDR", "127.0.0.1"),
                 ("MASTER_PORT", "29541")):
        os.environ.setdefault(k, v)
    dist.init_process_group("nccl")
    import bench
    from paper_2603_11868_b200 import distributed as D
    from paper_2603_11868_b200.physics import force_scalars
    name = sys.argv[1] if len(sys.argv) > 1 else "2d1m"
    reg, grid = bench.build_case(name)
    dev = torch.device("cuda", 0)
    owned = {f: reg.raw_view(f) for f in D.FIELDS}
    sing = {k: reg.singular(k) for k in ("rho0", "c0", "h", "g")}
    be = D.EngineBackend(force_scalars(reg, grid), sing, grid, dev)
    sim = D.DistributedSimulation(D.Comm(dev), be, grid, owned, sing)
    T = {}

    def wrap(obj, name, key):
        f = getattr(obj, name)

        def g(*a, **k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = f(*a, **k)
            torch.cuda.synchronize()
            T[key] = T.get(key, 0.0) + time.perf_counter() - t0
            return r
        setattr(obj, name, g)

    for nm in ("_migrate", "_build_local", "_rebalance"):
        wrap(sim, nm, nm)
    for nm in ("load", "set_halo", "norms", "prepare", "substeps", "counters", "stability",
               "export_owned", "kick_drift", "continuity_du", "wall_pressure", "momentum_kick"):
        if hasattr(be, nm):
            wrap(be, nm, "be." + nm)
    sim.initialize()
    for _ in range(3):
        sim.advance()
    T.clear()
    K = 4
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        sim.advance()
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print(f"{name}: {1e3 * tot / K:.2f} ms/step (native_loop={be.native_loop})")
    for k, v in sorted(T.items(), key=lambda kv: -kv[1]):
        print(f"  {k:22s} {1e3 * v / K:8.3f} ms")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
