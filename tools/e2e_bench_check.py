"""bench.e2e_run vs its phases on the same simulation state (diagnostic)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2603_11868_b200 import ExecutionPolicy
    from paper_2603_11868_b200.physics import Simulation, _ENGINE_FIELDS
    reg, grid = bench.build_case(sys.argv[1] if len(sys.argv) > 1 else "2d1m")
    sim = Simulation(reg, grid, ExecutionPolicy.cuda(0))
    sim.initialize()
    for _ in range(3):
        sim.advance()
    dev = torch.device("cuda", 0)
    for rep in range(3):
        r = bench.e2e_run(sim, reg, 3, 1, dev)
        print("e2e_run", r["value"], 1e3 * reg.particle_count / r["value"], "ms/step")
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim._ensure_device()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sim.advance()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        for f in _ENGINE_FIELDS:
            reg.view(f)
        t3 = time.perf_counter()
        print(f"push {1e3*(t1-t0):.2f} advance {1e3*(t2-t1):.2f} pull {1e3*(t3-t2):.2f}")


if __name__ == "__main__":
    main()
