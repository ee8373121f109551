"""Does a push (host registry -> engine) change the cost of the next advance?
Times advance() alone, with and without a preceding push, at the same
point of the run (diagnostic for the e2e leg of bench.py)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2603_11868_b200 import ExecutionPolicy
    from paper_2603_11868_b200.physics import Simulation
    reg, grid = bench.build_case(sys.argv[1] if len(sys.argv) > 1 else "2d1m")
    sim = Simulation(reg, grid, ExecutionPolicy.cuda(0))
    sim.initialize()
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 10):
        sim.advance()

    def timed(push):
        if push:
            sim.host_modified()
            sim._ensure_device()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim.advance()
        torch.cuda.synchronize()
        return 1e3 * (time.perf_counter() - t0), sim.last_nsub, sim.last_nfix, sim._dev["E"].skin

    for push in (False, True, False, True):
        print("push" if push else "plain", [tuple(round(v, 5) if isinstance(v, float) else v
                                              for v in timed(push)) for _ in range(3)])


if __name__ == "__main__":
    main()
