"""Time the per-step skin-list build alone (CUDA events) on a configuration."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from bench import build_case
    from paper_2603_11868_b200 import ExecutionPolicy
    from paper_2603_11868_b200.physics import Simulation
    reg, grid = build_case(sys.argv[1] if len(sys.argv) > 1 else "2d1m")
    sim = Simulation(reg, grid, ExecutionPolicy.cuda(0))
    sim.initialize()
    sim.advance()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record()
        sim._build_lists(0.02 * float(sim._dev["E"].cutoff))
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(os.environ.get("SPH_B200_LIB", "main"), "skin build ms", min(ts))


if __name__ == "__main__":
    main()
