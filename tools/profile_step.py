"""Small fixed workload for ncu: build a configuration, initialize, run
--warmup untimed steps and --steps steps through the engine.  Used for the
launch lists and `ncu --set full` captures committed under profiles/."""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2d1m")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    import torch
    from bench import build_case
    from paper_2603_11868_b200 import ExecutionPolicy
    from paper_2603_11868_b200.physics import Simulation
    reg, grid = build_case(args.config)
    sim = Simulation(reg, grid, ExecutionPolicy.cuda(0))
    sim.initialize()
    for _ in range(args.warmup + args.steps):
        sim.advance()
    torch.cuda.synchronize()
    print(f"ok {args.config} N={reg.particle_count} steps={sim.step_count} "
          f"nsub={sim.last_nsub} interactions={sim.interaction_count}")


if __name__ == "__main__":
    main()
