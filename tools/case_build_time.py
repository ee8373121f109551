"""Case placement time: host builder (cases.build_case, the reference's numpy
lattice) vs device placement (cases.build_case_device, csrc/cases.cu), and
the placement kernels' own device time.  Prints one JSON line per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_11868_b200 import cases  # noqa: E402

DP = {"3d4m": 0.00608, "3d16m": 0.00371, "3d64m": 0.00229, "2d1m": 0.00144}


def cfg_of(name):
    if name.startswith("2d"):
        return cases.CaseConfig(case="dambreak2d", dp=DP[name], precision="f32")
    return cases.kleefsman_config(dp=DP[name], precision="f32")


def main():
    names = sys.argv[1:] or ["2d1m", "3d4m", "3d16m"]
    torch.zeros(1, device="cuda")
    for name in names:
        cfg = cfg_of(name)
        cases.build_case_device(cfg)          # warm (module load, allocator)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reg, grid, st = cases.build_case_device(cfg)
        torch.cuda.synchronize()
        t_dev = time.perf_counter() - t0
        n = reg.particle_count
        del st
        t_host = None
        if name != "3d64m":
            t0 = time.perf_counter()
            hreg, _ = cases.build_case(cfg)
            t_host = time.perf_counter() - t0
            assert hreg.particle_count == n
        print(json.dumps({"config": name, "particles": n, "device_build_s": t_dev,
                          "host_build_s": t_host}), flush=True)


if __name__ == "__main__":
    main()
