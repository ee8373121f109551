"""profiles/ncu_traffic.json from tools/ncu_summary.py text summaries (the
.ncu-rep files stay on the GPU box): per sub-step kernel the mean DRAM bytes,
issue-slot utilisation and warp instructions per launch.
usage: python tools/traffic_from_summary.py OUT.json CONFIG=SUMMARY.txt ..."""
import json
import re
import sys

NAMES = {"k_kick_drift": "kick_drift", "k_cont_du": "continuity_du",
         "k_wall": "wall_pressure", "k_wall_g": "wall_pressure", "k_mark_refresh": "list_filter", "k_mom": "momentum_kick", "k_mark": "list_filter",
         "k_mask": "list_filter", "k_skin_tile": "skin_build", "k_skin_warp": "skin_build"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def parse(path):
    acc, cur = {}, None
    for line in open(path):
        if line.startswith("----"):
            base = line.split()[2].split("<")[0].split("(")[0]
            cur = NAMES.get(base)
            if cur:
                acc.setdefault(cur, []).append({})
            continue
        m = re.match(r"\s+(\S+)\s+([\d.]+)\s*(\S*)", line)
        if cur and m:
            acc[cur][-1][m.group(1)] = float(m.group(2)) * SCALE.get(m.group(3), 1)
    out = {}
    for k, runs in acc.items():
        n = len(runs)
        out[k] = {"dram_bytes": sum(r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)
                                    for r in runs) / n,
                  "issue_active_pct": sum(r.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0)
                                          for r in runs) / n,
                  "warp_inst": sum(r.get("smsp__inst_executed.sum", 0) for r in runs) / n,
                  "launches": n}
    return out


def main(out, specs):
    res = {}
    for s in specs:
        cfg, path = s.split("=", 1)
        res[cfg] = parse(path)
        res[cfg]["_source"] = path.split("/")[-1]
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
