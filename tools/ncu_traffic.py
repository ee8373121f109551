"""Per-launch DRAM traffic, issue-slot utilisation and instruction count of
the engine's kernels from `ncu --set full` captures ->
profiles/ncu_traffic.json (read by bench.py's roofline `traffic` and
`issue_active_frac` fields).

usage: python tools/ncu_traffic.py OUT.json CONFIG=REP.ncu-rep [CONFIG=REP ...]
"""
import csv
import io
import json
import subprocess
import sys

# csrc kernel -> bench.py sub-step name (physics.SUBSTEP_KERNELS)
NAMES = {"k_kick_drift": "kick_drift", "k_cont_du": "continuity_du",
         "k_wall": "wall_pressure", "k_wall_g": "wall_pressure", "k_mark_refresh": "list_filter", "k_mom": "momentum_kick",
         "k_skin_tile": "skin_build", "k_skin_warp": "skin_build", "k_mark": "list_filter",
         "k_mask": "list_filter"}


def _val(r, hdr, units, key):
    v = float(r[hdr.index(key)].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return v * scale.get(units[hdr.index(key)], 1)


def traffic(path):
    r = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                       capture_output=True, text=True)
    if r.returncode != 0:   # a capture that failed to import: no entry
        return {}
    raw = r.stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    acc = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        base = name.split("<")[0].split("(")[0].replace("void ", "").split("::")[-1].strip()
        if base not in NAMES:
            continue
        b = (_val(r, hdr, units, "dram__bytes_read.sum")
             + _val(r, hdr, units, "dram__bytes_write.sum"))
        issue = _val(r, hdr, units, "smsp__issue_active.avg.pct_of_peak_sustained_active")
        inst = _val(r, hdr, units, "smsp__inst_executed.sum")
        acc.setdefault(NAMES[base], []).append((b, issue, inst))
    out = {}
    for k, v in acc.items():
        m = len(v)
        out[k] = {"dram_bytes": sum(x[0] for x in v) / m,
                  "issue_active_pct": sum(x[1] for x in v) / m,
                  "warp_inst": sum(x[2] for x in v) / m, "launches": m}
    return out


def main(out, specs):
    res = {}
    for s in specs:
        cfg, path = s.split("=", 1)
        res[cfg] = traffic(path)
        res[cfg]["_source"] = path.split("/")[-1]
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
