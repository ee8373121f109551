"""Key metrics per kernel from an ncu report (raw page)."""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]
STALLS = "smsp__average_warps_issue_stalled_"


def main(path, kernel_filter=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        if kernel_filter not in name:
            continue
        print("----", name[:90])
        for w in WANT:
            if w in hdr:
                print(f"  {w:70s} {r[hdr.index(w)]} {units[hdr.index(w)]}")
        st = []
        for k, h in enumerate(hdr):
            if h.startswith(STALLS) and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[k]), h[len(STALLS):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        if not st:
            for k, h in enumerate(hdr):
                if "warp_issue_stalled" in h and h.endswith("_per_warp_active.pct"):
                    try:
                        st.append((float(r[k]), h))
                    except ValueError:
                        pass
        st.sort(reverse=True)
        print("  stalls:", ", ".join(f"{n}={v:.2f}" for v, n in st[:8]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
