"""Per-source-line instruction / stall shares of one kernel from an ncu
report (--page source --print-source sass,cuda)."""
import csv
import subprocess
import sys


def main(path, kernel, top=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "-k", f"regex:{kernel}",
                          "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    cur, hdr, agg = None, None, {}
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0].isdigit():
            continue
        try:
            ie = float(r[hdr.index("Instructions Executed")] or 0)
            st = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        a = agg.setdefault((cur, int(r[0])), [0.0, 0.0, r[1][:90]])
        a[0] += ie
        a[1] += st
    tot = sum(v[0] for v in agg.values()) or 1
    tst = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {tot:.4g}, stall samples {tst:.4g}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0]}:{k[1]:5d} inst {100 * v[0] / tot:5.1f}% stall {100 * v[1] / tst:5.1f}%  {v[2]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
