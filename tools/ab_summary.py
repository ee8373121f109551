"""Summarise A/B bench lines: per config and variant, PU/s of each rep and
per-launch kernel ms (roofline.kernel_ms_per_launch)."""
import collections
import json
import re
import sys

rows = collections.defaultdict(list)
for p in sys.argv[1:]:
    m = re.search(r"ab_([^_]+)_(.+)_(\d+)\.json$", p)
    if not m:
        continue
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception:
        print(p, "no line")
        continue
    rows[(m.group(1), m.group(2))].append(d)
for (c, v), ds in sorted(rows.items()):
    vals = " ".join("%.4g" % d["value"] for d in ds)
    k = ds[-1]["roofline"].get("kernel_ms_per_launch", {})
    ks = " ".join("%s=%.3f" % (a[:8], b) for a, b in sorted(k.items()))
    print(f"{c:6s} {v:12s} {vals}   {ks}")
