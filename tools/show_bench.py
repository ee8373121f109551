"""Print value and per-kernel sub-step times of bench JSON lines."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f.split("/")[-1], "%.3e" % d["value"],
              {k: round(v, 4) for k, v in r["kernel_ms_per_substep"].items()})
    except Exception as e:   # noqa: BLE001
        print(f, "ERR", e)
