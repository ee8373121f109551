"""Print value, e2e and per-launch kernel times of bench JSON lines."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        if "unavailable" in d or d.get("impl") == "reference":
            print(f.split("/")[-1], "reference", "%.4g" % d["value"], d.get("steps"),
                  d.get("nsub_per_step"), d["cpu_baseline"].get("cores"))
            continue
        r = d["roofline"]
        e = d.get("e2e") or {}
        print(f.split("/")[-1], "value %.4g" % d["value"], "e2e %.4g" % e.get("value", 0),
              "ms/step %.2f" % d["ms_per_step"],
              {k: round(v, 3) for k, v in r.get("kernel_ms_per_launch", {}).items()},
              "frac %.3f" % r["frac"], "cpu", (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e:   # noqa: BLE001
        print(f, "ERR", e)
