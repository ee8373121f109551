"""SASS instruction count (and a few mnemonics) per kernel of a built
library: python tools/sass_count.py LIB.so [name-substring ...]"""
import re
import subprocess
import sys

lib, keys = sys.argv[1], sys.argv[2:]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, counts = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = {"n": 0, "BSSY": 0, "MUFU": 0, "DFMA": 0, "CALL": 0}
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if cur and m:
        c = counts[cur]
        c["n"] += 1
        op = m.group(2).split(".")[0]
        if op in c:
            c[op] += 1
for f, c in counts.items():
    if all(k in f for k in keys):
        print(f"{c['n']:6d} BSSY={c['BSSY']:3d} MUFU={c['MUFU']:3d} DFMA={c['DFMA']:3d} "
              f"CALL={c['CALL']:3d}  {f[:110]}")
