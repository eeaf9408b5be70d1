"""Per CUDA source line: shared-memory wavefronts (actual vs ideal) from an ncu source CSV."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur = "?"
hdr = None
agg = defaultdict(lambda: [0.0, 0.0, ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ci = {k: i for i, k in enumerate(hdr)}
        continue
    if hdr is None or not r[0].isdigit() or r[2] != "-":
        continue
    try:
        act = float(r[ci["L1 Wavefronts Shared"]] or 0)
        ideal = float(r[ci["L1 Wavefronts Shared Ideal"]] or 0)
    except (KeyError, ValueError):
        continue
    k = (cur, int(r[0]))
    agg[k][0] += act
    agg[k][1] += ideal
    agg[k][2] = r[1][:80]
tot = sum(v[0] for v in agg.values()) or 1
print(f"total shared wavefronts {tot:.3e}, ideal {sum(v[1] for v in agg.values()):.3e}")
for (f, ln), (a, i, src) in sorted(agg.items(), key=lambda kv: -(kv[1][0] - kv[1][1]))[:top]:
    print(f"{f:14s}{ln:5d} wavefronts {a:10.3e} ideal {i:10.3e} excess {a - i:10.3e}  {src}")
