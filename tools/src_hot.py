"""Aggregate an ncu cuda,sass source CSV by CUDA source line."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = "?"
hdr = None
agg = defaultdict(lambda: [0.0, 0.0, ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    if r[0].isdigit() and r[2] == "-":          # a cuda source line summary row
        ie = float(r[7] or 0)
        ws = float(r[4] or 0)
        key = (cur_file, int(r[0]))
        agg[key][0] += ie
        agg[key][1] += ws
        agg[key][2] = r[1][:90]
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instr {tot_i:.3e}  stall samples {tot_s:.0f}")
for (f, ln), (ie, ws, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f:16s}{ln:5d} instr {ie/tot_i:6.1%} stall {ws/tot_s:6.1%}  {src}")
if len(sys.argv) > 3 and sys.argv[3] == "stall":
    print("--- by stall samples")
    for (f, ln), (ie, ws, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{f:16s}{ln:5d} instr {ie/tot_i:6.1%} stall {ws/tot_s:6.1%}  {src}")
