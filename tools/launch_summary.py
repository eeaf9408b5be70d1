"""Summarise an ncu --metrics gpu__time_duration.sum launch-list CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0][:80] + ("  grid " + d["Grid Size"] if d.get("Grid Size") else "")
    agg.setdefault(k, []).append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
print(f"{'launches':>8} {'mean_us':>10} {'total_us':>10} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):8d} {sum(v)/len(v)/1e3:10.1f} {sum(v)/1e3:10.1f} {sum(v)/tot:6.1%}  {k}")
