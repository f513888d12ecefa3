"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
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
agg = collections.defaultdict(list)
unit = ""
for d in data:
    if d["Metric Name"] == "gpu__time_duration.sum":
        unit = d["Metric Unit"]
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("vs::<unnamed>::", "")
        agg[name].append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(unit, 1.0)
print(f"{'kernel':55s} {'launches':>8s} {'mean_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k[:55]:55s} {len(v):8d} {sum(v)/len(v)*scale:9.2f} {sum(v)/tot:6.3f}")
