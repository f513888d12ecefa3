"""Per-region instruction / stall breakdown of one kernel in an ncu report.

    python tools/sass_hot.py report.ncu-rep [units]   (units: divide counts by this)
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = [dict(zip(h, x)) for x in r[2:] if len(x) == len(h)]
tot = sum(int(d["Instructions Executed"]) for d in rows)
smp = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in rows)
print(f"total warp-inst {tot}  ({tot / units:.1f} per unit)")
# basic blocks: split at instructions whose count differs from the previous one
blocks, cur = [], None
for i, d in enumerate(rows):
    n = int(d["Instructions Executed"])
    if cur is None or n != cur["n"]:
        cur = {"start": i, "n": n, "len": 0, "smp": 0, "first": d["Source"].strip()[:70]}
        blocks.append(cur)
    cur["len"] += 1
    cur["smp"] += int(d["Warp Stall Sampling (All Samples)"] or 0)
blocks.sort(key=lambda b: -b["n"] * b["len"])
print(f"{'start':>6} {'len':>4} {'exec/unit':>9} {'inst%':>6} {'stall%':>6}  first")
for b in blocks[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{b['start']:6d} {b['len']:4d} {b['n'] / units:9.3f} {100 * b['n'] * b['len'] / tot:6.2f} "
          f"{100 * b['smp'] / max(1, smp):6.2f}  {b['first']}")
