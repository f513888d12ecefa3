"""Summarise gpurun_out/ ncu captures into profiles/<round>/ (tracked).

    python tools/collect_profiles.py round1
"""
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))
from ncu_summary import KEYS, load  # noqa: E402

rnd = sys.argv[1]
src = ROOT / "gpurun_out"
dst = ROOT / "profiles" / rnd
dst.mkdir(parents=True, exist_ok=True)
summary = {}
for rep in ("k1_fullwidth", "k1_decode", "step_kernels", "k1t_fw", "k1t_573", "k5_1300", "dec_attention"):
    p = src / f"{rep}.ncu-rep"
    if not p.exists():
        continue
    rows = load(str(p))
    summary[rep] = [{k: d[k][0] for k in KEYS + ["Kernel Name"]} for d in rows]
    with open(dst / f"{rep}_ncu.txt", "w") as f:
        for d in rows:
            f.write(d["Kernel Name"][0][:120] + "\n")
            for k in KEYS:
                f.write(f"  {k:62s} {d[k][0]} {d[k][1] or ''}\n")
    # per-instruction stall summary (top-level)
    out = subprocess.run(["ncu", "-i", str(p), "--page", "details", "--csv"], capture_output=True, text=True).stdout
    (dst / f"{rep}_details.csv").write_text(out)
    if rep.startswith("k1t"):  # SASS-region breakdown of the split-row kernel
        units = {"k1t_fw": 134400, "k1t_573": 12033}[rep]
        out = subprocess.run([sys.executable, str(ROOT / "tools" / "sass_hot.py"), str(p), str(units), "30"],
                             capture_output=True, text=True).stdout
        (dst / f"{rep}_sass_regions.txt").write_text(out)
for name in ("launches_decode", "dec_launches"):
    if not (src / f"{name}.csv").exists():
        continue
    shutil.copy(src / f"{name}.csv", dst / f"{name}.csv")
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "launch_summary.py"), str(src / f"{name}.csv")],
                         capture_output=True, text=True).stdout
    (dst / f"{name}_summary.txt").write_text(out)
if False:
    shutil.copy(src / "launches_decode.csv", dst / "launches_decode.csv")
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "launch_summary.py"), str(src / "launches_decode.csv")],
                         capture_output=True, text=True).stdout
    (dst / "launches_decode_summary.txt").write_text(out)
for name in ("bench.json", "bench_ref.json", "pytest_gpu.log", "smoke.log"):
    if (src / name).exists():
        shutil.copy(src / name, dst / name)
(dst / "summary.json").write_text(json.dumps(summary, indent=1))
# K1 DRAM traffic per launch (full-width capture: R=6400 x 42024 bf16)
fw = summary.get("k1_fullwidth")
if fw:
    rd = float(fw[0]["dram__bytes_read.sum"]) * 1e6
    wr = float(fw[0]["dram__bytes_write.sum"]) * 1e6
    (ROOT / "profiles" / "k1_traffic.json").write_text(json.dumps({
        "round": rnd, "kernel": fw[0]["Kernel Name"][:80], "R": 6400, "V": 42024, "dtype": "bf16",
        "algorithmic_bytes_per_launch": 6400 * 42024 * 2,
        "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
        "source": f"profiles/{rnd}/k1_fullwidth_ncu.txt (ncu --set full, L2 flushed before launch)"}, indent=1))
print("wrote", dst)
