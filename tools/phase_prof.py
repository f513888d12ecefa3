"""Phase timing of the fused beam-step kernel (profiling build, -DVS_PHASE_PROF).

    python tools/phase_prof.py --build      # here: builds _lib/libvarstream_prof.so
    python tools/phase_prof.py [--n-inputs 10000]   # on the GPU box

Prints the mean time (µs since CTA 0's start) at which CTA 0 reaches each
beam phase and the last CTA reaches each scheduler phase."""
import argparse
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
PROF_LIB = ROOT / "paper_2010_02164_b200" / "_lib" / "libvarstream_prof.so"
NAMES = {1: "beam: candidates loaded", 2: "beam: pool built", 3: "beam: ranked", 4: "beam: children",
         5: "beam: emission plan", 6: "beam: hist+emit done", 7: "beam: CTA0 done",
         8: "all CTAs arrived", 9: "sched: loads", 12: "sched: counters", 13: "sched: removal",
         10: "sched: refill", 11: "sched: selection", 15: "sched: row list done"}

ap = argparse.ArgumentParser()
ap.add_argument("--build", action="store_true")
ap.add_argument("--n-inputs", type=int, default=10000)
a = ap.parse_args()
if a.build:
    import __graft_entry__ as g
    srcs = sorted(str(p) for p in g.CSRC.glob("*.cu"))
    subprocess.run([g.NVCC, *g.NVCC_FLAGS, "-DVS_PHASE_PROF", "-o", str(PROF_LIB), *srcs], check=True,
                   capture_output=True)
    print("built", PROF_LIB)
    sys.exit(0)
os.environ["VARSTREAM_LIB"] = str(PROF_LIB)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2010_02164_b200 import DecodeConfig, Vocabulary  # noqa: E402
from paper_2010_02164_b200 import _native as N  # noqa: E402
from paper_2010_02164_b200.engine import SearchEngine  # noqa: E402
from paper_2010_02164_b200.harness import flatten  # noqa: E402
from paper_2010_02164_b200.scorers import DeviceHashScorer  # noqa: E402

w = dict(bench.WORKLOADS["wmt19_k50"], N=a.n_inputs)
corpus = bench._corpus(w)
vocab = Vocabulary(w["V"], w["sos"], w["eos"])
cfg = DecodeConfig(k=w["k"], n=w["n"], epsilon=w["eps"], delta=w["delta"], max_candidates=w["M"],
                   max_len=w["max_len"])
sc = DeviceHashScorer(vocab, w["scorer_seed"], scale=w["scale"], power=w["power"], eos_bias=w["eos_bias"],
                      dtype=w["dtype"])
eng = SearchEngine(cfg, vocab)
lib = eng.lib
tok, off = flatten(corpus)
d_tok, d_off = torch.from_numpy(tok).cuda(), torch.from_numpy(off).cuda()
acc = (C.c_ulonglong * 32)()
for it in range(2):
    lib.vs_debug_phase_times(acc)
    _, rep = eng.run_async(None, sc, admit_mode=N.VS_ADMIT_VARSTREAM, select_mode=N.VS_SELECT_MIN_LT,
                           src_tok=d_tok, src_off=d_off, materialize=False)
    torch.cuda.synchronize()
lib.vs_debug_phase_times(acc)
n = max(1, acc[31])
print(f"{n} fused launches ({rep.timesteps} steps); CTA 0 (beam 0, then the scheduler), mean SM cycles "
      "since it started:")
for i, name in NAMES.items():
    print(f"  {i:2d} {name:28s} {acc[i] / n:9.0f}")
print("slowest beam CTA per launch (max over CTAs of cycles since that CTA started), mean over launches:")
for i in range(1, 8):
    print(f"  {i:2d} {NAMES[i]:28s} {acc[16 + i] / n:9.0f}")
