"""One single-batch VarStream decode of a bench workload, for ncu launch
lists: warm-up decode (captures the step graphs), then one decode inside
cudaProfilerStart/Stop (run ncu with --profile-from-start off).

    ncu --profile-from-start off --metrics gpu__time_duration.sum \
        --clock-control none --cache-control none --csv --log-file X.csv \
        python tools/step_profile.py [--workload wmt19_k50] [--n-inputs 1000]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2010_02164_b200 import DecodeConfig, Vocabulary  # noqa: E402
from paper_2010_02164_b200 import _native as N  # noqa: E402
from paper_2010_02164_b200.engine import SearchEngine  # noqa: E402
from paper_2010_02164_b200.harness import flatten  # noqa: E402
from paper_2010_02164_b200.scorers import DeviceHashScorer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="wmt19_k50")
ap.add_argument("--n-inputs", type=int, default=1000)
a = ap.parse_args()
w = dict(bench.WORKLOADS[a.workload], N=a.n_inputs)
corpus = bench._corpus(w)
vocab = Vocabulary(w["V"], w["sos"], w["eos"])
cfg = DecodeConfig(k=w["k"], n=w["n"], epsilon=w["eps"], delta=w["delta"], max_candidates=w["M"],
                   max_len=w["max_len"])
sc = DeviceHashScorer(vocab, w["scorer_seed"], scale=w["scale"], power=w["power"], eos_bias=w["eos_bias"],
                      dtype=w["dtype"])
eng = SearchEngine(cfg, vocab)
tok, off = flatten(corpus)
d_tok, d_off = torch.from_numpy(tok).cuda(), torch.from_numpy(off).cuda()
for prof in (False, False, True):
    if prof:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, rep = eng.run_async(None, sc, admit_mode=N.VS_ADMIT_VARSTREAM, select_mode=N.VS_SELECT_MIN_LT,
                           src_tok=d_tok, src_off=d_off, materialize=False)
    e1.record()
    torch.cuda.synchronize()
    if prof:
        torch.cuda.cudart().cudaProfilerStop()
    print(f"decode {len(corpus)} inputs: {rep.timesteps} steps, {e0.elapsed_time(e1):.2f} ms, "
          f"{1e3 * e0.elapsed_time(e1) / max(1, rep.timesteps):.1f} us/step", flush=True)
