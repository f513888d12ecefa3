"""e2e timing of run_varstream(streams=4) from host lists, and of its results() phase."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2010_02164_b200 as P  # noqa: E402
from paper_2010_02164_b200 import engine as E  # noqa: E402
from paper_2010_02164_b200.scorers import DeviceHashScorer  # noqa: E402

w = bench.WORKLOADS["wmt19_k50"]
corpus = bench._corpus(w)
vocab = P.Vocabulary(w["V"], w["sos"], w["eos"])
cfg = P.DecodeConfig(k=w["k"], n=w["n"], epsilon=w["eps"], delta=w["delta"], max_candidates=w["M"],
                     max_len=w["max_len"])
sc = DeviceHashScorer(vocab, w["scorer_seed"], scale=w["scale"], power=w["power"], eos_bias=w["eos_bias"],
                      dtype=w["dtype"])
res_t = []
orig = E.SearchEngine.results


def timed(self):
    t0 = time.perf_counter()
    r = orig(self)
    res_t.append(time.perf_counter() - t0)
    return r


E.SearchEngine.results = timed
lc_t = []
orig_lc = E.SearchEngine.load_corpus


def timed_lc(self, *a, **k):
    t0 = time.perf_counter()
    r = orig_lc(self, *a, **k)
    lc_t.append(time.perf_counter() - t0)
    return r


E.SearchEngine.load_corpus = timed_lc
for i in range(5):
    res_t.clear()
    lc_t.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    outs, rep = P.run_varstream(corpus, sc, cfg, streams=4)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"e2e {dt*1e3:.1f} ms ({len(corpus)/dt:.0f} seq/s)  results {sum(res_t)*1e3:.1f} ms  load_corpus {sum(lc_t)*1e3:.1f} ms")
