"""Host-side profile of the e2e path (run_varstream with host lists; argv[1] concurrent batches, default 6)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2010_02164_b200 as P  # noqa: E402
from paper_2010_02164_b200.scorers import DeviceHashScorer  # noqa: E402

STREAMS = int(sys.argv[1]) if len(sys.argv) > 1 else 6
w = bench.WORKLOADS["wmt19_k50"]
corpus = bench._corpus(w)
vocab = P.Vocabulary(w["V"], w["sos"], w["eos"])
cfg = P.DecodeConfig(k=w["k"], n=w["n"], epsilon=w["eps"], delta=w["delta"], max_candidates=w["M"],
                     max_len=w["max_len"])
sc = DeviceHashScorer(vocab, w["scorer_seed"], scale=w["scale"], power=w["power"], eos_bias=w["eos_bias"],
                      dtype=w["dtype"])
for _ in range(2):
    P.run_varstream(corpus, sc, cfg, streams=STREAMS)
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
outs, rep = P.run_varstream(corpus, sc, cfg, streams=STREAMS)
torch.cuda.synchronize()
pr.disable()
print("e2e s", time.perf_counter() - t0, "seq/s", len(corpus) / (time.perf_counter() - t0))
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
