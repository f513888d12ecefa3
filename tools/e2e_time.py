"""e2e breakdown of run_varstream(streams=S) from host lists: total, load_corpus, Harvest
materialisation and the device-side decode alone.  python tools/e2e_time.py [S]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import bench
    import paper_2010_02164_b200 as P
    from paper_2010_02164_b200.scorers import DeviceHashScorer

    S = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    w = bench.WORKLOADS["wmt19_k50"]
    corpus = bench._corpus(w)
    vocab = P.Vocabulary(w["V"], w["sos"], w["eos"])
    cfg = P.DecodeConfig(k=w["k"], n=w["n"], epsilon=w["eps"], delta=w["delta"], max_candidates=w["M"],
                         max_len=w["max_len"])
    sc = DeviceHashScorer(vocab, w["scorer_seed"], scale=w["scale"], power=w["power"], eos_bias=w["eos_bias"],
                          dtype=w["dtype"])
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if i == 3:
            pr = cProfile.Profile()
            pr.enable()
        outs, rep = P.run_varstream(corpus, sc, cfg, streams=S)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i == 3:
            pr.disable()
        print(f"e2e {dt * 1e3:.1f} ms ({len(corpus) / dt:.0f} seq/s)", flush=True)
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
