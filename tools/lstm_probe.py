"""C3 LSTM leg probe: one batch, host cProfile of the synchronous driver and
device time per step.  python tools/lstm_probe.py [N]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import bench
    from paper_2010_02164_b200 import DecodeConfig, Vocabulary
    from paper_2010_02164_b200 import _native as N
    from paper_2010_02164_b200.decoder import LSTMScorer
    from paper_2010_02164_b200.engine import SearchEngine

    w = bench.WORKLOADS["parse_c3"]
    n_in = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
    corpus = bench._corpus(w)[:n_in]
    vocab = Vocabulary(w["V"], w["sos"], w["eos"])
    cfg = DecodeConfig(k=w["k"], n=w["n"], epsilon=w["eps"], delta=w["delta"], max_candidates=w["M"],
                       max_len=w["max_len"])
    dec = LSTMScorer(vocab, **bench.LSTM_KW)
    eng = SearchEngine(cfg, vocab)
    run = lambda: eng.run(corpus, dec, admit_mode=N.VS_ADMIT_VARSTREAM,  # noqa: E731
                          select_mode=N.VS_SELECT_MIN_LT, flush_enabled=False)
    run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pr = cProfile.Profile()
    pr.enable()
    _, rep = run()
    torch.cuda.synchronize()
    pr.disable()
    dt = time.perf_counter() - t0
    print(f"{n_in} inputs: {dt * 1e3:.1f} ms, {rep.timesteps} steps, {1e6 * dt / rep.timesteps:.1f} us/step")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
