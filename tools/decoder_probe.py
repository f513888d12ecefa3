"""WMT'19-shape decoder scorer probe: calibration (tau, eos_bias) and timing.

    python tools/decoder_probe.py [N] [tau] [eos_bias] [--eager]
"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_02164_b200 import DecodeConfig, Vocabulary  # noqa: E402
from paper_2010_02164_b200 import _native as N  # noqa: E402
from paper_2010_02164_b200.decoder import GraphedTransformerScorer  # noqa: E402
from paper_2010_02164_b200.engine import SearchEngine  # noqa: E402
from paper_2010_02164_b200.harness import bucket_by_length, generate_synthetic_corpus  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
Nin = int(args[0]) if args else 500
tau = float(args[1]) if len(args) > 1 else 4.0
eb = float(args[2]) if len(args) > 2 else 12.0
V = 42024
vocab = Vocabulary(V, 0, 2)
cfg = DecodeConfig(k=50, n=128, epsilon=1 / 6, delta=1.5, max_candidates=5, max_len=256)
corpus = bucket_by_length(generate_synthetic_corpus(99, Nin, V, mean_len=25.0, clip=200))[0]
t0 = time.perf_counter()
dec = GraphedTransformerScorer(vocab, tau=tau, eos_bias=eb, use_graphs="--eager" not in sys.argv)
eng = SearchEngine(cfg, vocab)
print(f"init {time.perf_counter() - t0:.1f}s", flush=True)
import cProfile  # noqa: E402
import pstats  # noqa: E402

for rep_i in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prof = cProfile.Profile() if (rep_i == 1 and "--prof" in sys.argv) else None
    if prof:
        prof.enable()
    out, rep = eng.run(corpus, dec, admit_mode=N.VS_ADMIT_VARSTREAM, select_mode=N.VS_SELECT_MIN_LT,
                       flush_enabled=False)
    if prof:
        prof.disable()
        pstats.Stats(prof).sort_stats("tottime").print_stats(22)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    lens = [len(c.tokens) for per in out for c in per[:1]]
    print(f"run{rep_i} tau={tau} eos_bias={eb}: {len(corpus) / dt:.1f} seq/s, {dt:.2f}s, "
          f"steps {rep.timesteps}, exp/step {rep.expansions_per_step:.1f}, ms/step {1e3 * dt / rep.timesteps:.3f}, "
          f"mean out len {sum(lens) / len(lens):.1f}, max {max(lens)}, graphs {len(dec.graphs)}", flush=True)
