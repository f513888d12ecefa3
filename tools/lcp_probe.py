"""How much of the decoder's self-attention reads are shared within a beam: per
step, the longest common prefix (LCP) of each selected beam's active rows
(token histories), vs the positions every row reads.  WMT shape, transformer-big
scorer, a strided sample.  python tools/lcp_probe.py [N]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import bench
    from paper_2010_02164_b200 import DecodeConfig, Vocabulary
    from paper_2010_02164_b200 import _native as N
    from paper_2010_02164_b200.decoder import GraphedTransformerScorer
    from paper_2010_02164_b200.engine import SearchEngine

    n_in = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    w = bench.WORKLOADS["wmt19_k50"]
    corpus = bench._corpus(w)
    sample = corpus[::max(1, len(corpus) // n_in)][:n_in]
    vocab = Vocabulary(w["V"], w["sos"], w["eos"])
    cfg = DecodeConfig(k=w["k"], n=w["n"], epsilon=w["eps"], delta=w["delta"], max_candidates=w["M"],
                       max_len=w["max_len"])
    dec = GraphedTransformerScorer(vocab, tau=bench.DEC_TAU, eos_bias=bench.DEC_EOS_BIAS, max_src=256, seed=0)
    eng = SearchEngine(cfg, vocab)
    tot = {"read": 0, "shared": 0, "rows": 0}
    orig = eng._step

    def probe(scorer, st, **kw):
        R, nsel = int(st[N.ST_R]), int(st[N.ST_NSEL])
        if R:
            t, L = eng.t, eng.max_len
            off = t["sel_off"][: nsel + 1].cpu().tolist()
            phys = t["row_phys"][:R].long()
            ln = t["row_len"][:R]
            hist = t["hist"].view(-1, L)[phys]  # [R, L]
            for b in range(nsel):
                a, z = off[b], off[b + 1]
                h = hist[a:z]
                Lb = int(ln[a])
                eq = (h[:, :Lb] == h[:1, :Lb]).all(dim=0)
                lcp = int(torch.cumprod(eq.int(), 0).sum())
                tot["read"] += (z - a) * Lb
                tot["shared"] += (z - a - 1) * lcp if z - a > 1 else 0
                tot["rows"] += z - a
        return orig(scorer, st, **kw)

    eng._step = probe
    eng.run(sample, dec, admit_mode=N.VS_ADMIT_VARSTREAM, select_mode=N.VS_SELECT_MIN_LT, flush_enabled=False)
    print(f"rows {tot['rows']}, positions read {tot['read']}, of which a beam's common prefix beyond its "
          f"first row: {tot['shared']} ({tot['shared'] / max(1, tot['read']):.3f})")


if __name__ == "__main__":
    main()
