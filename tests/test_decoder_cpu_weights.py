"""CPU check: the oracle's CPU transformer scorer (bench decoder baseline) is
built from exactly the product decoder's random-init weights, and its rows
are normalised log-probs (bb/model.py:216-217)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def test_torch_decoder_cpu_matches_product_weights_and_normalises():
    from oracle.scorers import TorchDecoderCPU
    from paper_2010_02164_b200.core import Vocabulary
    from paper_2010_02164_b200.decoder import TransformerScorer

    V = 97
    prod = TransformerScorer(Vocabulary(V, 0, 2), d=64, heads=1, layers=2, enc_layers=1, ffn=128, seed=5,
                             tau=3.0, dtype=torch.bfloat16, device="cpu")
    cpu = TorchDecoderCPU(V, 0, 2, d=64, heads=1, layers=2, enc_layers=1, ffn=128, seed=5, tau=3.0,
                          eos_bias=4.0)
    assert torch.equal(prod.emb.float(), cpu.emb)
    assert torch.equal(prod.dec[1]["f2"].float(), cpu.dec[1]["f2"])
    assert torch.equal((prod.out.float() * 3.0).to(torch.bfloat16).float(), cpu.out_s)

    class C:
        tokens = (0, 5, 7)

    enc = cpu.encode([3, 4, 5, 6], input_id=1)
    row = cpu.score_next(enc, C)
    assert row.shape == (V,)
    assert abs(math.log(np.exp(row).sum())) < 1e-9


def test_torch_decoder_cpu_f32_is_the_product_model():
    """weights='f32': the CPU reference scorer computes the same function as
    the product TransformerScorer in fp32 (its cache-free forward), so the
    decoder agreement test compares one model under two implementations."""
    from oracle.scorers import TorchDecoderCPU
    from paper_2010_02164_b200.core import Vocabulary
    from paper_2010_02164_b200.decoder import TransformerScorer

    V = 101
    kw = dict(d=32, heads=4, layers=2, enc_layers=1, ffn=64, seed=3, tau=3.0)
    prod = TransformerScorer(Vocabulary(V, 0, 2), eos_bias=3.0, dtype=torch.float32, device="cpu", **kw)
    cpu = TorchDecoderCPU(V, 0, 2, eos_bias=3.0, weights="f32", **kw)

    class C:
        tokens = (0, 5, 7, 9)

    src = [3, 4, 5, 6, 8]
    row = cpu.score_next(cpu.encode(src, input_id=0), C)
    lg = prod.full_forward(src, C.tokens).double()
    want = (lg - torch.logsumexp(lg, 0)).numpy()
    assert np.max(np.abs(row - want)) < 1e-4


def test_torch_decoder_cpu_incremental_matches_full_recompute():
    """The CPU reference model's per-prefix K/V cache (used for the decoder
    agreement run) computes the same rows as whole-prefix recompute."""
    from oracle.scorers import TorchDecoderCPU

    kw = dict(d=32, heads=4, layers=2, enc_layers=1, ffn=64, seed=3, tau=3.0, eos_bias=3.0)
    full = TorchDecoderCPU(97, 0, 2, **kw)
    inc = TorchDecoderCPU(97, 0, 2, **kw)
    inc.incremental = True

    class C:
        def __init__(self, tokens, score=0.0, finalized=False, input_id=0):
            self.tokens = tokens

    src = [5, 6, 7, 8]
    e1, e2 = full.encode(src, 0), inc.encode(src, 0)
    for pre in [(0,), (0, 9), (0, 9, 4), (0, 9, 4, 11), (0, 12)]:
        a, b = full.score_next(e1, C(pre)), inc.score_next(e2, C(pre))
        assert np.max(np.abs(a - b)) < 1e-4


def test_torch_decoder_cpu_score_batch_matches_rows():
    from oracle.scorers import TorchDecoderCPU

    kw = dict(d=32, heads=4, layers=2, enc_layers=1, ffn=64, seed=3, tau=3.0, eos_bias=3.0)
    a = TorchDecoderCPU(97, 0, 2, **kw)
    b = TorchDecoderCPU(97, 0, 2, **kw)
    b.incremental = True

    class C:
        def __init__(self, tokens):
            self.tokens = tokens

    e1, e2 = a.encode([5, 6, 7], 0), b.encode([5, 6, 7], 0)
    b.score_batch(e2, [C((0,))])
    b.score_batch(e2, [C((0, 9)), C((0, 4))])
    got = b.score_batch(e2, [C((0, 9, 1)), C((0, 4, 7)), C((0, 9, 3))])
    for g, t in zip(got, [(0, 9, 1), (0, 4, 7), (0, 9, 3)]):
        assert np.max(np.abs(g - a.score_next(e1, C(t)))) < 1e-4
