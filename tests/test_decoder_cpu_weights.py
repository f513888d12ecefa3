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
