"""CLI and file formats (drop-in for bb/cli.py and bb/harness.py I/O)."""
import json

import pytest

from paper_2010_02164_b200 import cli
from paper_2010_02164_b200.harness import (Corpus, ResultsDocument, generate_synthetic_corpus, load_corpus,
                                           save_corpus)
from paper_2010_02164_b200.errors import DataError


def test_corpus_round_trip_and_errors(tmp_path):
    c = [(1, 2, 3), (4,), (5, 6)]
    p = tmp_path / "c.txt"
    save_corpus(c, p)
    got = load_corpus(p)
    assert isinstance(got, Corpus) and got.inputs == tuple(c) and len(got) == 3 and got[1] == (4,)
    (tmp_path / "bad.txt").write_text("1 2\nx 3\n")
    with pytest.raises(DataError, match="line 2"):
        load_corpus(tmp_path / "bad.txt")
    (tmp_path / "neg.txt").write_text("1 -2\n")
    with pytest.raises(DataError, match="negative"):
        load_corpus(tmp_path / "neg.txt")
    (tmp_path / "empty.txt").write_text("\n\n")
    with pytest.raises(DataError, match="empty"):
        load_corpus(tmp_path / "empty.txt")


def test_results_document_round_trip(tmp_path):
    doc = ResultsDocument("varstream", {"decode": {"k": 2}}, {"timesteps": 3},
                          [{"input_id": 0, "candidates": [{"tokens": [0, 5, 1], "score": -1.25}]}])
    doc.write(tmp_path / "r.json")
    back = ResultsDocument.read(tmp_path / "r.json")
    assert back.to_dict() == doc.to_dict()


def test_generator_matches_reference_golden_corpus():
    from goldens import load

    fx = load("runs.json")[0]  # generate_synthetic_corpus(4242, 240, 50, mean 8) by the reference
    got = generate_synthetic_corpus(4242, 240, 50, mean_len=8.0)
    assert [list(x) for x in got] == fx["corpus"]


@pytest.mark.parametrize("argv,code", [
    (["--engine", "varstream"], 1),                                      # k/n missing
    (["--engine", "bogus", "--k", "2", "--n", "2"], 1),                 # bad flag value
    (["--engine", "varstream", "--k", "2", "--n", "2"], 1),             # model missing
    (["--engine", "varstream", "--k", "2", "--n", "2", "--delta", "x"], 1),
])
def test_cli_config_errors_exit_1(argv, code, capsys):
    assert cli.main(argv) == code


def test_cli_missing_model_file_exits_2(tmp_path):
    assert cli.main(["--engine", "varstream", "--k", "2", "--n", "2", "--model",
                     str(tmp_path / "nope.json"), "--corpus", str(tmp_path / "c.txt")]) == 2


def test_cli_unknown_model_kind_exits_2(tmp_path):
    m = tmp_path / "m.json"
    m.write_text(json.dumps({"kind": "mystery", "vocab_size": 10, "sos": 0, "eos": 1}))
    assert cli.main(["--engine", "varstream", "--k", "2", "--n", "2", "--model", str(m),
                     "--corpus", str(tmp_path / "c.txt")]) == 2


@pytest.mark.gpu
def test_cli_device_run_writes_results_and_trace(tmp_path):
    m = tmp_path / "m.json"
    m.write_text(json.dumps({"kind": "device_hash", "vocab_size": 1000, "sos": 0, "eos": 2, "seed": 3,
                             "eos_bias": 4.0}))
    out = tmp_path / "r.json"
    cfgf = tmp_path / "cfg.json"
    cfgf.write_text(json.dumps({"engine": "varstream", "corpus": {"synthetic": {"n_inputs": 40, "mean_len": 6}},
                                "decode": {"k": 5, "n": 8, "delta": "1.5", "max_candidates": 3, "max_len": 30}}))
    assert cli.main(["--config", str(cfgf), "--model", str(m), "--out", str(out), "--trace"]) == 0
    doc = ResultsDocument.read(out)
    assert len(doc.records) == 40 and all(1 <= len(r["candidates"]) <= 5 for r in doc.records)
    assert (tmp_path / "r.json.trace.csv").read_text().startswith("timestep,expansions")
    # against the reference algorithm (oracle, pinned to bb/*) computing its own fp64
    # log-softmax rows of the same logits, in the reference's experiment order
    # (synthesise, bucket, decode, restore input order: bb/harness.py:280-331)
    import math

    from oracle import varstream_oracle as O
    from oracle.scorers import HashLogitsCPU

    corpus = O.generate_synthetic_corpus(0, 40, 1000, mean_len=6.0)
    bucketed, perm = O.bucket_by_length(corpus)
    sc = HashLogitsCPU(1000, 0, 2, 3, scale=0.5, power=0, eos_bias=4.0, dtype="bf16")
    cfg = O.OConfig(k=5, n=8, delta=1.5, max_candidates=3, max_len=30)
    want, wrep = O.run_varstream(bucketed, sc, cfg)
    same = 0
    for pos, orig in enumerate(perm):
        got = [(tuple(c["tokens"]), c["score"]) for c in doc.records[orig]["candidates"]]
        ref = [(c.tokens, c.score) for c in want[pos]]
        same += len(got) == len(ref) and all(
            a[0] == b[0] and math.isclose(a[1], b[1], rel_tol=1e-5) for a, b in zip(got, ref))
    assert same >= 0.995 * 40, same
    assert doc.metrics["candidate_expansions"] == wrep.candidate_expansions


def test_experiment_config_validation_matches_reference():
    """bb/harness.py:140-168: engine name, exactly one corpus source, trace
    needs an output path, fixed engines need pruning off."""
    import math

    from paper_2010_02164_b200.core import DecodeConfig
    from paper_2010_02164_b200.errors import ConfigError
    from paper_2010_02164_b200.harness import ExperimentConfig, SyntheticCorpusSpec

    m = {"kind": "device_hash", "vocab_size": 50, "sos": 0, "eos": 1}
    dec = DecodeConfig(k=3, n=4)
    syn = SyntheticCorpusSpec.from_dict({"n_inputs": 5})
    ExperimentConfig("varstream", m, dec, synthetic=syn)
    for bad in (dict(engine="nope", synthetic=syn), dict(engine="varstream"),
                dict(engine="varstream", synthetic=syn, corpus_path="x"),
                dict(engine="varstream", synthetic=syn, trace=True),
                dict(engine="fixed", synthetic=syn, decode=DecodeConfig(k=3, n=4, delta=1.5))):
        eng, d = bad.pop("engine"), bad.pop("decode", dec)
        with pytest.raises(ConfigError):
            ExperimentConfig(eng, m, d, **bad)
    ExperimentConfig("fixed", m, DecodeConfig(k=3, n=4, delta=math.inf, max_candidates=3), synthetic=syn)
    with pytest.raises(ConfigError):
        SyntheticCorpusSpec.from_dict({"mean_len": 3})


def test_cli_rejects_out_of_scope_model_kinds(tmp_path):
    """The reference's seeded-hash / n-gram scorers are out of scope and the
    CLI never imports the reference package: exit code 2 with a message."""
    mp = tmp_path / "m.json"
    mp.write_text(json.dumps({"kind": "seeded_hash", "vocab_size": 50, "sos": 0, "eos": 1, "seed": 3}))
    cp = tmp_path / "c.txt"
    cp.write_text("3 4 5\n")
    assert cli.main(["--engine", "varstream", "--k", "2", "--n", "2", "--model", str(mp),
                     "--corpus", str(cp)]) == 2


def test_corpus_checks_match_reference_messages():
    """harness.check_corpus (run by the engine before a decode) raises the
    reference's DataErrors (bb/model.py:90-102)."""
    import numpy as np

    from paper_2010_02164_b200.harness import check_corpus

    check_corpus(np.array([1, 2, 3]), np.array([0, 2, 3]), 10)
    with pytest.raises(DataError, match="inputs must be nonempty"):
        check_corpus(np.array([1, 2]), np.array([0, 2, 2]), 10)
    with pytest.raises(DataError, match=r"token 12 at position 1 is outside the vocabulary \(size 10\)"):
        check_corpus(np.array([1, 2, 3, 12]), np.array([0, 2, 4]), 10)
    with pytest.raises(DataError, match="token -1 at position 0"):
        check_corpus(np.array([-1]), np.array([0, 1]), 10)
