"""Generate golden vectors by running the UNMODIFIED reference (build container only).

    python oracle/gen_golden.py            # writes tests/golden/*.json

Imports ``beambatch`` from /root/reference/pkg/src and its test helpers
(``support.py``: random_beam_case, staged fixtures) from /root/reference/pkg/tests.
The fixtures are committed; nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import json
import math
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.dont_write_bytecode = True

import beambatch as bb  # noqa: E402
import support  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def f(x: float):
    """JSON-safe float (inf/-inf as strings; repr round-trips fp64 exactly)."""
    if x == math.inf:
        return "inf"
    if x == -math.inf:
        return "-inf"
    return x


def cand_json(c):
    return {"tokens": list(c.tokens), "score": f(c.score), "finalized": bool(c.finalized)}


def cfg_json(cfg):
    return {"k": cfg.k, "n": cfg.n, "epsilon": cfg.epsilon, "delta": f(cfg.delta),
            "max_candidates": cfg.max_candidates, "max_len": cfg.max_len,
            "policy": cfg.policy.value, "capacity": cfg.capacity,
            "flush_interval": cfg.flush_interval, "cost_c0": cfg.cost_c0, "cost_c1": cfg.cost_c1}


def expand_case(beam, rows, cfg, vocab):
    nxt, emitted = bb.expand_beam(beam, rows, cfg, vocab)
    return {
        "vocab": {"size": vocab.size, "sos": vocab.sos, "eos": vocab.eos},
        "config": cfg_json(cfg),
        "beam": {"l_t": beam.l_t, "emitted": beam.emitted,
                 "candidates": [cand_json(c) for c in beam.candidates]},
        "rows": [[f(x) for x in r] for r in rows],
        "want": {"next": [cand_json(c) for c in nxt.candidates], "l_t": nxt.l_t,
                 "emitted_total": nxt.emitted, "emitted": [cand_json(c) for c in emitted]},
    }


def gen_expand():
    cases = []
    # 1) the reference's own random case generator (grid-snapped ties), seed of C6
    rng = random.Random(20_260_810)
    for _ in range(600):
        cases.append(expand_case(*support.random_beam_case(rng)))
    # 2) wider cases: bigger k/M/V, many ties, both policies
    rng = random.Random(616)
    for _ in range(300):
        cases.append(expand_case(*support.random_beam_case(rng, max_k=8, max_vocab=24, len_cap=9)))
    # 3) the documented gap: row-value pre-truncation vs summed score
    vocab = bb.Vocabulary(size=8, sos=0, eos=7)
    beam = bb.Beam(0, (bb.Candidate((0, 1), -1e17, False),), 2, 0)
    row = [-5.0] * 8
    row[5], row[3] = -0.1, -0.2
    cfg = bb.DecodeConfig(k=2, n=1, max_candidates=1, max_len=10)
    cases.append(expand_case(beam, [row], cfg, vocab))
    # 4) masked (-inf) entries in rows
    vocab = bb.Vocabulary(size=6, sos=0, eos=5)
    beam = bb.Beam(0, (bb.Candidate((0, 2), -1.0, False), bb.Candidate((0, 3), -1.5, False)), 2, 0)
    rows = [[-math.inf, -0.5, -1.0, -math.inf, -2.0, -1.2],
            [-0.2, -math.inf, -math.inf, -0.7, -3.0, -0.9]]
    for pol in ("deferred", "immediate"):
        cfg = bb.DecodeConfig(k=3, n=1, delta=1.0, max_candidates=2, max_len=6, policy=pol)
        cases.append(expand_case(beam, rows, cfg, vocab))
    (OUT / "expand_cases.json").write_text(json.dumps(cases))
    return len(cases)


def run_fixture(name, runner, corpus, scorer_desc, scorer, cfg):
    events = []
    outputs, report = runner(corpus, scorer, cfg, trace=True, on_step=events.append)
    return {
        "name": name,
        "runner": runner.__name__,
        "scorer": scorer_desc,
        "corpus": [list(x) for x in corpus],
        "config": cfg_json(cfg),
        "outputs": [[{"tokens": list(c.tokens), "score": c.score} for c in per] for per in outputs],
        "report": {"timesteps": report.timesteps,
                   "candidate_expansions": report.candidate_expansions,
                   "simulated_cost": report.simulated_cost,
                   "trace": [list(r) for r in report.per_step_trace],
                   "summary": report.summarize()},
        "events": [{"timestep": e.timestep, "phase": e.phase, "refilled": list(e.refilled),
                    "selected": list(e.selected), "expansions": e.expansions,
                    "effective_len": e.effective_len, "finished": list(e.finished),
                    "live_after": list(e.live_after)} for e in events],
    }


def gen_runs():
    fixtures = []
    # acceptance criterion 1/2 workload (tests/test_acceptance.py:58-101), 240 inputs
    v50 = bb.Vocabulary(size=50, sos=0, eos=1)
    sc = bb.SeededHashScorer(v50, seed=31337, eos_bias=2.0)
    corpus = bb.generate_synthetic_corpus(4242, 240, 50, distribution="geometric",
                                          mean_len=8.0).inputs
    desc = {"kind": "seeded_hash", "vocab_size": 50, "sos": 0, "eos": 1, "seed": 31337,
            "eos_bias": 2.0}
    for eps in (1 / 12, 1 / 6, 1 / 4):
        cfg = bb.DecodeConfig(k=5, n=16, epsilon=eps, delta=1.5, max_candidates=3, max_len=48)
        fixtures.append(run_fixture(f"c1_varstream_eps{eps:.4f}", bb.run_varstream, corpus,
                                    desc, sc, cfg))
    cfg = bb.DecodeConfig(k=5, n=16, epsilon=1 / 6, delta=1.5, max_candidates=3, max_len=48)
    fixtures.append(run_fixture("c1_varbeam", bb.run_varbeam, corpus, desc, sc, cfg))
    fixtures.append(run_fixture("c1_varfifo", bb.run_varfifo, corpus, desc, sc, cfg))
    cfg = bb.DecodeConfig(k=5, n=16, epsilon=1 / 6, max_len=48)  # fixed / fixedstream
    fixtures.append(run_fixture("c1_fixedstream", bb.run_varstream, corpus, desc, sc, cfg))
    cfg = bb.DecodeConfig(k=5, n=16, epsilon=1 / 6, delta=1.5, max_candidates=3, max_len=48,
                          flush_interval=7)
    fixtures.append(run_fixture("c1_varstream_flush7", bb.run_varstream, corpus, desc, sc, cfg))
    cfg = bb.DecodeConfig(k=5, n=16, epsilon=1 / 6, delta=1.5, max_candidates=3, max_len=48,
                          capacity=23)
    fixtures.append(run_fixture("c1_varstream_cap23", bb.run_varstream, corpus, desc, sc, cfg))
    cfg = bb.DecodeConfig(k=4, n=8, epsilon=1 / 4, delta=2.0, max_candidates=2, max_len=20,
                          policy="immediate")
    fixtures.append(run_fixture("c1_varstream_immediate", bb.run_varstream, corpus[:80], desc,
                                sc, cfg))
    # staged event golden (tests/test_scheduler.py:131-185)
    staged = support.FnScorer  # noqa: F841 (documented: the staged scorer is restated in tests)
    (OUT / "runs.json").write_text(json.dumps(fixtures))
    return len(fixtures)


def gen_staged():
    from test_scheduler import STAGED_CORPUS, staged_scorer  # noqa: E402

    cfg = bb.DecodeConfig(k=2, n=3, epsilon=1 / 3, max_len=10)
    fx = run_fixture("staged", bb.run_varstream, STAGED_CORPUS,
                     {"kind": "staged"}, staged_scorer(), cfg)
    (OUT / "staged.json").write_text(json.dumps(fx))


def gen_metrics():
    rows = []
    for e, s in ((5071, 126), (14154, 248), (57550, 1469), (10, 4), (3, 2), (1, 3)):
        r = bb.MetricsReport(timesteps=s, candidate_expansions=e)
        rows.append({"expansions": e, "steps": s, "summary": r.summarize()})
    (OUT / "metrics.json").write_text(json.dumps(rows))


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    print("expand cases:", gen_expand())
    print("run fixtures:", gen_runs())
    gen_staged()
    gen_metrics()
    print("wrote", OUT)
