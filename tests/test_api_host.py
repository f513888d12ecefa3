"""CPU checks of the host-side API pieces (paper_2010_02164_b200.api) against
the oracle restatement of bb/heuristics.py and bb/scheduler.py."""
import math
import random

import pytest

from oracle import varstream_oracle as O
from paper_2010_02164_b200 import api as A
from paper_2010_02164_b200.core import Beam, Candidate, DecodeConfig, Proposal, Vocabulary
from paper_2010_02164_b200.errors import ConfigError, InvariantViolation


def _pool(rng, n):
    pool = []
    for _ in range(n):
        tok = None if rng.random() < 0.15 else rng.randrange(20)
        pool.append(Proposal(round(-rng.random() * 4, rng.choice([1, 2, 6])), rng.randrange(6), tok))
    return pool


@pytest.mark.parametrize("seed", range(40))
def test_apply_heuristics_matches_oracle(seed):
    rng = random.Random(seed)
    pool = _pool(rng, rng.randrange(1, 40))
    k, M = rng.randrange(1, 9), rng.randrange(1, 5)
    delta = rng.choice([0.0, 0.5, 1.5, math.inf])
    got = A.apply_heuristics(pool, k=k, delta=delta, max_candidates=M)
    opool = [O.Proposal(p.score, p.parent, p.token) for p in pool]
    want = O.apply_heuristics(opool, k=k, delta=delta, max_candidates=M)
    assert [tuple(p) for p in got] == [tuple(p) for p in want]
    assert A.HeuristicConfig(delta, M).apply(pool, k) == got


def test_heuristic_config_and_empty_pool_errors():
    with pytest.raises(ConfigError):
        A.HeuristicConfig(-1.0, 2)
    with pytest.raises(ConfigError):
        A.HeuristicConfig(1.0, 0)
    with pytest.raises(InvariantViolation):
        A.apply_heuristics([], k=2, delta=1.0, max_candidates=1)


class _Enc:
    def __init__(self, i):
        self.input_id = i


class _Sc:
    vocab = Vocabulary(10, 0, 1)

    def encode(self, toks, input_id=0):
        return _Enc(input_id)


def test_refill_and_selection_match_oracle():
    cfg = DecodeConfig(k=3, n=5, capacity=7)
    st = A.BatchState()
    ost = O.BatchState()

    class OSc:
        sos = 0

        def encode(self, toks, input_id=0):
            return _Enc(input_id)

    corpus = [(1, 2)] * 9
    assert A.refill(st, corpus, cfg, _Sc()) == O.refill(ost, corpus, O.as_oconfig(cfg), OSc()) == [0, 1, 2, 3, 4]
    widths = [(2, 3), (3, 1), (2, 2), (1, 4), (3, 2)]  # (l_t, active width)
    for s, os_, (lt, w) in zip(st.beams, ost.beams, widths):
        cands = tuple(Candidate((0,) * lt, -0.1 * j, False, s.input_id) for j in range(w))
        s.beam = Beam(s.input_id, cands, lt, 0)
        os_.beam = O.Beam(s.input_id, tuple(O.Candidate(c.tokens, c.score, False, s.input_id) for c in cands), lt, 0)
    for mine, ref in ((A.select_min_lt, O.select_min_lt), (A.select_fifo_max_lt, O.select_fifo_max_lt)):
        sel = mine(st, cfg.capacity)
        chosen, total, eff = ref(ost, cfg.capacity)
        assert [s.input_id for s in sel.selected] == [s.input_id for s in chosen]
        assert (sel.total_expansions, sel.effective_len) == (total, eff)
    with pytest.raises(ConfigError):
        A.select_min_lt(st, 2)


def test_merge_reports_sums_counters_and_renumbers_trace():
    from paper_2010_02164_b200.metrics import CostParams, MetricsReport, merge_reports

    a, b = MetricsReport.new(trace=True), MetricsReport.new(trace=True)
    cp = CostParams(1.0, 1.0)
    for r, steps in ((a, [(4, 1), (6, 2)]), (b, [(3, 1), (5, 2), (2, 3)])):
        for e, L in steps:
            r.record_step(e, L, cp)
    m = merge_reports([a, b], trace=True)
    assert (m.timesteps, m.candidate_expansions) == (5, 20)
    assert m.simulated_cost == a.simulated_cost + b.simulated_cost
    assert [r.timestep for r in m.per_step_trace] == [1, 2, 3, 4, 5]
    assert [(r.expansions, r.effective_len) for r in m.per_step_trace] == [(4, 1), (6, 2), (3, 1), (5, 2), (2, 3)]


def test_flatten_checked_matches_numpy_path_and_reference_errors():
    """The C corpus flattening for the device upload (_vsmat.flatten) equals
    the numpy path and rejects inputs with the reference's DataErrors
    (bb/model.py:90-102): empty input, token outside [0, V), non-int items."""
    import numpy as np

    from paper_2010_02164_b200.errors import DataError
    from paper_2010_02164_b200.harness import flatten, flatten_checked

    rng = random.Random(3)
    corpus = [tuple(rng.randrange(50) for _ in range(rng.randrange(1, 30))) for _ in range(300)]
    corpus += [list(c) for c in corpus[:20]] + [range(3, 9)]
    tok, off = flatten_checked(corpus, 50)
    wt, wo = flatten(corpus)
    assert tok.dtype == np.int32 and off.dtype == np.int32
    assert np.array_equal(tok, wt) and np.array_equal(off, wo)
    with pytest.raises(DataError, match="nonempty"):
        flatten_checked([(1, 2), ()], 50)
    with pytest.raises(DataError, match="token 50 at position 1 is outside"):
        flatten_checked([(1, 2), (3, 50)], 50)
    with pytest.raises(DataError, match="token -1 at position 0"):
        flatten_checked([(-1,)], 50)
    t2, o2 = flatten_checked([[np.int64(5), 6], (7,)], 50)
    assert t2.tolist() == [5, 6, 7] and o2.tolist() == [0, 2, 3]
