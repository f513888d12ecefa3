"""Batched decoding drivers (drop-ins for bb/scheduler.py:290-367 and
bb/harness.py:241-260), executed by the device engine.

Signatures match the reference: ``run_varstream(corpus, scorer, config, *,
trace=False, on_step=None) -> (outputs, MetricsReport)`` where outputs[i] is
the list of Candidates emitted for input i (in input order).  ``scorer`` may
be a BatchedScorer (device) or any reference-protocol Scorer
(bb/model.py:78-87), which is wrapped in HostScorerAdapter.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .core import Candidate, DecodeConfig, Vocabulary
from .engine import SearchEngine, drive_concurrent
from .errors import ConfigError
from .harness import flatten_checked, shard
from .metrics import CostParams, MetricsReport, merge_reports
from .scorers import HostScorerAdapter

ENGINES = ("greedy", "fixed", "varbeam", "varstream", "varfifo", "fixedstream")
_PRUNING_OFF = {"fixed": "varbeam", "fixedstream": "varstream"}


def _as_batched(scorer, corpus):
    if all(hasattr(scorer, a) for a in ("bind", "on_admit", "logits", "after_step")):
        return scorer
    return HostScorerAdapter(scorer, corpus)


def _vocab(scorer) -> Vocabulary:
    v = scorer.vocab
    return v if isinstance(v, Vocabulary) else Vocabulary(v.size, v.sos, v.eos)


_ENGINES: dict = {}


def _engine(config: DecodeConfig, vocab: Vocabulary, q: int = 0):
    """Engines (and their streams) are reused across calls with the same
    config and vocabulary on the current device: their buffers and captured
    step graphs persist, so a repeated call costs only the decode."""
    key = (config, (vocab.size, vocab.sos, vocab.eos), torch.cuda.current_device(), q)
    hit = _ENGINES.get(key)
    if hit is None:
        eng = SearchEngine(config, vocab)
        hit = _ENGINES[key] = (eng, torch.cuda.Stream(eng.device) if q else None)
    return hit


def _fork_for(eng: SearchEngine, scorer):
    sig = getattr(scorer, "signature", None)
    if sig is None:
        return scorer.fork()
    if sig not in eng._forks:
        eng._forks[sig] = scorer.fork()
    return eng._forks[sig]


def _run_concurrent(corpus, scorer, config, admit, select, trace, streams):
    """`streams` independent refilling batches (each of config.n slots), the
    length-sorted corpus dealt snake-wise over them as across GPUs, driven
    concurrently on separate CUDA streams of one device.  Every input's output
    is independent of batch composition (bb SPEC.md:379), so the candidates
    equal a single-batch run's; the MetricsReport sums the batches' counters."""
    # flattened once; the reference's input checks over the whole corpus
    # before any batch launches
    tok, off = flatten_checked(corpus, _vocab(scorer).size)
    lens = np.diff(off)
    shards = [shard(len(corpus), streams, q) for q in range(streams)]
    out = [[] for _ in range(len(corpus))]
    engines, jobs = [], []
    for q in range(streams):
        eng, stream = _engine(config, _vocab(scorer), q)
        sc = scorer if q == 0 else _fork_for(eng, scorer)
        ids = np.asarray(shards[q], dtype=np.int64)
        sub_off = np.zeros(len(ids) + 1, dtype=np.int32)
        np.cumsum(lens[ids], out=sub_off[1:])
        gather = np.repeat(off[ids].astype(np.int64) - sub_off[:-1], lens[ids]) + np.arange(int(sub_off[-1]))
        # outputs stream into `out` (global ids) while the batches decode
        gen = eng.async_steps(None, sc, admit_mode=admit, select_mode=select, trace=trace,
                              src_tok=tok[gather], src_off=sub_off, harvest_into=out, gids=shards[q])
        engines.append(eng)
        jobs.append((stream, gen))
    reports = drive_concurrent(jobs)
    # counters summed over the batches; trace renumbered (metrics.merge_reports)
    return out, merge_reports(reports, trace)


def _run(corpus, scorer, config, admit, select, flush, trace, on_step, fast, streams=1):
    if not len(corpus):
        raise ConfigError("corpus must be nonempty")
    bs = _as_batched(scorer, corpus)
    if streams > 1:
        if on_step is not None or (flush and config.flush_interval) or not hasattr(bs, "fork"):
            raise ConfigError("streams > 1 needs a forkable device scorer, no on_step and no flush valve")
        return _run_concurrent(corpus, bs, config, admit, select, trace, streams)
    if fast and on_step is None and not (flush and config.flush_interval):
        if not isinstance(bs, HostScorerAdapter) and not getattr(bs, "host_sync", False):
            eng = _engine(config, _vocab(bs))[0] if getattr(bs, "graph_safe", False) else \
                SearchEngine(config, _vocab(bs))
            return eng.run_async(corpus, bs, admit_mode=admit, select_mode=select, trace=trace)
    eng = SearchEngine(config, _vocab(bs))
    return eng.run(corpus, bs, admit_mode=admit, select_mode=select, flush_enabled=flush,
                   trace=trace, on_step=on_step)


def run_varstream(corpus, scorer, config: DecodeConfig, *, trace: bool = False, on_step=None,
                  fast: bool = True, streams: int = 1):
    """ε-refill + min-l_t selection (bb/scheduler.py:314-340).  ``streams`` > 1
    runs that many independent refilling batches concurrently on one GPU."""
    return _run(corpus, scorer, config, N.VS_ADMIT_VARSTREAM, N.VS_SELECT_MIN_LT, True, trace,
                on_step, fast, streams)


def run_varbeam(corpus, scorer, config: DecodeConfig, *, trace: bool = False, on_step=None,
                fast: bool = True):
    """Traditional batching: admit only when empty (bb/scheduler.py:290-311)."""
    return _run(corpus, scorer, config, N.VS_ADMIT_VARBEAM, N.VS_SELECT_MIN_LT, False, trace,
                on_step, fast)


def run_varfifo(corpus, scorer, config: DecodeConfig, *, trace: bool = False, on_step=None,
                fast: bool = True):
    """Always-full batch, most-advanced first (bb/scheduler.py:343-367)."""
    return _run(corpus, scorer, config, N.VS_ADMIT_VARFIFO, N.VS_SELECT_FIFO, False, trace,
                on_step, fast)


def run_greedy(corpus, scorer, config: DecodeConfig, *, trace: bool = False):
    """Greedy decoding of every input (bb/search.py:38-49 greedy_decode via
    bb/harness.py:222-238 _run_greedy): repeatedly append the argmax token
    (ties to the lower id) until EOS or max_len.

    The reference decodes one input at a time; here all inputs stream
    through one device batch as width-1 beams (k=1, M=1, δ=inf, ε-refill with
    n = config.n * config.k slots), which yields the same candidates
    (bb tests/test_harness.py:177-182: greedy == width-one fixed).  The
    MetricsReport keeps the reference's unbatched accounting: one step of one
    expansion per appended token, effective_len = prefix length
    (bb/harness.py:235-236)."""
    n = max(1, min(N.VS_MAX_SLOTS, config.n * config.k))
    g = DecodeConfig(k=1, n=n, epsilon=config.epsilon, delta=math.inf, max_candidates=1,
                     max_len=config.max_len, cost_c0=config.cost_c0, cost_c1=config.cost_c1)
    outs, _ = run_varstream(corpus, scorer, g)
    report = MetricsReport.new(trace=trace)
    cost = CostParams(config.cost_c0, config.cost_c1)
    for per in outs:
        for length in range(1, len(per[0].tokens)):
            report.record_step(1, length, cost)
    return [[per[0]] for per in outs], report


def dispatch_engine(engine: str, corpus, scorer, config: DecodeConfig, *, trace: bool = False):
    """bb/harness.py:241-260."""
    if engine == "greedy":
        return run_greedy(corpus, scorer, config, trace=trace)
    runner = {"fixed": run_varbeam, "varbeam": run_varbeam, "varstream": run_varstream,
              "fixedstream": run_varstream, "varfifo": run_varfifo}.get(engine)
    if runner is None:
        raise ConfigError(f"unknown engine {engine!r}")
    if engine in _PRUNING_OFF and (config.delta != math.inf or config.max_candidates != config.k):
        raise ConfigError(f"engine {engine!r} requires pruning off: delta=inf and max_candidates=k")
    return runner(corpus, scorer, config, trace=trace)
