"""The reference's per-beam and per-batch entry points (bb/__init__.py:72-125),
for callers that drive the search themselves instead of through
``run_varstream``.

Every expansion below runs on the device: ``advance_beam`` / ``beam_decode``
/ ``greedy_decode`` score rows through the reference Scorer protocol
(bb/model.py:78-87) and expand with K1-f64 + K2 (``search.expand_beams``);
``flush_all`` and ``execute_step`` advance ALL selected beams of a step in one
device launch pair.  The scheduler bookkeeping (``refill``, ``select_*``) and
the pure pool filters (``apply_heuristics`` and friends) operate on the same
host value types the reference exposes; they carry no arithmetic beyond the
fp64 comparisons the reference specifies.

Reference: search bb/search.py:38-49, :205-242; heuristics
bb/heuristics.py:21-93; scheduler bb/scheduler.py:48-234.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Sequence

from .core import Beam, Candidate, DecodeConfig, Proposal, Vocabulary, proposal_order
from .errors import ConfigError, InvariantViolation
from .metrics import CostParams, MetricsReport


def _vocab(scorer) -> Vocabulary:
    v = scorer.vocab
    return v if isinstance(v, Vocabulary) else Vocabulary(v.size, v.sos, v.eos)


# ------------------------------------------------------------------ search
def beam_finished(beam: Beam, config: DecodeConfig) -> bool:
    """bb/search.py:205-212: empty, k emitted, or at the length cap."""
    return not beam.candidates or beam.emitted >= config.k or beam.l_t >= config.max_len


def _rows(beam: Beam, encoding, scorer):
    # rows for the active candidates, in beam order (bb/search.py:223-225)
    return [scorer.score_next(encoding, c) for c in beam.candidates if not c.finalized]


def advance_beam(beam: Beam, encoding, scorer, config: DecodeConfig):
    """bb/search.py:215-230: score the active candidates, expand on the
    device, drain at the length cap.  Returns (next beam, emitted)."""
    from .search import expand_beam

    return expand_beam(beam, _rows(beam, encoding, scorer), config, _vocab(scorer), drain=True)


def beam_decode(encoding, scorer, config: DecodeConfig) -> list[Candidate]:
    """bb/search.py:233-242: the unbatched search of one input."""
    beam = Beam.initial(encoding.input_id, _vocab(scorer).sos)
    out: list[Candidate] = []
    while True:
        beam, emitted = advance_beam(beam, encoding, scorer, config)
        out += emitted
        if beam_finished(beam, config):
            return out


def greedy_decode(encoding, scorer, max_len: int) -> Candidate:
    """bb/search.py:38-49: argmax (ties to the lower id) until EOS or max_len —
    a width-one fixed beam, which is what the device runs (k=1, M=1, δ=inf)."""
    cfg = DecodeConfig(k=1, n=1, delta=math.inf, max_candidates=1, max_len=max_len)
    return beam_decode(encoding, scorer, cfg)[0]


# -------------------------------------------------------------- heuristics
@dataclass(frozen=True, slots=True)
class HeuristicConfig:
    """bb/heuristics.py:21-39: δ = +inf and max_candidates = k disable pruning."""

    delta: float
    max_candidates: int

    def __post_init__(self) -> None:
        if not self.delta >= 0.0:
            raise ConfigError(f"delta must be >= 0 or +inf, got {self.delta}")
        if self.max_candidates < 1:
            raise ConfigError(f"max_candidates must be >= 1, got {self.max_candidates}")

    def apply(self, pool: Sequence[Proposal], k: int) -> list[Proposal]:
        return apply_heuristics(pool, k=k, delta=self.delta, max_candidates=self.max_candidates)


def max_candidates_filter(pool: Sequence[Proposal], max_candidates: int, k: int) -> list[Proposal]:
    """bb/heuristics.py:42-64 over a proposal_order-sorted pool: at most
    max_candidates per expanding parent, no-ops exempt but counted, k total."""
    taken: dict[int, int] = {}
    out: list[Proposal] = []
    for p in pool:
        if len(out) == k:
            break
        if p.token is not None:
            if taken.get(p.parent, 0) >= max_candidates:
                continue
            taken[p.parent] = taken.get(p.parent, 0) + 1
        out.append(p)
    return out


def absolute_threshold_filter(candidates: Sequence, delta: float, best_score: float) -> list:
    """bb/heuristics.py:67-78: keep score >= best_score - delta (fp64, inclusive)."""
    if delta == math.inf:
        return list(candidates)
    floor_ = best_score - delta
    return [c for c in candidates if c.score >= floor_]


def apply_heuristics(pool: Sequence[Proposal], *, k: int, delta: float,
                     max_candidates: int) -> list[Proposal]:
    """bb/heuristics.py:81-93: rank, cap, threshold against the rank-1 score."""
    if not pool:
        raise InvariantViolation("pruning an empty expansion pool")
    capped = max_candidates_filter(sorted(pool, key=proposal_order), max_candidates, k)
    return absolute_threshold_filter(capped, delta, capped[0].score)


# --------------------------------------------------------------- scheduler
@dataclass
class BeamSlot:
    """bb/scheduler.py:48-54: a live beam with its input's encoding."""

    beam: Beam
    encoding: object
    input_id: int


@dataclass
class BatchState:
    """bb/scheduler.py:57-65: live beams in arrival order, outputs, cursor, timestep."""

    beams: list = field(default_factory=list)
    outputs: dict = field(default_factory=dict)
    cursor: int = 0
    timestep: int = 0


@dataclass(frozen=True)
class StepSelection:
    """bb/scheduler.py:68-74."""

    selected: tuple
    total_expansions: int
    effective_len: int


def refill(state: BatchState, corpus, config: DecodeConfig, scorer) -> list[int]:
    """bb/scheduler.py:94-116: admit inputs in stream order until n are live."""
    sos = _vocab(scorer).sos
    room = max(0, min(config.n - len(state.beams), len(corpus) - state.cursor))
    admitted = list(range(state.cursor, state.cursor + room))
    for i in admitted:
        state.beams.append(BeamSlot(Beam.initial(i, sos), scorer.encode(corpus[i], input_id=i), i))
        state.outputs[i] = []
    state.cursor += room
    return admitted


def _pack(slots, capacity: int):
    # bb/scheduler.py:119-132: greedy arrival-order fill that skips a beam
    # which would overflow and keeps scanning
    chosen, rows = [], 0
    for s in slots:
        w = s.beam.active_width()
        if w > capacity:
            raise ConfigError(f"a single beam needs {w} expansions but capacity is {capacity}")
        if rows + w <= capacity:
            chosen.append(s)
            rows += w
    return chosen, rows


def select_min_lt(state: BatchState, capacity: int) -> StepSelection:
    """bb/scheduler.py:135-144: the beams at the smallest l_t, arrival order."""
    if not state.beams:
        raise InvariantViolation("selection requires at least one live beam")
    low = min(s.beam.l_t for s in state.beams)
    chosen, rows = _pack([s for s in state.beams if s.beam.l_t == low], capacity)
    return StepSelection(tuple(chosen), rows, low)


def select_fifo_max_lt(state: BatchState, capacity: int) -> StepSelection:
    """bb/scheduler.py:147-157: longest l_t first, arrival order within ties."""
    if not state.beams:
        raise InvariantViolation("selection requires at least one live beam")
    order = sorted(range(len(state.beams)), key=lambda i: (-state.beams[i].beam.l_t, i))
    chosen, rows = _pack([state.beams[i] for i in order], capacity)
    return StepSelection(tuple(chosen), rows, max((s.beam.l_t for s in chosen), default=0))


def _select_all(state: BatchState, capacity: int) -> StepSelection:
    chosen, rows = _pack(state.beams, capacity)
    return StepSelection(tuple(chosen), rows, max((s.beam.l_t for s in chosen), default=0))


def execute_step(state: BatchState, selection: StepSelection, scorer, config: DecodeConfig,
                 report: MetricsReport, *, phase: str = "stream", refilled=(),
                 on_step: Callable | None = None) -> None:
    """bb/scheduler.py:168-205: advance every selected beam — all of them in
    one device expansion (K1-f64 + one beam-step launch) — record the step,
    remove finished beams stably, emit the StepEvent."""
    from .engine import StepEvent
    from .search import expand_beams

    sel = list(selection.selected)
    rows = [_rows(s.beam, s.encoding, scorer) for s in sel]
    for s, (nxt, emitted) in zip(sel, expand_beams([s.beam for s in sel], rows, config, _vocab(scorer),
                                                   drain=True)):
        s.beam = nxt
        state.outputs[s.input_id].extend(emitted)
    state.timestep += 1
    report.record_step(selection.total_expansions, selection.effective_len,
                       CostParams(config.cost_c0, config.cost_c1))
    finished = tuple(s.input_id for s in sel if beam_finished(s.beam, config))
    state.beams = [s for s in state.beams if not beam_finished(s.beam, config)]
    if on_step is not None:
        on_step(StepEvent(state.timestep, phase, tuple(refilled), tuple(s.input_id for s in sel),
                          selection.total_expansions, selection.effective_len, finished,
                          tuple(s.input_id for s in state.beams)))


def flush_all(state: BatchState, scorer, config: DecodeConfig, report: MetricsReport | None = None,
              on_step: Callable | None = None) -> BatchState:
    """bb/scheduler.py:208-234: run every live beam to termination, honouring
    capacity; the cursor is untouched."""
    report = report if report is not None else MetricsReport.new()
    while state.beams:
        execute_step(state, _select_all(state, config.capacity), scorer, config, report, phase="flush",
                     on_step=on_step)
    return state
