"""End-to-end agreement between a device decode and the reference search on
the same model (TEST / BASELINE INFRASTRUCTURE — only tests/ and bench.py's
reference legs import this).

north_star: decoded sequences match the reference on >= 99.5% of inputs, with
divergences explained only by fp ties.  The device computes its logits with
its own arithmetic (tensor-core GEMMs, fused kernels); the reference computes
them on the CPU.  Identical algorithms on slightly different rows can only
disagree where the reference search itself made a decision by a margin
smaller than the rows' numerical discrepancy.  ``decision_margin`` re-runs
the reference's unbatched per-input search (bb/search.py:233-242, restated in
varstream_oracle.beam_decode — outputs are independent of batching,
bb SPEC.md:379) and returns the smallest margin of every decision it made:

* per-parent top-M boundary: row[M-th] - row[(M+1)-th]   (bb/search.py:69)
* pool order of the entries that decide the beam and the emissions: gaps
  between consecutive scores among the first k+1 ranked proposals
  (bb/core.py:156-158, bb/heuristics.py:42-64)
* δ threshold: |score - (best - δ)| of every ranked proposal (bb/heuristics.py:67-78)

A divergent input is an "fp near-tie" when that margin is below the stated
tolerance of the two arithmetics.
"""

from __future__ import annotations

import math

import numpy as np

from . import varstream_oracle as O


def compare(got, want, rel: float = 1e-5):
    """got/want: per-input lists of (tokens, score).  Returns (all_same, top1_same)."""
    same = len(got) == len(want) and all(
        tuple(a[0]) == tuple(b[0]) and abs(a[1] - b[1]) <= rel * max(1.0, abs(b[1]))
        for a, b in zip(got, want))
    top1 = bool(got) and bool(want) and tuple(got[0][0]) == tuple(want[0][0])
    return same, top1


def compare_detail(got, want, rel: float = 1e-5) -> dict:
    """Per-input agreement classes (got/want: per-input lists of (tokens, score)):
    ``sequences`` — the same decoded token sequences in the same order (north_star:
    "decoded sequences match"); ``set`` — the same sequences, order aside (a swap of
    two near-equal scores); ``scores`` — sequences identical and every score within
    ``rel`` relative; ``top1``; ``max_rel`` — the largest relative score difference
    over a sequence-identical input (None otherwise)."""
    ta = [tuple(a[0]) for a in got]
    tb = [tuple(b[0]) for b in want]
    seq = ta == tb
    worst = None
    if seq:
        worst = max((abs(a[1] - b[1]) / max(1.0, abs(b[1])) for a, b in zip(got, want)), default=0.0)
    return {"sequences": seq, "set": sorted(ta) == sorted(tb), "scores": seq and worst <= rel,
            "top1": bool(ta) and bool(tb) and ta[0] == tb[0], "max_rel": worst}


def summarize(details: list) -> dict:
    """Fractions over compare_detail results (the agreement report's keys)."""
    n = max(1, len(details))
    rels = [d["max_rel"] for d in details if d["max_rel"] is not None]
    return {"sequences_identical_fraction": round(sum(d["sequences"] for d in details) / n, 4),
            "sequence_set_identical_fraction": round(sum(d["set"] for d in details) / n, 4),
            "identical_fraction": round(sum(d["scores"] for d in details) / n, 4),
            "top1_fraction": round(sum(d["top1"] for d in details) / n, 4),
            "max_rel_score_diff_of_identical_sequences": float(f"{max(rels):.3g}") if rels else None}


def decision_margin(encoding, scorer, cfg: O.OConfig) -> float:
    """Smallest decision margin of the reference's deferred-policy search for
    one input (see module docstring)."""
    return decode_with_margin(encoding, scorer, cfg)[1]


def decode_with_margin(encoding, scorer, cfg: O.OConfig):
    """The reference's unbatched search of one input (bb/search.py:233-242)
    and its smallest decision margin, in one pass: (outputs, margin)."""
    beam = O.Beam.initial(encoding.input_id, scorer.sos)
    margin = math.inf
    outputs = []
    while True:
        actives = [(i, c) for i, c in enumerate(beam.candidates) if not c.finalized]
        if getattr(scorer, "incremental", False) and actives:  # the same rows, one batched model pass
            rows = [np.asarray(r, dtype=np.float64) for r in scorer.score_batch(encoding, [c for _, c in actives])]
        else:
            rows = [np.asarray(scorer.score_next(encoding, c), dtype=np.float64) for _, c in actives]
        for row in rows:
            m = min(cfg.max_candidates, row.shape[0])
            if m < row.shape[0]:
                top = np.sort(row)[::-1][: m + 1]
                margin = min(margin, float(top[m - 1] - top[m]))
        pool = O.candidate_pool(beam, actives, rows, cfg.max_candidates, include_noops=True)
        ranked = sorted(pool, key=O.proposal_order)
        head = [p.score for p in ranked[: cfg.k + 1]]
        for a, b in zip(head, head[1:]):
            margin = min(margin, a - b)
        if cfg.delta != math.inf:
            cutoff = ranked[0].score - cfg.delta
            for p in ranked[: cfg.k + 1]:
                margin = min(margin, abs(p.score - cutoff))
        nxt, emitted = O.expand_beam(beam, rows, cfg, scorer.vocab_size, scorer.eos)
        if nxt.l_t >= cfg.max_len and nxt.candidates:
            nxt, drained = O.drain_at_length_cap(nxt, cfg)
            emitted = emitted + drained
        outputs += emitted
        beam = nxt
        if O.beam_finished(beam, cfg):
            return outputs, margin


def agreement_report(corpus, ids, gpu_sig, cpu_sig, scorer, cfg: O.OConfig, tie_tol: float,
                     rel: float = 1e-5):
    """gpu_sig/cpu_sig: {input id: [(tokens, score), ...]}.  Returns a dict with
    the identical fraction (every candidate: tokens equal, score within `rel`),
    the top-1 fraction, and for every divergent input its reference decision
    margin and whether it is an fp near-tie (margin <= tie_tol)."""
    same = top1 = 0
    div = []
    for i in ids:
        s, t = compare(gpu_sig[i], cpu_sig[i], rel)
        same += s
        top1 += t
        if not s:
            enc = scorer.encode(corpus[i], input_id=i)
            m = decision_margin(enc, scorer, cfg)
            div.append({"input": int(i), "top1_same": bool(t), "margin": m, "near_tie": m <= tie_tol})
    n = len(ids)
    return {"inputs": n, "identical_fraction": same / n, "top1_fraction": top1 / n,
            "divergent": len(div), "explained_by_near_ties": sum(d["near_tie"] for d in div),
            "tie_tolerance": tie_tol, "divergences": div}
