"""Synthetic inputs and length-balanced sharding.

``generate_synthetic_corpus`` draws the same inputs as the reference generator
(bb/harness.py:85-115, Python ``random.Random(seed)``: geometric or uniform
lengths, uniform tokens); ``clip`` additionally truncates geometric lengths at
the encoder's maximum positions.  ``bucket_by_length`` is the
stable descending length sort of bb/harness.py:72-82.  ``shard`` deals the
length-sorted stream snake-wise across ranks: every shard
stays sorted and length-balanced and keeps its global input ids.
"""

from __future__ import annotations

import math
import random

import numpy as np

from .errors import ConfigError, DataError


def generate_synthetic_corpus(seed: int, n_inputs: int, vocab_size: int, *,
                              distribution: str = "geometric", mean_len: float = 8.0,
                              min_len: int = 1, max_len: int = 16, clip: int | None = None):
    if n_inputs < 1:
        raise ConfigError(f"n_inputs must be >= 1, got {n_inputs}")
    if vocab_size < 2:
        raise ConfigError(f"vocab_size must be >= 2, got {vocab_size}")
    rng = random.Random(seed)
    draw_len = None
    if distribution == "geometric":
        if mean_len < 1.0:
            raise ConfigError(f"mean_len must be >= 1, got {mean_len}")
        p = 1.0 / mean_len
        lg = math.log(1.0 - p) if p < 1.0 else None
        draw_len = (lambda: int(math.log(1.0 - rng.random()) / lg) + 1) if lg else (lambda: 1)
    elif distribution == "uniform":
        if not 1 <= min_len <= max_len:
            raise ConfigError(f"bad uniform length range [{min_len}, {max_len}]")
        draw_len = lambda: rng.randint(min_len, max_len)  # noqa: E731
    else:
        raise ConfigError(f"unknown length distribution {distribution!r}")
    out = []
    for _ in range(n_inputs):
        n = draw_len()
        toks = tuple(rng.randrange(vocab_size) for _ in range(n))
        out.append(toks[:clip] if clip else toks)
    return out


def bucket_by_length(corpus):
    """Stable descending length sort; returns (sorted corpus, permutation)."""
    if not len(corpus):
        raise DataError("cannot bucket an empty corpus")
    perm = sorted(range(len(corpus)), key=lambda i: -len(corpus[i]))
    return [corpus[i] for i in perm], perm


def shard(n_items: int, world: int, rank: int) -> np.ndarray:
    """Snake deal of positions 0..n-1 (already length-sorted) over `world`
    ranks: round r gives rank q position r*world + (q or world-1-q)."""
    idx = np.arange(n_items)
    rnd, pos = idx // world, idx % world
    owner = np.where(rnd % 2 == 0, pos, world - 1 - pos)
    return idx[owner == rank]


def flatten(corpus) -> tuple[np.ndarray, np.ndarray]:
    """(src_tok int32 [total], src_off int32 [N+1]) for SearchEngine.load_corpus."""
    lens = np.fromiter((len(x) for x in corpus), dtype=np.int64, count=len(corpus))
    off = np.zeros(len(corpus) + 1, dtype=np.int32)
    np.cumsum(lens, out=off[1:])
    tok = np.fromiter((t for x in corpus for t in x), dtype=np.int32, count=int(off[-1]))
    return tok, off


# ---------------------------------------------------------------- file formats
# Drop-in for the reference's experiment I/O (bb/harness.py:47-69 corpus text,
# :170-206 results JSON, :209-219 trace CSV, :280-331 run_experiment).

def load_corpus(path):
    """One input per line, whitespace-separated token ids; blank lines skipped."""
    from pathlib import Path

    inputs = []
    for number, line in enumerate(Path(path).read_text().splitlines(), start=1):
        if not line.strip():
            continue
        try:
            toks = tuple(int(x) for x in line.split())
        except ValueError as exc:
            raise DataError(f"{path}: malformed token on line {number}") from exc
        if any(t < 0 for t in toks):
            raise DataError(f"{path}: negative token on line {number}")
        inputs.append(toks)
    if not inputs:
        raise DataError(f"{path}: empty corpus")
    return inputs


def save_corpus(corpus, path) -> None:
    from pathlib import Path

    Path(path).write_text("".join(" ".join(str(t) for t in x) + "\n" for x in corpus))


class ResultsDocument:
    """Per-input candidates (original input order), run metrics, config echo."""

    def __init__(self, engine: str, config: dict, metrics: dict, records):
        self.engine, self.config, self.metrics, self.records = engine, config, metrics, tuple(records)

    def to_dict(self) -> dict:
        return {"engine": self.engine, "config": self.config, "metrics": self.metrics,
                "records": list(self.records)}

    @classmethod
    def from_dict(cls, raw: dict) -> "ResultsDocument":
        return cls(raw["engine"], raw["config"], raw["metrics"], raw["records"])

    def write(self, path) -> None:
        import json
        from pathlib import Path

        Path(path).write_text(json.dumps(self.to_dict(), indent=2) + "\n")

    @classmethod
    def read(cls, path) -> "ResultsDocument":
        import json
        from pathlib import Path

        try:
            raw = json.loads(Path(path).read_text())
        except json.JSONDecodeError as exc:
            raise DataError(f"results file {path} is not valid JSON: {exc}") from exc
        return cls.from_dict(raw)


def trace_path_for(out_path):
    from pathlib import Path

    return Path(str(out_path) + ".trace.csv")


def write_trace(report, path) -> None:
    import csv

    if report.per_step_trace is None:
        raise ConfigError("run was not executed with tracing enabled")
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["timestep", "expansions", "effective_len", "cost"])
        w.writerows(report.per_step_trace)


def decode_config_echo(config) -> dict:
    return {"k": config.k, "n": config.n, "epsilon": config.epsilon,
            "delta": "inf" if config.delta == math.inf else config.delta,
            "max_candidates": config.max_candidates, "max_len": config.max_len,
            "policy": getattr(config.policy, "value", config.policy), "capacity": config.capacity,
            "flush_interval": config.flush_interval, "cost_c0": config.cost_c0,
            "cost_c1": config.cost_c1}


def run_experiment(engine: str, scorer, decode, *, corpus=None, synthetic: dict | None = None,
                   out_path=None, trace: bool = False, seed: int = 0, model_echo: dict | None = None):
    """Load/synthesise the corpus, bucket by length, decode on the device with
    `engine` (dispatch_engine), restore input order, optionally write results
    and trace.  Returns a ResultsDocument."""
    from .scheduler import dispatch_engine

    if (corpus is None) == (synthetic is None):
        raise ConfigError("exactly one of corpus or synthetic is required")
    if trace and out_path is None:
        raise ConfigError("trace output requires an output path")
    if synthetic is not None:
        spec = dict(synthetic)
        n_inputs = int(spec.pop("n_inputs"))
        corpus = generate_synthetic_corpus(seed, n_inputs, scorer.vocab.size, **spec)
        corpus_echo = {"synthetic": dict(synthetic) | {"seed": seed}}
    else:
        corpus_echo = {"inputs": len(corpus)}
    bucketed, perm = bucket_by_length(corpus)
    outputs, report = dispatch_engine(engine, bucketed, scorer, decode, trace=trace)
    records = [None] * len(corpus)
    for pos, orig in enumerate(perm):
        records[orig] = {"input_id": orig,
                         "candidates": [{"tokens": list(c.tokens), "score": c.score} for c in outputs[pos]]}
    doc = ResultsDocument(engine, {"decode": decode_config_echo(decode), "model": model_echo or {},
                                   "corpus": corpus_echo, "seed": seed}, report.summarize(), records)
    if out_path is not None:
        doc.write(out_path)
        if trace:
            write_trace(report, trace_path_for(out_path))
    return doc
