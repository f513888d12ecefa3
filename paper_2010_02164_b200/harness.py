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

import itertools
import math
import random
from dataclasses import dataclass

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


def check_corpus(tok: np.ndarray, off: np.ndarray, vocab_size: int) -> None:
    """The reference's input checks (bb/model.py:90-102 _check_input_tokens,
    run at encode time there) over a flattened corpus at once: every input
    nonempty, every token inside the vocabulary; raises DataError with the
    reference's messages."""
    lens = np.diff(off)
    if (lens <= 0).any():
        raise DataError("inputs must be nonempty")
    bad = np.flatnonzero((tok < 0) | (tok >= vocab_size))
    if bad.size:
        j = int(bad[0])
        i = int(np.searchsorted(off, j, side="right")) - 1
        raise DataError(f"token {int(tok[j])} at position {j - int(off[i])} is outside the vocabulary "
                        f"(size {vocab_size})")


def flatten(corpus, dtype=np.int32) -> tuple[np.ndarray, np.ndarray]:
    """(src_tok [total], src_off int32 [N+1]) for SearchEngine.load_corpus
    (tokens as `dtype`: int64 to range-check them before narrowing)."""
    lens = np.fromiter((len(x) for x in corpus), dtype=np.int64, count=len(corpus))
    off = np.zeros(len(corpus) + 1, dtype=np.int32)
    np.cumsum(lens, out=off[1:])
    tok = np.fromiter(itertools.chain.from_iterable(corpus), dtype=dtype, count=int(off[-1]))
    return tok, off


def flatten_checked(corpus, vocab_size: int) -> tuple[np.ndarray, np.ndarray]:
    """flatten + check_corpus for the device upload: (src_tok int32, src_off
    int32), one C pass (host extension _vsmat.flatten) instead of Python
    iteration; on any rejected input the numpy path re-checks and raises the
    reference's DataError (bb/model.py:90-102)."""
    from ._native import load_vsmat

    res = load_vsmat().flatten(corpus, int(vocab_size))
    if res is not None and res[2]:
        return np.frombuffer(res[0], dtype=np.int32), np.frombuffer(res[1], dtype=np.int32)
    tok, off = flatten(corpus, dtype=np.int64)
    check_corpus(tok, off, vocab_size)
    return tok.astype(np.int32), off


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
    return Corpus(inputs)


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


class Corpus(tuple):
    """bb/harness.py:35-44: ordered token-id inputs (``Corpus(inputs)``;
    ``.inputs``, ``len``, indexing)."""

    def __new__(cls, inputs=()):
        return super().__new__(cls, (tuple(int(t) for t in x) for x in inputs))

    @property
    def inputs(self) -> tuple:
        return tuple(self)


@dataclass(frozen=True)
class SyntheticCorpusSpec:
    """bb/harness.py:118-138."""

    n_inputs: int
    distribution: str = "geometric"
    mean_len: float = 8.0
    min_len: int = 1
    max_len: int = 16

    @classmethod
    def from_dict(cls, raw: dict) -> "SyntheticCorpusSpec":
        try:
            return cls(int(raw["n_inputs"]), str(raw.get("distribution", "geometric")),
                       float(raw.get("mean_len", 8.0)), int(raw.get("min_len", 1)), int(raw.get("max_len", 16)))
        except (KeyError, TypeError, ValueError) as exc:
            raise ConfigError(f"bad synthetic corpus spec: {exc}") from exc


def build_scorer(model: dict):
    """A scorer from a model description (the CLI's model file): ``device_hash``
    (csrc/hash_scorer.cu), ``transformer`` (decoder.TransformerScorer) or
    ``lstm`` (decoder.LSTMScorer).  The reference's seeded-hash and n-gram
    table scorers are out of scope; reference Scorer objects
    plug in directly through the Python API (scorers.HostScorerAdapter)."""
    from .core import Vocabulary

    try:
        kind = model["kind"]
        vocab = Vocabulary(int(model["vocab_size"]), int(model["sos"]), int(model["eos"]))
    except KeyError as exc:
        raise DataError(f"model file missing field {exc}") from exc
    if kind == "device_hash":
        from .scorers import DeviceHashScorer

        return DeviceHashScorer(vocab, int(model.get("seed", 0)), scale=float(model.get("scale", 0.5)),
                                power=int(model.get("power", 0)), eos_bias=float(model.get("eos_bias", 4.0)),
                                dtype=str(model.get("dtype", "bf16")))
    if kind in ("transformer", "lstm"):
        from . import decoder

        keys = ("d", "heads", "layers", "enc_layers", "ffn", "max_src", "seed", "hidden", "emb")
        kw = {k: int(model[k]) for k in keys if k in model}
        for k in ("tau", "eos_bias"):
            if k in model:
                kw[k] = float(model[k])
        cls = decoder.TransformerScorer if kind == "transformer" else decoder.LSTMScorer
        return cls(vocab, **kw)
    raise DataError(f"unknown model kind {kind!r} (this build: device_hash, transformer, lstm; "
                    "the reference's seeded_hash / ngram_table scorers are out of scope)")


@dataclass(frozen=True)
class ExperimentConfig:
    """bb/harness.py:140-168.  ``scorer_spec`` is a model description dict
    (``build_scorer``) or a scorer object (BatchedScorer or reference-protocol
    Scorer)."""

    engine: str
    scorer_spec: object
    decode: object
    corpus_path: str | None = None
    synthetic: SyntheticCorpusSpec | None = None
    out_path: str | None = None
    trace: bool = False
    seed: int = 0

    def __post_init__(self) -> None:
        from .scheduler import ENGINES

        if self.engine not in ENGINES:
            raise ConfigError(f"unknown engine {self.engine!r}; expected one of {', '.join(ENGINES)}")
        if (self.corpus_path is None) == (self.synthetic is None):
            raise ConfigError("exactly one of corpus_path or synthetic is required")
        if self.trace and self.out_path is None:
            raise ConfigError("trace output requires an output path")
        if self.engine in ("fixed", "fixedstream") and (
                self.decode.delta != math.inf or self.decode.max_candidates != self.decode.k):
            raise ConfigError(f"engine {self.engine!r} requires pruning off: delta=inf and max_candidates=k")


def run_experiment(config: ExperimentConfig) -> ResultsDocument:
    """bb/harness.py:280-331: load or synthesise the corpus, bucket by length,
    decode on the device with the configured engine (dispatch_engine),
    restore input order, optionally write the results and the trace."""
    from .scheduler import dispatch_engine

    spec = config.scorer_spec
    scorer = build_scorer(spec) if isinstance(spec, dict) else spec
    if config.corpus_path is not None:
        corpus = load_corpus(config.corpus_path)
        corpus_echo: dict = {"path": str(config.corpus_path)}
    else:
        syn = config.synthetic
        corpus = generate_synthetic_corpus(config.seed, syn.n_inputs, scorer.vocab.size,
                                           distribution=syn.distribution, mean_len=syn.mean_len,
                                           min_len=syn.min_len, max_len=syn.max_len)
        corpus_echo = {"synthetic": dict(syn.__dict__) | {"seed": config.seed}}
    bucketed, perm = bucket_by_length(corpus)
    outputs, report = dispatch_engine(config.engine, bucketed, scorer, config.decode, trace=config.trace)
    records = [None] * len(corpus)
    for pos, orig in enumerate(perm):
        records[orig] = {"input_id": orig,
                         "candidates": [{"tokens": list(c.tokens), "score": c.score} for c in outputs[pos]]}
    model_echo = spec if isinstance(spec, dict) else {"kind": type(spec).__name__}
    doc = ResultsDocument(config.engine, {"decode": decode_config_echo(config.decode), "model": model_echo,
                                          "corpus": corpus_echo, "seed": config.seed},
                          report.summarize(), records)
    if config.out_path is not None:
        doc.write(config.out_path)
        if config.trace:
            write_trace(report, trace_path_for(config.out_path))
    return doc
