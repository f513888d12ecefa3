"""Command-line experiment runner (drop-in for bb/cli.py:30-173).

    python -m paper_2010_02164_b200.cli --engine varstream --model model.json \
        --corpus corpus.txt --k 5 --n 16 --delta 1.5 --max-candidates 3 --out res.json

Same flags and JSON-config merge as the reference; exit codes 0 success,
1 configuration error, 2 I/O or data error, 3 internal invariant violation
(bb/cli.py:154-162).  Model files (JSON "kind"):
  device_hash  -> DeviceHashScorer (seed, scale, power, eos_bias, dtype)
  transformer  -> TransformerScorer (seed, d, heads, layers, enc_layers, ffn, max_src, tau, eos_bias)
  lstm         -> LSTMScorer (seed, emb, hidden, tau, eos_bias)
The reference's seeded_hash / ngram_table scorers are out of scope (SURVEY.md
§2.1): exit code 2.  Reference Scorer objects plug in through the Python API
(run_experiment(ExperimentConfig(..., scorer_spec=<scorer>)), HostScorerAdapter).
"""

from __future__ import annotations

import argparse
import json
import math
import sys
from pathlib import Path

from .core import DecodeConfig, Vocabulary
from .errors import ConfigError, DataError, InvariantViolation

ENGINES = ("greedy", "fixed", "varbeam", "varstream", "varfifo", "fixedstream")
_DECODE = ("k", "n", "epsilon", "delta", "max_candidates", "max_len", "policy", "capacity",
           "flush_interval", "cost_c0", "cost_c1")


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # bad flags are configuration errors (exit 1)
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        raise SystemExit(1)


def _parser():
    p = _Parser(prog="varstream-b200", description="Run one device VarStream experiment.")
    p.add_argument("--config")
    p.add_argument("--engine", choices=ENGINES)
    p.add_argument("--model")
    p.add_argument("--corpus")
    p.add_argument("--out")
    p.add_argument("--k", type=int)
    p.add_argument("--n", type=int)
    p.add_argument("--epsilon", type=float)
    p.add_argument("--delta")
    p.add_argument("--max-candidates", type=int, dest="max_candidates")
    p.add_argument("--max-len", type=int, dest="max_len")
    p.add_argument("--policy", choices=["immediate", "deferred"])
    p.add_argument("--capacity", type=int)
    p.add_argument("--flush-interval", type=int, dest="flush_interval")
    p.add_argument("--cost-c0", type=float, dest="cost_c0")
    p.add_argument("--cost-c1", type=float, dest="cost_c1")
    p.add_argument("--trace", action="store_true", default=None)
    p.add_argument("--seed", type=int)
    return p


def _delta(v):
    if isinstance(v, str):
        if v.strip().lower() in ("inf", "+inf", "infinity"):
            return math.inf
        try:
            return float(v)
        except ValueError as exc:
            raise ConfigError(f"bad delta value {v!r}") from exc
    return float(v)


def main(argv=None) -> int:
    try:
        args = _parser().parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        file_cfg = {}
        if args.config:
            try:
                file_cfg = json.loads(Path(args.config).read_text())
            except json.JSONDecodeError as exc:
                raise DataError(f"config file {args.config} is not valid JSON: {exc}") from exc
        dec = dict(file_cfg.get("decode", {}))
        for name in _DECODE:
            v = getattr(args, name, None)
            if v is not None:
                dec[name] = v
        engine = args.engine or file_cfg.get("engine")
        if engine is None:
            raise ConfigError("an engine is required (--engine or config file)")
        if "k" not in dec or "n" not in dec:
            raise ConfigError("k and n must be stated explicitly")
        if "delta" in dec:
            dec["delta"] = _delta(dec["delta"])
        decode = DecodeConfig(**{k: v for k, v in dec.items() if v is not None})
        model = args.model or file_cfg.get("model")
        if model is None:
            raise ConfigError("a model is required (--model or config file)")
        if not isinstance(model, dict):
            try:
                model = json.loads(Path(model).read_text())
            except json.JSONDecodeError as exc:
                raise DataError(f"model file is not valid JSON: {exc}") from exc
        corpus = args.corpus or file_cfg.get("corpus")
        seed = args.seed if args.seed is not None else int(file_cfg.get("seed", 0))
        trace = args.trace if args.trace is not None else bool(file_cfg.get("trace", False))
        out = args.out or file_cfg.get("out")
        from .harness import ExperimentConfig, SyntheticCorpusSpec, run_experiment

        if isinstance(corpus, dict):
            if "synthetic" not in corpus:
                raise ConfigError("corpus object form must contain a 'synthetic' block")
            exp = ExperimentConfig(engine, model, decode, synthetic=SyntheticCorpusSpec.from_dict(corpus["synthetic"]),
                                   out_path=out, trace=trace, seed=seed)
        elif corpus is not None:
            exp = ExperimentConfig(engine, model, decode, corpus_path=corpus, out_path=out, trace=trace, seed=seed)
        else:
            raise ConfigError("a corpus is required (--corpus or config file)")
        doc = run_experiment(exp)
    except ConfigError as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return 1
    except (DataError, OSError) as exc:
        print(f"i/o error: {exc}", file=sys.stderr)
        return 2
    except InvariantViolation as exc:
        print(f"internal error: {exc}", file=sys.stderr)
        return 3
    m = doc.metrics
    print(f"engine={doc.engine} inputs={len(doc.records)} timesteps={m['timesteps']} "
          f"expansions={m['candidate_expansions']} expansions_per_step={m['expansions_per_step']} "
          f"simulated_cost={m['simulated_cost']}")
    if out:
        print(f"results written to {out}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
