"""B200-native VarStream: streaming variable-width beam search (arXiv 2010.02164).

Drop-in for the reference ``beambatch`` search loop: the same decode API
(``DecodeConfig``, ``run_varstream``/``run_varbeam``/``run_varfifo``,
``dispatch_engine``, ``Candidate``, ``MetricsReport``, ``StepEvent``) with the
per-step search executed by hand-written sm_100a CUDA kernels behind the
C-ABI in include/varstream.h.  There is no CPU fallback.
"""

from .core import (Beam, Candidate, DecodeConfig, FinalizationPolicy, Proposal, Vocabulary,
                   extend, proposal_order, top_k_select)
from .errors import ConfigError, DataError, InvariantViolation
from .metrics import CostParams, MetricsReport, StepRecord, round_half_up, step_cost

__version__ = "0.1.0"

_LAZY = {
    "SearchEngine": "engine", "StepEvent": "engine", "Harvest": "engine",
    "refill_threshold": "engine",
    "DeviceHashScorer": "scorers", "HostScorerAdapter": "scorers", "BatchedScorer": "scorers",
    "run_varstream": "scheduler", "run_varbeam": "scheduler", "run_varfifo": "scheduler",
    "run_greedy": "scheduler",
    "dispatch_engine": "scheduler", "ENGINES": "scheduler",
    "expand_beam": "search", "expand_beams": "search", "row_lse_topm": "search",
    "beam_finished": "api", "advance_beam": "api", "beam_decode": "api", "greedy_decode": "api",
    "HeuristicConfig": "api", "max_candidates_filter": "api", "absolute_threshold_filter": "api",
    "apply_heuristics": "api", "BeamSlot": "api", "BatchState": "api", "StepSelection": "api",
    "refill": "api", "select_min_lt": "api", "select_fifo_max_lt": "api", "flush_all": "api",
    "execute_step": "api",
    "Corpus": "harness", "SyntheticCorpusSpec": "harness", "ExperimentConfig": "harness",
    "run_experiment": "harness", "ResultsDocument": "harness", "load_corpus": "harness",
    "save_corpus": "harness", "bucket_by_length": "harness", "generate_synthetic_corpus": "harness",
    "build_scorer": "harness",
}


def __getattr__(name):  # torch-dependent modules load on first use
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = ["Beam", "Candidate", "ConfigError", "CostParams", "DataError", "DecodeConfig",
           "FinalizationPolicy", "InvariantViolation", "MetricsReport", "Proposal", "StepRecord",
           "Vocabulary", "extend", "proposal_order", "round_half_up", "step_cost",
           "top_k_select", *_LAZY]
