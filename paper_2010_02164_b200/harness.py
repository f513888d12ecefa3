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
