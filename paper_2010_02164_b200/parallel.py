"""Multi-GPU VarStream: length-balanced input sharding + one final output gather.

SURVEY.md §8(e): every input's output is independent of batch composition
(bb SPEC.md:379, tests/test_acceptance.py:70-81), so N length-sorted inputs
are dealt snake-wise across ranks (harness.shard), each rank runs its own
refilling batch with no communication, and the ragged outputs are gathered
once at the end (NCCL over NVLink on B200; gloo in the CPU tests).  The
collective moves only emitted candidates: per-input counts, per-candidate
lengths and fp64 scores, and the flat token stream.
"""

from __future__ import annotations

from collections.abc import Sequence

import numpy as np
import torch
import torch.distributed as dist

from .core import Candidate
from .harness import shard


def pack_results(count: torch.Tensor, lens: torch.Tensor, scores: torch.Tensor, toks: torch.Tensor,
                 k: int, max_len: int):
    """Compact engine output buffers (device or CPU tensors) to the emitted
    candidates only: (count [N] i32, lens [E] i32, scores [E] f64, flat tokens [T] i32)."""
    n = count.numel()
    dev = count.device
    emitted = (torch.arange(k, device=dev)[None, :] < count[:, None].long()).reshape(-1)
    lens_e = lens.reshape(-1)[emitted].to(torch.int32)
    scores_e = scores.reshape(-1)[emitted].to(torch.float64)
    rows = toks.reshape(n * k, max_len)[emitted]
    mask = torch.arange(max_len, device=dev)[None, :] < lens_e[:, None].long()
    flat = rows[mask].to(torch.int32)
    return count.to(torch.int32), lens_e, scores_e, flat


def _all_gather_ragged(t: torch.Tensor, group=None) -> list[torch.Tensor]:
    world = dist.get_world_size(group)
    size = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(size) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(max(sizes), 1)
    pad = torch.zeros(mx, dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t.reshape(-1)
    bufs = [torch.empty(mx, dtype=t.dtype, device=t.device) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return [b[:s] for b, s in zip(bufs, sizes)]


class ShardedResults(Sequence):
    """Global-order per-input candidate lists assembled on the gathering rank."""

    def __init__(self, n_total: int, parts):
        self.n = n_total
        self.index = [None] * n_total  # input -> (part, first candidate, count)
        self.parts = []
        for gids, count, lens, scores, toks in parts:
            offs = np.zeros(len(lens) + 1, dtype=np.int64)
            np.cumsum(lens, out=offs[1:])
            cstart = np.zeros(len(count) + 1, dtype=np.int64)
            np.cumsum(count, out=cstart[1:])
            p = len(self.parts)
            self.parts.append((lens, scores, toks, offs))
            for li, g in enumerate(gids):
                self.index[int(g)] = (p, int(cstart[li]), int(count[li]))

    def __len__(self) -> int:
        return self.n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(self.n))]
        p, c0, cnt = self.index[i]
        lens, scores, toks, offs = self.parts[p]
        return [Candidate(tuple(int(t) for t in toks[offs[c]:offs[c + 1]]), float(scores[c]), True, i)
                for c in range(c0, c0 + cnt)]


def gather_results(packed, n_total: int, group=None, dst: int = 0):
    """All-gather every rank's packed results; rank `dst` returns
    ShardedResults in global input order, the others return None."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    gathered = [_all_gather_ragged(t, group) for t in packed]
    if rank != dst:
        return None
    parts = []
    for r in range(world):
        gids = shard(n_total, world, r)
        count, lens, scores, toks = (g[r].cpu().numpy() for g in gathered)
        parts.append((gids, count, lens, scores, toks))
    return ShardedResults(n_total, parts)


def run_varstream_sharded(corpus, scorer, config, *, group=None, dst: int = 0):
    """Public multi-GPU entry: this rank decodes its snake-dealt shard of the
    (length-sorted) corpus on its current CUDA device; outputs are gathered
    to rank `dst`.  Returns (ShardedResults | None, local MetricsReport)."""
    from . import _native as N
    from .engine import SearchEngine
    from .scheduler import _vocab

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = shard(len(corpus), world, rank)
    local = [corpus[i] for i in mine]
    dev = torch.device(f"cuda:{torch.cuda.current_device()}")
    if local:
        eng = SearchEngine(config, _vocab(scorer))
        _, rep = eng.run_async(local, scorer, admit_mode=N.VS_ADMIT_VARSTREAM,
                               select_mode=N.VS_SELECT_MIN_LT, materialize=False)
        packed = pack_results(eng.t["out_count"], eng.t["out_len"], eng.t["out_score"],
                              eng.t["out_tok"], eng.k, eng.max_len)
    else:  # more ranks than inputs
        from .metrics import MetricsReport

        rep = MetricsReport.new()
        packed = (torch.zeros(0, dtype=torch.int32, device=dev), torch.zeros(0, dtype=torch.int32, device=dev),
                  torch.zeros(0, dtype=torch.float64, device=dev), torch.zeros(0, dtype=torch.int32, device=dev))
    return gather_results(packed, len(corpus), group, dst), rep
