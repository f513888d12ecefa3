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


def _excl_cumsum(x: torch.Tensor) -> torch.Tensor:
    return torch.cumsum(x.long(), 0) - x.long()


def _ragged_index(starts: torch.Tensor, lens: torch.Tensor) -> torch.Tensor:
    """Concatenation of ranges [starts[i], starts[i] + lens[i])."""
    total = int(lens.sum())
    seg = torch.repeat_interleave(torch.arange(lens.numel(), device=lens.device), lens.long(), output_size=total)
    return starts.long()[seg] + (torch.arange(total, device=lens.device) - _excl_cumsum(lens)[seg])


def merge_packs(packs, sub_ids, n_local: int):
    """Merge the packed outputs of concurrent batches (pack q holds the inputs
    ``sub_ids[q]`` of this rank's shard, in that order) into one pack in the
    shard's order — the layout gather_results expects."""
    counts = torch.cat([p[0] for p in packs]).long()
    lens = torch.cat([p[1] for p in packs])
    scores = torch.cat([p[2] for p in packs])
    toks = torch.cat([p[3] for p in packs])
    dev = counts.device
    order = torch.cat([torch.as_tensor(np.asarray(ids), dtype=torch.int64) for ids in sub_ids]).to(dev)
    perm = torch.empty(n_local, dtype=torch.int64, device=dev)
    perm[order] = torch.arange(order.numel(), device=dev)  # local input -> position in the concatenation
    count_l = counts[perm]
    cand = _ragged_index(_excl_cumsum(counts)[perm], count_l)
    lens_l = lens[cand]
    tok = _ragged_index(_excl_cumsum(lens)[cand], lens_l)
    return count_l.to(torch.int32), lens_l.to(torch.int32), scores[cand], toks[tok].to(torch.int32)


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
    """Global-order per-input candidate lists assembled on the gathering rank
    (index arrays built with numpy: no per-input Python work up front)."""

    def __init__(self, n_total: int, parts):
        self.n = n_total
        self.part = np.full(n_total, -1, dtype=np.int32)      # input -> part
        self.cfirst = np.zeros(n_total, dtype=np.int64)       # input -> first candidate in its part
        self.ccount = np.zeros(n_total, dtype=np.int64)
        self.parts = []
        for gids, count, lens, scores, toks in parts:
            gids = np.asarray(gids, dtype=np.int64)
            count = np.asarray(count, dtype=np.int64)
            offs = np.zeros(len(lens) + 1, dtype=np.int64)
            np.cumsum(lens, out=offs[1:])
            cstart = np.zeros(len(count) + 1, dtype=np.int64)
            np.cumsum(count, out=cstart[1:])
            p = len(self.parts)
            self.parts.append((lens, scores, toks, offs))
            self.part[gids] = p
            self.cfirst[gids] = cstart[:-1]
            self.ccount[gids] = count

    def __len__(self) -> int:
        return self.n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(self.n))]
        p, c0, cnt = int(self.part[i]), int(self.cfirst[i]), int(self.ccount[i])
        lens, scores, toks, offs = self.parts[p]
        return [Candidate(tuple(int(t) for t in toks[offs[c]:offs[c + 1]]), float(scores[c]), True, i)
                for c in range(c0, c0 + cnt)]


def gather_packed(packed, group=None):
    """The one collective: all-gather every rank's packed (ragged) results;
    returns, per field, the list of every rank's tensor (device-resident)."""
    return [_all_gather_ragged(t, group) for t in packed]


def gather_results(packed, n_total: int, group=None, dst: int = 0):
    """All-gather every rank's packed results; rank `dst` returns
    ShardedResults in global input order, the others return None."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    gathered = gather_packed(packed, group)
    if rank != dst:
        return None
    parts = []
    for r in range(world):
        gids = shard(n_total, world, r)
        count, lens, scores, toks = (g[r].cpu().numpy() for g in gathered)
        parts.append((gids, count, lens, scores, toks))
    return ShardedResults(n_total, parts)


def run_varstream_sharded(corpus, scorer, config, *, group=None, dst: int = 0, streams: int = 1):
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
    if local and streams > 1 and len(local) >= streams:  # concurrent batches on this GPU
        from .engine import drive_concurrent
        from .scheduler import _engine, _fork_for

        subs = [shard(len(local), streams, q) for q in range(streams)]
        engs, jobs = [], []
        for q in range(streams):
            eng, stream = _engine(config, _vocab(scorer), q)
            sc = scorer if q == 0 else _fork_for(eng, scorer)
            engs.append(eng)
            jobs.append((stream, eng.async_steps([local[int(i)] for i in subs[q]], sc,
                                                 admit_mode=N.VS_ADMIT_VARSTREAM,
                                                 select_mode=N.VS_SELECT_MIN_LT)))
        reps = drive_concurrent(jobs)
        for st, _ in jobs:
            if st is not None:
                torch.cuda.current_stream().wait_stream(st)
        rep = reps[0]
        for r_ in reps[1:]:
            rep.timesteps += r_.timesteps
            rep.candidate_expansions += r_.candidate_expansions
            rep.simulated_cost += r_.simulated_cost
        packed = merge_packs([pack_results(e.t["out_count"], e.t["out_len"], e.t["out_score"], e.t["out_tok"],
                                           e.k, e.max_len) for e in engs], subs, len(local))
    elif local:
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
