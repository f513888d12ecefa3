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

import numpy as np
import torch
import torch.distributed as dist

from .harness import shard


def pack_results(count: torch.Tensor, lens: torch.Tensor, scores: torch.Tensor, offs: torch.Tensor,
                 toks: torch.Tensor, k: int):
    """Compact engine output buffers (device or CPU tensors; the append layout
    of include/varstream.h: count [n], lens / scores / offs [n*k], tokens
    appended at offs) to the emitted candidates in input order:
    (count [n] i32, lens [E] i32, scores [E] f64, flat tokens [T] i32)."""
    n = count.numel()
    dev = count.device
    emitted = (torch.arange(k, device=dev)[None, :] < count[:, None].long()).reshape(-1)
    lens_e = lens.reshape(-1)[: n * k][emitted].to(torch.int32)
    scores_e = scores.reshape(-1)[: n * k][emitted].to(torch.float64)
    offs_e = offs.reshape(-1)[: n * k][emitted].long()
    flat = toks.reshape(-1)[_ragged_index(offs_e, lens_e)].to(torch.int32)
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


def serialize_pack(packed) -> torch.Tensor:
    """One uint8 buffer per rank: 4 int64 sizes, then count | lens | tokens
    (int32) and scores (fp64, 8-byte aligned) — a single message per rank."""
    count, lens, scores, toks = packed
    dev = count.device
    sizes = torch.tensor([count.numel(), lens.numel(), toks.numel(), scores.numel()], dtype=torch.int64,
                         device=dev)
    parts = [sizes.view(torch.uint8), count.contiguous().view(torch.uint8), lens.contiguous().view(torch.uint8),
             toks.contiguous().view(torch.uint8)]
    ints = sum(p.numel() for p in parts[1:])
    if ints % 8:
        parts.append(torch.zeros(8 - ints % 8, dtype=torch.uint8, device=dev))
    parts.append(scores.contiguous().view(torch.uint8))
    return torch.cat(parts)


def deserialize_pack(buf: np.ndarray):
    """Inverse of serialize_pack on the host: (count, lens, scores, toks) numpy arrays."""
    nc, nl, nt, ns = (int(x) for x in buf[:32].view(np.int64))
    o = 32
    count = buf[o:o + 4 * nc].view(np.int32)
    o += 4 * nc
    lens = buf[o:o + 4 * nl].view(np.int32)
    o += 4 * nl
    toks = buf[o:o + 4 * nt].view(np.int32)
    o += 4 * nt
    o += (-(o - 32)) % 8
    scores = buf[o:o + 8 * ns].view(np.float64)
    return count, lens, scores, toks


def materialize(out: list, gids, count, lens, scores, toks) -> None:
    """Candidate lists of a packed shard into `out` at global ids `gids`
    (bulk, in C: hostsrc/vsmat.c)."""
    from . import _native as N
    from .core import Candidate

    mat = N.load_vsmat()
    if len(toks):
        mat.reserve(int(np.max(toks)) + 1)
    mat.fill_packed(out, np.ascontiguousarray(np.asarray(gids), dtype=np.int64),
                               np.ascontiguousarray(count, dtype=np.int32), np.ascontiguousarray(lens, dtype=np.int32),
                               np.ascontiguousarray(scores, dtype=np.float64),
                               np.ascontiguousarray(toks, dtype=np.int32), Candidate)


def gather_packed(packed, group=None, dst: int = 0):
    """Ship every rank's packed results to rank `dst` as one self-describing
    message per rank (its header holds the sizes): an all-reduce of the
    message length, then one gather of the padded messages.  Returns the
    per-rank uint8 buffers on `dst` (device-resident), None elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    msg = serialize_pack(packed)
    mx = torch.tensor([msg.numel()], dtype=torch.int64, device=msg.device)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    pad = torch.zeros(int(mx.item()), dtype=torch.uint8, device=msg.device)
    pad[: msg.numel()] = msg
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    return bufs


def gather_results(packed, n_total: int, group=None, dst: int = 0):
    """The one data-plane exchange: every rank's packed
    results travel as ONE message to rank `dst` (a gather of the message
    sizes, then a gather of the size-padded messages — NCCL over NVLink on
    B200, gloo in the CPU tests).  Rank `dst` returns list[list[Candidate]]
    in global input order; the others return None."""
    world = dist.get_world_size(group)
    bufs = gather_packed(packed, group, dst)
    if bufs is None:
        return None
    out = [[] for _ in range(n_total)]
    for r in range(world):
        host = bufs[r].cpu().numpy()
        materialize(out, shard(n_total, world, r), *deserialize_pack(host))
    return out


def run_varstream_sharded(corpus, scorer, config, *, group=None, dst: int = 0, streams: int = 1):
    """Public multi-GPU entry: this rank decodes its snake-dealt shard of the
    (length-sorted) corpus on its current CUDA device; outputs are gathered
    to rank `dst`.  Returns (list[list[Candidate]] | None, local MetricsReport)."""
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
        from .metrics import merge_reports

        rep = merge_reports(reps)
        packed = merge_packs([e.packed() for e in engs], subs, len(local))
    elif local:
        eng = SearchEngine(config, _vocab(scorer))
        _, rep = eng.run_async(local, scorer, admit_mode=N.VS_ADMIT_VARSTREAM,
                               select_mode=N.VS_SELECT_MIN_LT, materialize=False)
        packed = eng.packed()
    else:  # more ranks than inputs
        from .metrics import MetricsReport

        rep = MetricsReport.new()
        packed = (torch.zeros(0, dtype=torch.int32, device=dev), torch.zeros(0, dtype=torch.int32, device=dev),
                  torch.zeros(0, dtype=torch.float64, device=dev), torch.zeros(0, dtype=torch.int32, device=dev))
    return gather_results(packed, len(corpus), group, dst), rep
