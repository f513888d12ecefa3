"""Multi-rank host logic on CPU (gloo, world_size 2): length-balanced snake
sharding and the final ragged output gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_02164_b200.harness import shard
from paper_2010_02164_b200.parallel import gather_results, pack_results

K, L, N_TOTAL = 4, 8, 23


def _expected(g):
    cnt = 1 + g % 3
    out = []
    for c in range(cnt):
        n = 2 + (g + c) % 5
        out.append((tuple(int((g * 7 + c * 3 + p) % 50) for p in range(n)), -(g + c / 10.0)))
    return out


def _rank_main(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gids = shard(N_TOTAL, world, rank)
    n = len(gids)
    count = torch.zeros(n, dtype=torch.int32)
    lens = torch.full((n * K,), 99, dtype=torch.int32)  # garbage beyond count must be ignored
    scores = torch.full((n * K,), 7.0, dtype=torch.float64)
    offs = torch.full((n * K,), 10 ** 6, dtype=torch.int32)
    toks = torch.full((n * K * L,), -5, dtype=torch.int32)
    fill = 0
    # the engine's append layout: emissions land in out_tok in device order,
    # not input order (here: inputs in reverse)
    for li in reversed(range(n)):
        ex = _expected(int(gids[li]))
        count[li] = len(ex)
        for c, (t, sc) in enumerate(ex):
            o = li * K + c
            lens[o] = len(t)
            scores[o] = sc
            offs[o] = fill
            toks[fill:fill + len(t)] = torch.tensor(t, dtype=torch.int32)
            fill += len(t)
    res = gather_results(pack_results(count, lens, scores, offs, toks, K), N_TOTAL)
    if rank == 0:
        got = [[(c.tokens, c.score) for c in res[g]] for g in range(N_TOTAL)]
        q.put(got)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_two_rank_gather_reassembles_global_order():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == [_expected(g) for g in range(N_TOTAL)]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_snake_shard_is_a_balanced_partition(world):
    n = 1000
    lens = np.sort(np.random.default_rng(0).geometric(1 / 25, n))[::-1]
    parts = [shard(n, world, r) for r in range(world)]
    allidx = np.sort(np.concatenate(parts))
    assert np.array_equal(allidx, np.arange(n))
    sums = [lens[p].sum() for p in parts]
    counts = [len(p) for p in parts]
    assert max(counts) - min(counts) <= 1
    assert max(sums) / max(1, min(sums)) < 1.05
    for p in parts:  # each shard stays length-sorted
        assert np.all(np.diff(lens[p]) <= 0)


def test_merge_packs_restores_shard_order():
    """Concurrent batches' packed outputs merge into the shard-order pack."""
    from paper_2010_02164_b200.harness import shard
    from paper_2010_02164_b200.parallel import merge_packs

    rng = np.random.default_rng(0)
    n = 23
    want = []
    for i in range(n):
        c = int(rng.integers(1, 4))
        want.append([(list(rng.integers(0, 50, int(rng.integers(1, 6)))), float(rng.random())) for _ in range(c)])
    subs = [shard(n, 3, q) for q in range(3)]
    packs = []
    for ids in subs:
        cnt = torch.tensor([len(want[i]) for i in ids], dtype=torch.int32)
        lens = torch.tensor([len(t) for i in ids for t, _ in want[i]], dtype=torch.int32)
        sc = torch.tensor([s for i in ids for _, s in want[i]], dtype=torch.float64)
        tk = torch.tensor([x for i in ids for t, _ in want[i] for x in t], dtype=torch.int32)
        packs.append((cnt, lens, sc, tk))
    cnt, lens, sc, tk = merge_packs(packs, subs, n)
    got, e, o = [], 0, 0
    for i in range(n):
        per = []
        for _ in range(int(cnt[i])):
            L = int(lens[e])
            per.append((tk[o:o + L].tolist(), float(sc[e])))
            o += L
            e += 1
        got.append(per)
    assert got == [[(list(map(int, t)), s) for t, s in w] for w in want]
