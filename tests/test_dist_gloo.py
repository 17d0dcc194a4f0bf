"""Multi-process CPU tests of the head-parallel plumbing (gloo backend, world_size 2 and 4, 127.0.0.1).

They cover the Ulysses reshard index math: seq_to_head / head_to_seq are inverse, seq_to_head gives every rank the
full sequence of exactly its heads, and the head partition covers every head once."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, B, N, H, d, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_18875_b200.dist import head_range, head_to_seq, seq_to_head
        g = torch.Generator().manual_seed(1234)
        full = torch.randn(B, N, H, d, generator=g)  # the same global tensor on every rank
        n = N // world
        local_seq = full[:, rank * n:(rank + 1) * n].contiguous()
        y = seq_to_head(local_seq)
        h0, h1 = head_range(H, rank, world)
        expect = full[:, :, h0:h1].permute(0, 2, 1, 3).contiguous()
        ok1 = torch.equal(y, expect)
        back = head_to_seq(y)
        ok2 = torch.equal(back, local_seq)
        q.put((rank, ok1, ok2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H", [(2, 4), (4, 8), (2, 24)])
def test_ulysses_reshard_roundtrip(world, H):
    B, N, d = 2, 24, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, N, H, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok1 and ok2 for _, ok1, ok2 in results), results


def test_head_range_partition():
    from paper_2505_18875_b200.dist import head_range
    for H, P in [(24, 8), (40, 8), (24, 2), (40, 4)]:
        covered = []
        for r in range(P):
            a, b = head_range(H, r, P)
            covered += list(range(a, b))
        assert covered == list(range(H))
    with pytest.raises(ValueError):
        head_range(24, 0, 5)


def _worker_uneven(rank, world, port, B, N, H, d, heads_per_rank, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_18875_b200.dist import heads_to_seq, seq_to_heads
        g = torch.Generator().manual_seed(99)
        full = torch.randn(B, N, H, d, generator=g)
        n = N // world
        local_seq = full[:, rank * n:(rank + 1) * n].contiguous()
        y = seq_to_heads(local_seq, heads_per_rank)
        expect = full[:, :, heads_per_rank[rank]].permute(0, 2, 1, 3).contiguous()
        ok1 = torch.equal(y, expect)
        back = heads_to_seq(y * 2, heads_per_rank, H)
        ok2 = torch.equal(back, local_seq * 2)
        q.put((rank, ok1, ok2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,heads_per_rank", [(2, [[0, 3, 4], [1, 2]]), (3, [[5], [0, 1, 2, 3], [4]])])
def test_uneven_reshard_roundtrip(world, heads_per_rank):
    """Balanced (uneven) head assignments: each rank receives all tokens of exactly its heads, and the way back
    restores every head of its token chunk."""
    B, N, H, d = 2, 12, sum(len(h) for h in heads_per_rank), 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_uneven, args=(r, world, port, B, N, H, d, heads_per_rank, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok1 and ok2 for _, ok1, ok2 in results), results


def test_balanced_assignment_lpt():
    from paper_2505_18875_b200.dist import balanced_assignment, makespan
    costs = [10, 1, 9, 2, 8, 3, 7, 4]
    a = balanced_assignment(costs, 2)
    assert sorted(h for hs in a for h in hs) == list(range(8))
    assert makespan(costs, a) == 22  # total 44: a perfect split exists and LPT finds it here
    # never worse than the contiguous equal-count split, and within 4/3 of the lower bound (LPT guarantee)
    rng = torch.Generator().manual_seed(3)
    for world in (2, 4, 8):
        c = (torch.rand(24, generator=rng) + 0.5).tolist()
        lb = max(sum(c) / world, max(c))
        a = balanced_assignment(c, world)
        per = 24 // world
        fixed = [list(range(r * per, (r + 1) * per)) for r in range(world)]
        assert makespan(c, a) <= makespan(c, fixed) + 1e-12
        assert makespan(c, a) <= 4.0 / 3.0 * lb + 1e-9


# ------------------------------------------------------------------ query-cluster split
@pytest.mark.parametrize("H,P", [(24, 8), (40, 8), (4, 8), (3, 8), (5, 2), (2, 4), (6, 4), (1, 8), (7, 3)])
def test_split_plan_covers_every_part_once(H, P):
    """Every (head, part) unit is owned by exactly one rank, every rank gets the same number of units, a head's parts
    on one rank are contiguous, and the library calls cover exactly the rank's units (whole heads as (0, 1, 1))."""
    from paper_2505_18875_b200.dist import split_plan, unit_calls
    plan = split_plan(H, P)
    assert len(plan) == P and len({len(u) for u in plan}) == 1
    units = [u for r in plan for u in r]
    k = units[0][2]
    assert sorted((h, p) for h, p, _ in units) == [(h, p) for h in range(H) for p in range(k)]
    assert k == 1 if H % P == 0 else True
    for r in plan:
        covered = set()
        for h0, h1, pb, pe, pc in unit_calls(r):
            for h in range(h0, h1):
                if (pb, pe, pc) == (0, 1, 1):
                    covered |= {(h, p) for p in range(k)}
                else:
                    assert pc == k
                    covered |= {(h, p) for p in range(pb, pe)}
        assert covered == {(h, p) for h, p, _ in r}


def _worker_or(rank, world, port, B, N, H, d, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_18875_b200.dist import heads_of, heads_to_seq_or, seq_to_heads, split_plan
        g = torch.Generator().manual_seed(7)
        full = torch.randn(B, N, H, d, generator=g).to(torch.bfloat16)
        n = N // world
        plan = split_plan(H, world)
        heads = [heads_of(u) for u in plan]
        local_seq = full[:, rank * n:(rank + 1) * n].contiguous()
        y = seq_to_heads(local_seq, heads)  # every rank gets all tokens of its (possibly shared) heads
        ok1 = torch.equal(y, full[:, :, heads[rank]].permute(0, 2, 1, 3).contiguous())
        # this rank "computes" its parts: tokens with (token index) % k in its part range keep their value
        keep = torch.zeros_like(y)
        for h, p, k in plan[rank]:
            a = heads[rank].index(h)
            idx = torch.arange(N) % k == p
            keep[:, a, idx] = y[:, a, idx]
        back = heads_to_seq_or(keep, heads, H)
        ok2 = torch.equal(back.view(torch.int16), local_seq.view(torch.int16))
        q.put((rank, ok1, ok2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H", [(2, 3), (4, 2), (4, 6), (2, 1)])
def test_split_reshard_or_merge_roundtrip(world, H):
    """H < P and H % P != 0: seq_to_heads with shared heads gives every rank all tokens of its heads; rows written by
    exactly one rank (zeros elsewhere) come back to their token shard bit for bit through the OR merge (also -0.0)."""
    B, N, d = 1, 24, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_or, args=(r, world, port, B, N, H, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok1 and ok2 for _, ok1, ok2 in results), results
