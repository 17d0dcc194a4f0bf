"""svg2_sparse_attention_layout on the GPU (SURVEY 8(b) strides, 8(e) reshard, 8(f) row 4): strided (token-major)
inputs read in place, output rows stored straight into token-sharded buffers (the fused unpermute + reverse
all-to-all), and the query-cluster split of a head over ranks.  Every variant must reproduce the plain fused call
bit for bit; the split must give every query cluster to exactly one part and balance the parts' selected pairs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from gpu_helpers import random_qkv, to_dev

pytestmark = pytest.mark.gpu

CQ, CK, ITERS, TOP_P = 12, 24, 3, 0.9


@pytest.fixture(scope="module")
def svg2():
    assert torch.cuda.is_available(), "the -m gpu tests need a CUDA device"
    import paper_2505_18875_b200 as m
    m.load_library()
    return m


def _qkv(B, H, N, d=128, seed=91):
    q, k, v = random_qkv(B, H, N, N, d, seed=seed, groups=10)
    return to_dev(q), to_dev(k), to_dev(v)


@pytest.mark.parametrize("B,H,N", [(1, 3, 2500), (2, 2, 1800)])
def test_token_major_inputs_read_in_place(svg2, B, H, N):
    """Q, K, V held token-major [B, N, H, d] (the Ulysses all-to-all layout), passed as permuted views: same output,
    pairs and caches as the contiguous call, bitwise, cold and warm (also through the FP8 PV path)."""
    Q, K, V = _qkv(B, H, N)
    O, pairs, ex = svg2.sparse_attention(Q, K, V, CQ, CK, ITERS, TOP_P)
    Qt, Kt, Vt = (t.permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3) for t in (Q, K, V))
    assert not Qt.is_contiguous() and Qt.stride(-1) == 1
    O2, pairs2, ex2 = svg2.sparse_attention(Qt, Kt, Vt, CQ, CK, ITERS, TOP_P)
    assert torch.equal(O2, O) and torch.equal(pairs2, pairs)
    assert torch.equal(ex2["q_centroids"], ex["q_centroids"]) and torch.equal(ex2["k_centroids"], ex["k_centroids"])
    Ow, _, _ = svg2.sparse_attention(Q, K, V, CQ, CK, 2, TOP_P, ex["q_centroids"].clone(), ex["k_centroids"].clone(),
                                     warm=True)
    Ow2, _, _ = svg2.sparse_attention(Qt, Kt, Vt, CQ, CK, 2, TOP_P, ex["q_centroids"].clone(),
                                      ex["k_centroids"].clone(), warm=True)
    assert torch.equal(Ow2, Ow)
    O8, _, _ = svg2.sparse_attention(Q, K, V, CQ, CK, 2, TOP_P, fp8=True)
    O82, _, _ = svg2.sparse_attention(Qt, Kt, Vt, CQ, CK, 2, TOP_P, fp8=True)
    assert torch.equal(O82, O8)
    Op, _, _ = svg2.sparse_attention(Q, K, V, CQ, CK, 2, TOP_P, init="kmeans++", seed=5)
    Op2, _, _ = svg2.sparse_attention(Qt, Kt, Vt, CQ, CK, 2, TOP_P, init="kmeans++", seed=5)
    assert torch.equal(Op2, Op)


def test_output_rows_into_token_shards(svg2):
    """out_shards: P = 3 token-sharded [B, N/P, Htot, d] buffers, this call's heads at head offset 2: every output row
    lands in its shard / row / head, bitwise equal to the plain call; nothing else is written."""
    B, H, N, P, Htot, off = 2, 2, 2400, 3, 5, 2
    Q, K, V = _qkv(B, H, N, seed=92)
    O, _, _ = svg2.sparse_attention(Q, K, V, CQ, CK, ITERS, TOP_P)
    n = N // P
    shards = [torch.full((B, n, Htot, 128), 0x7FBF, dtype=torch.int16, device="cuda").view(torch.bfloat16)
              for _ in range(P)]
    t0 = shards[0]
    O2, _, _ = svg2.sparse_attention(Q, K, V, CQ, CK, ITERS, TOP_P, out_shards=dict(
        shards=shards, shard_tokens=n, strides=(t0.stride(0), t0.stride(2), t0.stride(1)), head_offset=off))
    assert O2 is None
    full = torch.cat(shards, dim=1)  # [B, N, Htot, d]
    assert torch.equal(full[:, :, off:off + H].permute(0, 2, 1, 3), O)
    untouched = torch.cat([full[:, :, :off], full[:, :, off + H:]], dim=2).view(torch.int16)
    assert torch.all(untouched == 0x7FBF)


@pytest.mark.parametrize("count", [2, 3, 8])
def test_query_cluster_parts_partition_the_output(svg2, count):
    """part = (p, count): each part writes exactly the rows of its query clusters (cut by cumulative selected-pair
    cost), the parts are disjoint and cover every row, their union is the plain call bitwise, and each part's cost is
    within one cluster of total / count.  Contiguous part ranges (begin, end, count) equal the union of their parts."""
    B, H, N = 1, 3, 3000
    Q, K, V = _qkv(B, H, N, seed=93)
    O, pairs, ex = svg2.sparse_attention(Q, K, V, CQ, CK, ITERS, TOP_P, debug=True)
    lq = ex["q_labels"].cpu().numpy()
    mask = ex["mask"].cpu().numpy().astype(np.int64)
    sk = np.diff(ex["k_offsets"].cpu().numpy(), axis=-1)
    cover = torch.zeros(B, H, N, dtype=torch.int32, device="cuda")
    merged = torch.zeros_like(O).view(torch.int16)
    costs = np.zeros((H, count))
    for p in range(count):
        Op = torch.zeros_like(O)
        Op2, pp, exp_ = svg2.sparse_attention(Q, K, V, CQ, CK, ITERS, TOP_P, part=(p, count), out=Op, debug=True)
        assert torch.equal(pp, pairs)  # selection and caches are the whole head's on every part
        assert torch.equal(exp_["q_centroids"], ex["q_centroids"])
        written = (Op.view(torch.int16) != 0).any(-1)
        cover += written.int()
        merged |= Op.view(torch.int16)
        for h in range(H):
            rows = written[0, h].cpu().numpy()
            cl = np.unique(lq[0, h][rows])
            for i in cl:  # whole clusters only
                assert rows[lq[0, h] == i].all()
            costs[h, p] = sum(int((lq[0, h] == i).sum()) * int(mask[0, h, i] @ sk[0, h]) for i in cl)
    assert torch.all(cover == 1)
    assert torch.equal(merged.view(torch.bfloat16), O)
    for h in range(H):
        sq = np.bincount(lq[0, h], minlength=CQ)
        cmax = max(int(sq[i]) * int(mask[0, h, i] @ sk[0, h]) for i in range(CQ))
        assert costs[h].max() <= costs[h].sum() / count + cmax
    # a contiguous part range in one call
    Or = torch.zeros_like(O)
    svg2.sparse_attention(Q, K, V, CQ, CK, ITERS, TOP_P, part=(0, count - 1, count), out=Or)
    Olast = torch.zeros_like(O)
    svg2.sparse_attention(Q, K, V, CQ, CK, ITERS, TOP_P, part=(count - 1, count), out=Olast)
    assert torch.equal((Or.view(torch.int16) | Olast.view(torch.int16)).view(torch.bfloat16), O)


@pytest.mark.parametrize("H,P", [(2, 4), (3, 8), (5, 2), (4, 4)])
def test_virtual_ranks_split_plan_bitwise(svg2, H, P):
    """The split plan of dist.py for H heads on P ranks (H < P, uneven H % P), run rank by rank in one process with
    every rank's calls storing rows straight into the P token shards: the shards equal the one-process call in
    token-major order, bitwise (the multi-GPU output path with peer stores, ranks simulated on one GPU)."""
    from paper_2505_18875_b200.dist import split_plan, unit_calls
    B, N = 1, 2400
    Q, K, V = _qkv(B, H, N, seed=94)
    O, _, _ = svg2.sparse_attention(Q, K, V, CQ, CK, ITERS, TOP_P)
    n = N // P
    shards = [torch.zeros(B, n, H, 128, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
    t0 = shards[0]
    for units in split_plan(H, P):
        for h0, h1, pb, pe, pc in unit_calls(units):
            svg2.sparse_attention(Q[:, h0:h1], K[:, h0:h1], V[:, h0:h1], CQ, CK, ITERS, TOP_P, part=(pb, pe, pc),
                                  out_shards=dict(shards=shards, shard_tokens=n,
                                                  strides=(t0.stride(0), t0.stride(2), t0.stride(1)), head_offset=h0))
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(shards, dim=1), O.permute(0, 2, 1, 3))


# ---------------------------------------------------------------- two processes, peer stores through CUDA IPC
B2, H2, N2 = 1, 3, 2000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, world, port, to_peer, from_peer, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2505_18875_b200.dist import SplitSVG2
        Q, K, V = _qkv(B2, H2, N2, seed=95)
        n = N2 // world
        Qs, Ks, Vs = (t.permute(0, 2, 1, 3)[:, rank * n:(rank + 1) * n].contiguous() for t in (Q, K, V))
        mine = torch.zeros(B2, n, H2, 128, dtype=torch.bfloat16, device="cuda")
        to_peer.put(mine)  # CUDA IPC handle of this rank's output shard
        peer = from_peer.get(timeout=120)  # the other rank's shard, mapped into this process
        peers = [mine, peer] if rank == 0 else [peer, mine]
        attn = SplitSVG2(H2, CQ, CK, TOP_P, ITERS, 2)
        attn(Qs, Ks, Vs, out_peers=peers)  # cold
        torch.cuda.synchronize()
        dist.barrier()  # both ranks' stores into both shards are complete
        out_q.put((rank, mine.cpu().view(torch.int16).numpy().copy()))
        dist.barrier()  # keep the mapping alive until both have read
    finally:
        dist.destroy_process_group()


def test_two_processes_peer_store_split():
    """H = 3 heads on 2 ranks (head 1 split by query clusters): each process computes its units and stores the rows
    straight into both ranks' token shards (its own and the peer's, mapped through CUDA IPC); each shard equals the
    one-process call bitwise."""
    import paper_2505_18875_b200 as svg2
    Q, K, V = _qkv(B2, H2, N2, seed=95)
    O, _, _ = svg2.sparse_attention(Q, K, V, CQ, CK, ITERS, TOP_P)
    ref = O.permute(0, 2, 1, 3).cpu()
    world = 2
    ctx = mp.get_context("spawn")
    q01, q10 = ctx.Queue(), ctx.Queue()  # rank 0 -> rank 1 and back: each shard's IPC handle
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(0, world, port, q01, q10, out_q)),
             ctx.Process(target=_ipc_worker, args=(1, world, port, q10, q01, out_q))]
    for p in procs:
        p.start()
    got = [out_q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = N2 // world
    for rank, arr in got:
        assert torch.equal(torch.from_numpy(arr).view(torch.bfloat16), ref[:, rank * n:(rank + 1) * n]), rank
