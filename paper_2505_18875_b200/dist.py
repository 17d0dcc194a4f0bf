"""Head-parallel SVG2 across the GPUs of one node.

Every SVG2 step is per (b, h) with no cross-head data, so heads shard with no collective inside the method.  The
only exchange is the Ulysses-style reshard of a sequence-parallel DiT: activations arrive token-sharded
[B, N/P, H, d] on each rank, an all-to-all (NCCL over NVLink/NVSwitch via torch.distributed) turns them into
head-sharded [B, H/P, N, d] for attention, and the output goes back the same way.  Rank r owns heads
[r H/P, (r+1) H/P) for the whole run, so its centroid caches stay resident.

torch.distributed is plumbing here: the attention itself runs in libsvg2.so.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist


def head_range(H: int, rank: int, world: int):
    if H % world:
        raise ValueError(f"H={H} heads do not split over {world} ranks")
    per = H // world
    return rank * per, (rank + 1) * per


def _all_to_all(recv: torch.Tensor, send: torch.Tensor, group=None) -> None:
    """all_to_all_single; with a CPU-only backend (gloo, used to exercise the multi-rank path on one GPU) the CUDA
    buffers are staged through host memory."""
    if send.is_cuda and dist.get_backend(group) == "gloo":
        r = torch.empty_like(recv, device="cpu")
        dist.all_to_all_single(r, send.cpu(), group=group)
        recv.copy_(r)
    else:
        dist.all_to_all_single(recv, send, group=group)


def seq_to_head(x: torch.Tensor, group=None) -> torch.Tensor:
    """[B, N/P, H, d] (this rank's token chunk, all heads) -> [B, H/P, N, d] (all tokens, this rank's heads)."""
    world = dist.get_world_size(group)
    B, n, H, d = x.shape
    hp = H // world
    send = x.reshape(B, n, world, hp, d).permute(2, 0, 1, 3, 4).contiguous()  # [P(dest), B, n, H/P, d]
    recv = torch.empty_like(send)                                             # [P(src = token chunk), B, n, H/P, d]
    _all_to_all(recv, send, group)
    return recv.permute(1, 3, 0, 2, 4).reshape(B, hp, world * n, d).contiguous()


def head_to_seq(y: torch.Tensor, group=None) -> torch.Tensor:
    """Inverse of seq_to_head: [B, H/P, N, d] -> [B, N/P, H, d]."""
    world = dist.get_world_size(group)
    B, hp, N, d = y.shape
    n = N // world
    send = y.reshape(B, hp, world, n, d).permute(2, 0, 3, 1, 4).contiguous()  # [P(dest = token chunk), B, n, H/P, d]
    recv = torch.empty_like(send)                                              # [P(src = head group), B, n, H/P, d]
    _all_to_all(recv, send, group)
    return recv.permute(1, 2, 0, 3, 4).reshape(B, n, world * hp, d).contiguous()


# ------------------------------------------------------------------ load balancing
# Dynamic top-p gives every head its own density, so equal head counts per rank are not equal work.
# balanced_assignment() gives each rank a set of heads with near-equal estimated cost (longest-processing-time-first,
# deterministic); the uneven reshards below move each rank's token chunk to the owners of its heads and back.
# The mapping is chosen once (e.g. from the first sparse step's per-head work) and kept, so centroid caches stay
# resident on their rank.


def seq_to_head_overlapped(xs, comm_stream: torch.cuda.Stream, group=None):
    """seq_to_head of several tensors (Q, K, V) on `comm_stream`, one after the other, so that the SVG2 call can start
    on the first while the others are in flight: returns the head-sharded tensors and one CUDA event per tensor,
    recorded when it is complete (for sparse_attention(..., input_ready=events), svg2_sparse_attention_ex).  The
    returned tensors are marked as used by the current stream (caching-allocator safety)."""
    cur = torch.cuda.current_stream()
    comm_stream.wait_stream(cur)
    outs, events = [], []
    with torch.cuda.stream(comm_stream):
        for x in xs:
            x.record_stream(comm_stream)
            y = seq_to_head(x, group)
            ev = torch.cuda.Event()
            ev.record(comm_stream)
            outs.append(y)
            events.append(ev)
    for y in outs:
        y.record_stream(cur)
    return outs, events


def balanced_assignment(costs, world: int):
    """Heads -> ranks with near-equal total cost: heads in decreasing cost (ties: lower index first), each to the
    least-loaded rank (ties: lower rank).  Returns a list of sorted head lists, one per rank."""
    costs = [float(c) for c in costs]
    order = sorted(range(len(costs)), key=lambda h: (-costs[h], h))
    load = [0.0] * world
    heads = [[] for _ in range(world)]
    for h in order:
        r = min(range(world), key=lambda q: (load[q], q))
        heads[r].append(h)
        load[r] += costs[h]
    return [sorted(hs) for hs in heads]


def makespan(costs, heads_per_rank):
    """Largest per-rank total cost of an assignment."""
    return max(sum(float(costs[h]) for h in hs) for hs in heads_per_rank)


def seq_to_heads(x: torch.Tensor, heads_per_rank, group=None) -> torch.Tensor:
    """Uneven Ulysses reshard: [B, N/P, H, d] (this rank's token chunk, all heads) -> [B, |A_r|, N, d] (all tokens of
    the heads A_r = heads_per_rank[rank]).  Every head must appear in exactly one list."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B, n, H, d = x.shape
    send = torch.cat([x[:, :, hs].reshape(-1) for hs in heads_per_rank]).contiguous()
    splits_out = [B * n * len(hs) * d for hs in heads_per_rank]
    mine = heads_per_rank[rank]
    recv = torch.empty(world * B * n * len(mine) * d, dtype=x.dtype, device=x.device)
    _all_to_all_uneven(recv, send, [B * n * len(mine) * d] * world, splits_out, group)
    # recv: [P(src = token chunk), B, n, |A_r|, d] -> [B, |A_r|, N, d]
    return recv.view(world, B, n, len(mine), d).permute(1, 3, 0, 2, 4).reshape(B, len(mine), world * n, d).contiguous()


def heads_to_seq(y: torch.Tensor, heads_per_rank, H: int, group=None) -> torch.Tensor:
    """Inverse of seq_to_heads: [B, |A_r|, N, d] -> [B, N/P, H, d]."""
    world = dist.get_world_size(group)
    B, hr, N, d = y.shape
    n = N // world
    send = y.reshape(B, hr, world, n, d).permute(2, 0, 3, 1, 4).contiguous()  # [P(dest = token chunk), B, n, |A_r|, d]
    recv = torch.empty(sum(B * n * len(hs) * d for hs in heads_per_rank), dtype=y.dtype, device=y.device)
    _all_to_all_uneven(recv, send.reshape(-1), [B * n * len(hs) * d for hs in heads_per_rank],
                       [B * n * hr * d] * world, group)
    out = torch.empty(B, n, H, d, dtype=y.dtype, device=y.device)
    off = 0
    for hs in heads_per_rank:  # the part from rank q holds its heads A_q
        size = B * n * len(hs) * d
        out[:, :, hs] = recv[off:off + size].view(B, n, len(hs), d)
        off += size
    return out


def _all_to_all_uneven(recv, send, in_splits_recv, out_splits_send, group=None):
    if send.is_cuda and dist.get_backend(group) == "gloo":
        r = torch.empty_like(recv, device="cpu")
        dist.all_to_all_single(r, send.cpu(), output_split_sizes=in_splits_recv, input_split_sizes=out_splits_send,
                               group=group)
        recv.copy_(r)
    else:
        dist.all_to_all_single(recv, send, output_split_sizes=in_splits_recv, input_split_sizes=out_splits_send,
                               group=group)


# ------------------------------------------------------------------ query-cluster-granular split
# Heads that do not divide over the ranks (H < P, or H % P != 0) are cut into parts of their query clusters: every
# rank holding a part of head h receives all of h's tokens (K/V replicated), runs the same deterministic k-means and
# selection, and computes only its part's query clusters (svg2_sparse_attention_layout part_index / part_count; the
# parts are cut by the selected-pair cost per cluster, so they carry near-equal work).  Each output row is written by
# exactly one rank: straight into the owner's token-sharded output through peer memory (out_shards), or, without
# peer mappings, into a zero buffer that the reverse reshard merges by bitwise OR (exact: x | 0 = x).


def split_plan(H: int, world: int):
    """Per rank, its units (head, part_index, part_count): every head is cut into k = world / gcd(H, world) parts so
    the H*k units split evenly over the ranks (k = 1: the plain head split)."""
    k = world // math.gcd(H, world)
    units = [(h, p, k) for h in range(H) for p in range(k)]
    per = len(units) // world
    return [units[r * per:(r + 1) * per] for r in range(world)]


def unit_calls(units):
    """Group a rank's units into library calls (h0, h1, part_begin, part_end, part_count): per head the rank's
    contiguous parts [p0, p1) of k (all k parts = the whole head, (0, 1, 1)); consecutive heads with the same part
    range share one call."""
    by_head = {}
    for h, p, k in units:
        by_head.setdefault(h, []).append((p, k))
    calls = []
    for h in sorted(by_head):
        ps = sorted(p for p, _ in by_head[h])
        k = by_head[h][0][1]
        if ps != list(range(ps[0], ps[-1] + 1)):
            raise ValueError("a rank's parts of one head must be contiguous")
        spec = (0, 1, 1) if len(ps) == k else (ps[0], ps[-1] + 1, k)
        if calls and calls[-1][1] == h and calls[-1][2:] == spec:
            calls[-1] = (calls[-1][0], h + 1) + spec
        else:
            calls.append((h, h + 1) + spec)
    return calls


def heads_of(units):
    return sorted({h for h, _, _ in units})


def heads_to_seq_or(y: torch.Tensor, heads_per_rank, H: int, group=None) -> torch.Tensor:
    """Reverse reshard of a query-cluster split: [B, |A_r|, N, d] (this rank's rows of its heads, zeros elsewhere) ->
    [B, N/P, H, d]; heads held by several ranks are merged by bitwise OR of the bf16 patterns (each row has exactly one
    writer, so the merge is exact)."""
    world = dist.get_world_size(group)
    B, hr, N, d = y.shape
    n = N // world
    send = y.reshape(B, hr, world, n, d).permute(2, 0, 3, 1, 4).contiguous()  # [P(dest), B, n, |A_r|, d]
    recv = torch.empty(sum(B * n * len(hs) * d for hs in heads_per_rank), dtype=y.dtype, device=y.device)
    _all_to_all_uneven(recv, send.reshape(-1), [B * n * len(hs) * d for hs in heads_per_rank],
                       [B * n * hr * d] * world, group)
    out = torch.zeros(B, n, H, d, dtype=torch.int16, device=y.device)
    off = 0
    for hs in heads_per_rank:
        size = B * n * len(hs) * d
        out[:, :, hs] |= recv[off:off + size].view(torch.int16).view(B, n, len(hs), d)
        off += size
    return out.view(y.dtype)


class SplitSVG2:
    """Sequence-parallel in, sequence-parallel out, for any H and P: each rank runs its (head, part) units of the
    split plan with its own centroid caches (fixed plan, so the caches stay resident).  out_peers: None (reverse
    reshard with the OR merge) or the list of every rank's token-sharded output tensor [B, N/P, H, d] as mapped in
    this process (own tensor + peers' through CUDA IPC): rows are then stored straight into their owner's shard."""

    def __init__(self, H, Cq=100, Ck=500, top_p=0.9, iters_cold=5, iters_warm=2, group=None):
        self.group = group
        world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.plan = split_plan(H, world)
        self.heads = [heads_of(u) for u in self.plan]
        self.calls = unit_calls(self.plan[self.rank])
        self.H, self.Cq, self.Ck, self.top_p = H, Cq, Ck, top_p
        self.iters_cold, self.iters_warm = iters_cold, iters_warm
        self.cache = {}

    def __call__(self, q_seq, k_seq, v_seq, out_peers=None):
        from . import sparse_attention
        mine = self.heads[self.rank]
        Q, K, V = (seq_to_heads(t, self.heads, self.group) for t in (q_seq, k_seq, v_seq))  # [B, |A_r|, N, d]
        B, _, N, d = Q.shape
        y = None if out_peers is not None else torch.zeros_like(Q)
        for h0, h1, pb, pe, pc in self.calls:
            a, b = mine.index(h0), mine.index(h1 - 1) + 1
            key = (h0, h1, pb, pe, pc)
            warm = key in self.cache
            cq, ck = self.cache.get(key, (None, None))
            if out_peers is not None:  # rows straight into their owner's token shard (global head index)
                t0 = out_peers[0]
                shards = dict(shards=out_peers, shard_tokens=N // len(out_peers),
                              strides=(t0.stride(0), t0.stride(2), t0.stride(1)), head_offset=h0)
            else:  # rows into this rank's zero buffer y [B, |A_r|, N, d] (head offset a), merged by OR on the way back
                shards = dict(shards=[y], shard_tokens=N, strides=(y.stride(0), y.stride(1), y.stride(2)),
                              head_offset=a)
            _, _, ex = sparse_attention(Q[:, a:b], K[:, a:b], V[:, a:b], self.Cq, self.Ck,
                                        self.iters_warm if warm else self.iters_cold, self.top_p, cq, ck, warm=warm,
                                        part=(pb, pe, pc), out_shards=shards)
            self.cache[key] = (ex["q_centroids"], ex["k_centroids"])
        if out_peers is not None:
            return None
        return heads_to_seq_or(y, self.heads, self.H, self.group)


class HeadParallelSVG2:
    """Sequence-parallel in, sequence-parallel out; SVG2 on this rank's heads in between."""

    def __init__(self, Cq=100, Ck=500, top_p=0.9, iters_cold=5, iters_warm=2, group=None):
        from . import SVG2Attention
        self.attn = SVG2Attention(Cq, Ck, top_p, iters_cold, iters_warm)
        self.group = group

    def __call__(self, q_seq, k_seq, v_seq):
        if q_seq.shape[1] * dist.get_world_size(self.group) != k_seq.shape[1] * dist.get_world_size(self.group):
            raise ValueError("self-attention expects equal query / key sequence lengths")
        Q, K, V = (seq_to_head(t, self.group) for t in (q_seq, k_seq, v_seq))
        O = self.attn(Q, K, V)
        return head_to_seq(O, self.group)
