"""Head-parallel SVG2 across the GPUs of one node.

Every SVG2 step is per (b, h) with no cross-head data, so heads shard with no collective inside the method.  The
only exchange is the Ulysses-style reshard of a sequence-parallel DiT: activations arrive token-sharded
[B, N/P, H, d] on each rank, an all-to-all (NCCL over NVLink/NVSwitch via torch.distributed) turns them into
head-sharded [B, H/P, N, d] for attention, and the output goes back the same way.  Rank r owns heads
[r H/P, (r+1) H/P) for the whole run, so its centroid caches stay resident.

torch.distributed is plumbing here: the attention itself runs in libsvg2.so.
"""
from __future__ import annotations

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
