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
