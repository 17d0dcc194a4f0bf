"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every entry point of libsvg2.so on
the tiny config and on a reduced-N HunyuanVideo shape (N = 6000, 2 heads, d = 128, Cq/Ck = 100/500), cold (strided and
k-means++) and warm, bf16 and FP8 PV, the standalone stages, the host-buffer pipeline, the objective output, and the
layout entry (strided inputs, token-sharded outputs, query-cluster parts, p = 1).
    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import dataclasses
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402


def dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def run(wl, fp8):
    q, k, v = svg2_synth.generate(wl)
    Q, K, V = dev(q), dev(k), dev(v)
    O, pairs, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 3, wl.top_p, debug=True)
    O2, _, _ = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 2, wl.top_p, ex["q_centroids"], ex["k_centroids"],
                                     warm=True, fp8=fp8)
    svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 1, wl.top_p, init="kmeans++", seed=3)
    lq, sq, cq, pq, oq, obj = svg2.kmeans(Q, wl.Cq, 2, return_perm=True, return_objective=True)
    lk, sk, ck, pk, ok = svg2.kmeans(K, wl.Ck, 2, return_perm=True)
    _, _, Qp, _ = svg2.permute(lq, wl.Cq, Q)
    _, _, Kp, Vp = svg2.permute(lk, wl.Ck, K, V)
    mask, _ = svg2.select_topp(cq, ck, sq, sk, wl.top_p)
    Op, lse = svg2.varblock_attention(Qp, Kp, Vp, oq, ok, mask, return_lse=True)
    svg2.unpermute(Op, pq)
    Qh, Kh, Vh = (t.cpu().pin_memory() for t in (Q, K, V))
    svg2.sparse_attention_host(Qh, Kh, Vh, wl.Cq, wl.Ck, 2, wl.top_p)
    # svg2_sparse_attention_layout: token-major strided inputs, output rows into 2 token shards, query-cluster parts,
    # and the p = 1 dense stream
    Qt, Kt, Vt = (t.permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3) for t in (Q, K, V))
    B, H, N, d = Q.shape
    n = (N + 1) // 2
    shards = [torch.zeros(B, n, H, d, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    t0 = shards[0]
    for part in ((0, 2), (1, 2)):
        svg2.sparse_attention(Qt, Kt, Vt, wl.Cq, wl.Ck, 2, wl.top_p, part=part,
                              out_shards=dict(shards=shards, shard_tokens=n,
                                              strides=(t0.stride(0), t0.stride(2), t0.stride(1)), head_offset=0))
    svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 2, 1.0)
    torch.cuda.synchronize()
    print(f"{wl.name}: ok, density {float(pairs.double().mean()) / (wl.N * wl.N):.3f}", flush=True)


if __name__ == "__main__":
    run(svg2_synth.WORKLOADS["tiny"], fp8=False)
    hy = svg2_synth.WORKLOADS["hunyuan720p"]
    run(dataclasses.replace(hy, name="hunyuan720p_reduced", H=2, grid=(3, 40, 50)), fp8=True)
