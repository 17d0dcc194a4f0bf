"""Per-rank work of the head-parallel run on one GPU (measurement tool): the fused warm call on H/P heads of a
workload (what one rank computes at P GPUs, without the all-to-all), stage by stage, plus the ncu-free kernel list
from the library's stage events.  Usage: python tools/rank_slice.py [workload] [P ...]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402

wl = svg2_synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "hunyuan720p"]
Ps = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
res = {}
for P in Ps:
    hp = wl.H // P
    q, k, v = svg2_synth.generate(wl, heads=range(hp))
    Q, K, V = (torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda() for a in (q, k, v))
    _, _, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, wl.iters, wl.top_p)
    cq, ck = ex["q_centroids"], ex["k_centroids"]
    for _ in range(3):
        svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 2, wl.top_p, cq, ck, warm=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    n = 10
    for _ in range(n):
        svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 2, wl.top_p, cq, ck, warm=True)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / n
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 2, wl.top_p, cq, ck, warm=True, events=ev)
    torch.cuda.synchronize()
    names = ["kmeans_q", "kmeans_k", "permute", "select_topp", "worklist", "attention"]
    st = {nm: round(ev[i].elapsed_time(ev[i + 1]), 3) for i, nm in enumerate(names)}
    res[P] = {"heads": hp, "ms_per_call": round(t, 3), "ms_per_head": round(t / hp, 3), "stages_ms": st}
    print(json.dumps({"P": P, **res[P]}), flush=True)
    del Q, K, V, q, k, v
    torch.cuda.empty_cache()
