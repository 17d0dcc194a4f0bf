"""FP8 PV accuracy and speed (measurement tool): the fused call with and without SVG2_FP8_PV against the fp64 oracle
on sampled rows, and the attention time at the HunyuanVideo shape."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import oracle  # noqa: E402  (measurement of accuracy against the oracle: test infrastructure)
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402
from gpu_helpers import random_qkv, to_dev, to_f64  # noqa: E402


def err_vs_oracle(Q, K, V, Cq, Ck, p, fp8, rows):
    O, pairs, ex = svg2.sparse_attention(Q, K, V, Cq, Ck, 3, p, debug=True, fp8=fp8)
    torch.cuda.synchronize()
    d = Q.shape[-1]
    scale = float(np.float32(1.0 / math.sqrt(d)))
    out = []
    for h in range(Q.shape[1]):
        lq, lk, m = (ex[k][0, h].cpu().numpy() for k in ("q_labels", "k_labels", "mask"))
        ref = oracle.attention_rows(to_f64(Q)[0, h], to_f64(K)[0, h], to_f64(V)[0, h], scale, rows=rows, lq=lq,
                                    lk=lk, mask=m)
        got = to_f64(O)[0, h][rows]
        out.append(np.abs(got - ref))
    e = np.concatenate(out)
    return float(e.max()), float(e.mean())


q, k, v = random_qkv(1, 3, 4096, 4096, 128, seed=3)
Q, K, V = to_dev(q), to_dev(k), to_dev(v)
rows = np.arange(0, 4096, 3)
for fp8 in (False, True):
    print("random 3x4096", "fp8" if fp8 else "bf16", err_vs_oracle(Q, K, V, 30, 60, 0.9, fp8, rows), flush=True)
wl = svg2_synth.WORKLOADS["hunyuan720p"]
q, k, v = svg2_synth.generate(wl, heads=[0, 1])
Q, K, V = to_dev(q), to_dev(k), to_dev(v)
rows = np.sort(np.random.default_rng(0).choice(wl.N, 600, replace=False))
for fp8 in (False, True):
    print("hunyuan 2 heads", "fp8" if fp8 else "bf16", err_vs_oracle(Q, K, V, wl.Cq, wl.Ck, wl.top_p, fp8, rows),
          flush=True)
