"""Locate wrong output rows of the p = 1 case (dense attention through the sparse path) against torch fp32."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2505_18875_b200 as svg2
from gpu_helpers import random_qkv, to_dev
B, H, N, d = 1, 2, 3000, 128
q, k, v = random_qkv(B, H, N, N, d, seed=11)
Q, K, V = to_dev(q), to_dev(k), to_dev(v)
O, pairs, ex = svg2.sparse_attention(Q, K, V, 8, 16, 2, 1.0, debug=True)
ref = torch.softmax((Q.float() @ K.float().transpose(-1, -2)) * svg2.default_scale(d), -1) @ V.float()
err = (O.float() - ref).abs().amax(-1)  # [B,H,N]
for h in range(H):
    bad = torch.nonzero(err[0, h] > 0.02).flatten().cpu().numpy()
    perm = ex["q_perm"][0, h].cpu().numpy()
    inv = np.empty_like(perm); inv[perm] = np.arange(N)
    off = ex["q_offsets"][0, h].cpu().numpy()
    pos = np.sort(inv[bad])
    print(f"head {h}: {len(bad)} bad rows; q_offsets {off.tolist()}")
    print("  permuted positions:", pos[:60].tolist(), "..." if len(pos) > 60 else "")
    if len(pos):
        cl = np.searchsorted(off, pos, side="right") - 1
        print("  clusters:", np.unique(cl).tolist(), " rel pos in cluster:", sorted(set((pos - off[cl]).tolist()))[:40])
# same with top_p < 1 but all clusters selected: single query cluster
