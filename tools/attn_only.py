"""Minimal attention-kernel repro for debugging (tiny config, synchronised)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2505_18875_b200 as svg2
import svg2_synth
wl = svg2_synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "tiny"]
q, k, v = svg2_synth.generate(wl, heads=[0])
Q, K, V = (torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda() for a in (q, k, v))
lq, sq, cq, pq, oq = svg2.kmeans(Q, wl.Cq, wl.iters, return_perm=True)
lk, sk, ck, pk, ok = svg2.kmeans(K, wl.Ck, wl.iters, return_perm=True)
_, _, Qp, _ = svg2.permute(lq, wl.Cq, Q)
_, _, Kp, Vp = svg2.permute(lk, wl.Ck, K, V)
top_p = float(sys.argv[2]) if len(sys.argv) > 2 else wl.top_p
mask, pairs = svg2.select_topp(cq, ck, sq, sk, top_p)
torch.cuda.synchronize()
print("sizes q", sq.cpu().numpy().ravel()[:20], "density", float(pairs.double().sum()) / (wl.N * wl.N), flush=True)
O = svg2.varblock_attention(Qp, Kp, Vp, oq, ok, mask, q_perm=pq)
torch.cuda.synchronize()
print("attention ok, finite:", bool(torch.isfinite(O.float()).all()))
