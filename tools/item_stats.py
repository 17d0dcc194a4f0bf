"""Work-list statistics of the attention kernel for one head of a workload (measurement tool).

Prints how many work items carry one vs two 128-row Q tiles and the fraction of tile-slots wasted on padding rows
and on missing second tiles -- the latter run a full-length softmax/MMA chain for half the rows.
"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2505_18875_b200 as svg2
import svg2_synth

wl = svg2_synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "hunyuan720p"]
heads = [0, 1, 2, 3]
q, k, v = svg2_synth.generate(wl, heads=heads)
Q, K, V = (torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda() for a in (q, k, v))
O, pairs, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, wl.iters, wl.top_p, debug=True)
qo = ex["q_offsets"].cpu().numpy().reshape(len(heads), -1)
ko = ex["k_offsets"].cpu().numpy().reshape(len(heads), -1)
mask = ex["mask"].cpu().numpy().reshape(len(heads), wl.Cq, wl.Ck)
single = pair = 0
slot_rows = used_rows = 0.0
periods_pair = periods_single = 0.0
for h in range(len(heads)):
    qs = np.diff(qo[h])
    ks = np.diff(ko[h])
    for i in range(wl.Cq):
        keys = int((ks * mask[h, i]).sum())
        tiles = int(np.ceil(qs[i] / 128))
        T = np.ceil(keys / 128)
        n_items = (tiles + 1) // 2
        pair += tiles // 2
        single += tiles % 2
        periods_pair += (tiles // 2) * T
        periods_single += (tiles % 2) * T
        slot_rows += n_items * 256 * T
        used_rows += qs[i] * T
print(f"{wl.name}: items with two Q tiles {pair}, with one {single} ({single / (pair + single):.1%}); "
      f"row-slot efficiency {used_rows / slot_rows:.1%} (pair items x 256 rows x key tiles)")
scale = wl.H * wl.B / len(heads)
print(f"key-tile periods per call (all heads): pair items {periods_pair * scale:.0f}, single-tile items "
      f"{periods_single * scale:.0f} ({periods_single / (periods_pair + periods_single):.1%}); at 3200 cycles per "
      f"period, 148 SMs, 1.65 GHz: {(periods_pair + periods_single) * scale * 3200 / 148 / 1.65e6:.1f} ms")
