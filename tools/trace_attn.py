"""Cycle trace of the attention kernel (measurement build, -DSVG2_TRACE): the first work item of CTA 0 of a warm
HunyuanVideo call, per key tile: producer K/V issue, MMA S/PV issue per Q tile, softmax events per Q tile.

    python tools/trace_attn.py [workload] [heads]     (builds build/libsvg2_trace.so first if missing)
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.environ.get("SVG2_TRACE_LIB", os.path.join(ROOT, "build", "libsvg2_trace.so"))
os.environ["SVG2_LIBRARY"] = LIB
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402

EV = ["prodK", "prodV", "S_a", "S_b", "PV_a", "PV_b", "sfull_a", "sfull_b", "ld_a", "ld_b", "exp_a", "exp_b",
      "pfull_a", "pfull_b", "max_a", "max_b", "P_a0", "P_a1", "P_a2", "P_a3", "E_a0", "E_a1", "E_a2", "E_a3"]
wl = svg2_synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "hunyuan720p"]
nh = int(sys.argv[2]) if len(sys.argv) > 2 else 2
top_p = float(sys.argv[3]) if len(sys.argv) > 3 else wl.top_p
q, k, v = svg2_synth.generate(wl, heads=range(nh))
Q, K, V = (torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda() for a in (q, k, v))
O, pairs, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, wl.iters, top_p)
for _ in range(2):
    svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 2, top_p, ex["q_centroids"], ex["k_centroids"], warm=True)
torch.cuda.synchronize()
lib = svg2.load_library()
buf = (ctypes.c_longlong * (24 * 48))()
assert lib.svg2_trace_dump(buf) == 0
tr = np.array(buf, dtype=np.int64).reshape(24, 48)
t0 = tr[0, 0]
print("cycles relative to the first K issue; per key tile t (80 keys)")
print("t   " + " ".join(f"{e:>8}" for e in EV))
for t in range(48):
    row = tr[:, t]
    if not row.any():
        break
    print(f"{t:<3} " + " ".join(f"{(x - t0) if x else -1:>8}" for x in row))
d = np.diff(tr[6, 1:40])
print("softmax a period (median cycles per tile):", float(np.median(d[d > 0])) if (d > 0).any() else None)
d = np.diff(tr[2, 1:40])
print("S_a issue period:", float(np.median(d[d > 0])) if (d > 0).any() else None)

P = tr[16:20, 1:40].astype(np.float64)
E = tr[20:24, 1:40].astype(np.float64)
ok = (P > 0).all(0) & (E > 0).all(0)
print("tile a, per tile: spread of P-stored times over the 4 warps (median, p90):",
      float(np.median(P[:, ok].max(0) - P[:, ok].min(0))), float(np.quantile(P[:, ok].max(0) - P[:, ok].min(0), 0.9)))
print("exp phase length per warp (median):", [float(np.median((P - E)[w, ok])) for w in range(4)])
pv = tr[4, 1:40].astype(np.float64)
okp = ok & (pv > 0)
print("PV_a issue after the last warp's P (median cycles):", float(np.median(pv[okp] - P[:, okp].max(0))))
