"""Per-CTA start / exit times and item counts of the last attention launch (measurement build -DSVG2_CTA_TIMES):
how long the persistent CTAs wait for the last one to finish (the launch tail).

    python tools/cta_times.py [workload]     (SVG2_CTA_LIB = the measurement library, default build/libsvg2_ctatimes.so)
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SVG2_LIBRARY"] = os.environ.get("SVG2_CTA_LIB", os.path.join(ROOT, "build", "libsvg2_ctatimes.so"))
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402

wl = svg2_synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "hunyuan720p"]
q, k, v = svg2_synth.generate(wl)
Q, K, V = (torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda() for a in (q, k, v))
O, pairs, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, wl.iters, wl.top_p)
for _ in range(2):
    svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 2, wl.top_p, ex["q_centroids"], ex["k_centroids"], warm=True)
torch.cuda.synchronize()
lib = svg2.load_library()
buf = (ctypes.c_ulonglong * (1024 * 3))()
assert lib.svg2_cta_times_dump(buf) == 0
t = np.array(buf, dtype=np.float64).reshape(1024, 3)
t = t[t[:, 1] > 0]
start, end, items = t[:, 0], t[:, 1], t[:, 2]
t0 = start.min()
e = np.sort(end - t0) / 1e6
print(f"{len(t)} CTAs, items per CTA {items.min():.0f}-{items.max():.0f} (mean {items.mean():.1f})")
print(f"launch {e[-1]:.3f} ms; CTA exits: first {e[0]:.3f}, p10 {np.quantile(e, 0.1):.3f}, median {np.median(e):.3f}, "
      f"p90 {np.quantile(e, 0.9):.3f} ms")
print(f"idle SM-time after each CTA's exit: {np.mean(e[-1] - e):.3f} ms per SM "
      f"({np.mean(e[-1] - e) / e[-1] * 100:.1f}% of the launch)")
