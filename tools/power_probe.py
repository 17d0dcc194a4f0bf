"""Board power and SM clock while (a) the fused SVG2 call and (b) dense cuDNN attention run back to back for a few
seconds each on the HunyuanVideo shape (measurement tool).  Tells whether the kernels are power-capped."""
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402


def sample(fn, seconds=4.0):
    lines = []
    proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,power.limit,temperature.gpu",
                             "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    th = threading.Thread(target=lambda: [lines.append(x) for x in proc.stdout], daemon=True)
    th.start()
    t0, n = time.time(), 0
    while time.time() - t0 < seconds:
        fn()
        n += 1
    torch.cuda.synchronize()
    dt = time.time() - t0
    proc.terminate()
    vals = np.array([[float(v) for v in ln.split(",")] for ln in lines[5:] if ln.count(",") == 3])
    med = np.median(vals, axis=0) if len(vals) else [0, 0, 0, 0]
    return {"calls": n, "ms_per_call": 1e3 * dt / n, "sm_mhz": med[0], "power_w": med[1], "limit_w": med[2],
            "temp_c": med[3]}


wl = svg2_synth.WORKLOADS["hunyuan720p"]
q, k, v = svg2_synth.generate(wl)
Q, K, V = (torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda() for a in (q, k, v))
O, pairs, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 30, wl.top_p)
cq, ck = ex["q_centroids"].clone(), ex["k_centroids"].clone()
torch.cuda.synchronize()
print("svg2", sample(lambda: svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 2, wl.top_p, cq, ck, warm=True)), flush=True)
with torch.nn.attention.sdpa_kernel(torch.nn.attention.SDPBackend.CUDNN_ATTENTION):
    print("cudnn", sample(lambda: torch.nn.functional.scaled_dot_product_attention(Q, K, V)), flush=True)
print("svg2", sample(lambda: svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 2, wl.top_p, cq, ck, warm=True)), flush=True)
