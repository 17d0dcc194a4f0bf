"""Per-kernel device times of one warm fused call under torch.profiler (measurement tool; averages of 3 calls).
    python tools/kernel_times.py [workload] [Cq] [Ck]
"""
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2505_18875_b200 as svg2, svg2_synth
from torch.profiler import profile, ProfilerActivity
wl = svg2_synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "hunyuan720p"]
Cq = int(sys.argv[2]) if len(sys.argv) > 2 else wl.Cq
Ck = int(sys.argv[3]) if len(sys.argv) > 3 else wl.Ck
q, k, v = svg2_synth.generate(wl)
Q, K, V = (torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda() for a in (q, k, v))
O, pairs, ex = svg2.sparse_attention(Q, K, V, Cq, Ck, wl.iters, wl.top_p)
qc, kc = ex["q_centroids"], ex["k_centroids"]
for _ in range(2): svg2.sparse_attention(Q, K, V, Cq, Ck, 2, wl.top_p, qc, kc, warm=True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3): svg2.sparse_attention(Q, K, V, Cq, Ck, 2, wl.top_p, qc, kc, warm=True)
    torch.cuda.synchronize()
ev = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        ev.setdefault(e.name[:50], []).append(e.device_time_total)
for k_, v_ in sorted(ev.items(), key=lambda x: -sum(x[1])):
    print(round(sum(v_) / 3, 1), len(v_) // 3, k_)
