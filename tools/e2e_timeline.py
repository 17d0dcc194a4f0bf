"""Timeline of one warm host-buffer call (svg2_sparse_attention_host) under torch.profiler (measurement tool): when the
H2D and D2H copies and the attention kernels run, and where the GPU waits for data.
    python tools/e2e_timeline.py [workload]
"""
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2505_18875_b200 as svg2, svg2_synth
from torch.profiler import profile, ProfilerActivity
wl = svg2_synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "hunyuan720p"]
q, k, v = svg2_synth.generate(wl)
Qh, Kh, Vh = (torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).pin_memory() for a in (q, k, v))
O, pairs, ex = svg2.sparse_attention_host(Qh, Kh, Vh, wl.Cq, wl.Ck, wl.iters, wl.top_p)
qc, kc = ex["q_centroids"], ex["k_centroids"]
out = torch.empty_like(Qh).pin_memory()
for _ in range(2): svg2.sparse_attention_host(Qh, Kh, Vh, wl.Cq, wl.Ck, 2, wl.top_p, qc, kc, warm=True, out=out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    svg2.sparse_attention_host(Qh, Kh, Vh, wl.Cq, wl.Ck, 2, wl.top_p, qc, kc, warm=True, out=out)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in evs)
rows = []
for e in evs:
    n = e.name
    kind = "H2D" if "HtoD" in n else "D2H" if "DtoH" in n else ("ATT" if "varblock" in n else "K")
    rows.append((e.time_range.start - t0, e.time_range.end - t0, kind, n[:40]))
rows.sort()
# summarize: H2D intervals, D2H intervals, attention kernels
for kind in ("H2D", "D2H", "ATT"):
    iv = [(a, b) for a, b, k_, _ in rows if k_ == kind]
    busy = sum(b - a for a, b in iv)
    print(kind, "count", len(iv), "first start %.0f" % iv[0][0], "last end %.0f" % max(b for a, b in iv), "busy %.0f us" % busy)
    if kind != "ATT":
        print("   ", " ".join("%.0f-%.0f" % (a, b) for a, b in iv))
    else:
        print("   ", " ".join("%.0f-%.0f" % (a, b) for a, b in iv))
end = max(b for a, b, k_, _ in rows)
print("call span us %.0f" % end)
# GPU idle (no kernel running) intervals
ks = sorted((a, b) for a, b, k_, _ in rows if k_ in ("ATT", "K"))
idle, cur = 0.0, ks[0][1]
gaps = []
for a, b in ks[1:]:
    if a > cur:
        idle += a - cur
        if a - cur > 50: gaps.append((cur, a))
    cur = max(cur, b)
print("kernel-idle us %.0f, gaps > 50 us:" % idle, " ".join("%.0f-%.0f" % g for g in gaps[:20]))
