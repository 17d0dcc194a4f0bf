"""BASELINE configs[3] analogue (single GPU): a denoising sweep with the centroid cache.

Inputs drift from step to step as in SURVEY §8(d) (svg2_synth drift_step: group directions rotate by 0.02 per step,
AR(1) noise with rho = 0.95).  The first `--dense` steps run dense attention (the paper's 30% warm-up);
the first sparse step is a cold k-means, every later step warm-starts from the previous step's centroids.  Each sparse
step is also re-run cold (same inputs) to compare k-means latency and density: the warm path should reach comparable
density with far fewer Lloyd iterations (the paper reports up to 76x lower k-means latency with its k-means++ cold
start).  Writes a JSON file (default profiles/denoise_sweep_r01.json).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402


def to_dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def timed_call(Q, K, V, wl, iters, cq=None, ck=None, init="strided"):
    # each configuration runs twice on the same inputs (the cache input cloned) and the second run is timed: a single
    # first call on freshly uploaded inputs measured up to 20% slow attention (one-shot artifact, tools/cluster_stats)
    warm = cq is not None
    for rep in range(2):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
        O, pairs, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, iters, wl.top_p,
                                             cq.clone() if warm else None, ck.clone() if warm else None, warm=warm,
                                             events=ev, init=init, seed=2025)
        torch.cuda.synchronize()
    return O, {
        "iters": iters, "warm": warm, "ms_call": ev[0].elapsed_time(ev[7]),
        "ms_kmeans": ev[0].elapsed_time(ev[2]), "ms_attention": ev[5].elapsed_time(ev[6]),
        "density": float(pairs.double().sum()) / (wl.B * wl.H * wl.N * wl.N)}, ex


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="hunyuan720p")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--dense", type=int, default=3)
    ap.add_argument("--cold-iters", type=int, default=30)
    ap.add_argument("--warm-iters", type=int, default=2)
    ap.add_argument("--cold-init", default="strided", choices=["strided", "kmeans++"])
    ap.add_argument("--out", default="profiles/denoise_sweep_r01.json")
    args = ap.parse_args()
    wl = svg2_synth.WORKLOADS[args.workload]
    res = {"workload": wl.name, "cold_iters": args.cold_iters, "warm_iters": args.warm_iters,
           "cold_init": args.cold_init, "steps": []}
    cq = ck = None
    for s in range(args.steps):
        t0 = time.time()
        q, k, v = svg2_synth.generate(wl, drift_step=s)
        Q, K, V = to_dev(q), to_dev(k), to_dev(v)
        del q, k, v
        rec = {"step": s, "gen_s": time.time() - t0}
        if s < args.dense:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            torch.nn.functional.scaled_dot_product_attention(Q, K, V)
            b.record()
            torch.cuda.synchronize()
            rec["dense_ms"] = a.elapsed_time(b)
        else:
            ref = torch.nn.functional.scaled_dot_product_attention(Q, K, V)
            if cq is None:
                O, cold, ex = timed_call(Q, K, V, wl, args.cold_iters, init=args.cold_init)
                rec["cold"] = cold
            else:
                O, warm, ex = timed_call(Q, K, V, wl, args.warm_iters, cq, ck)
                rec["warm"] = warm
                Oc, cold, _ = timed_call(Q, K, V, wl, args.cold_iters, init=args.cold_init)
                rec["cold"] = cold
                rec["warm_vs_cold_kmeans_speedup"] = cold["ms_kmeans"] / warm["ms_kmeans"]
                rec["rel_l2_warm_vs_dense"] = float((O.float() - ref.float()).norm() / ref.float().norm())
                rec["rel_l2_cold_vs_dense"] = float((Oc.float() - ref.float()).norm() / ref.float().norm())
            cq, ck = ex["q_centroids"].clone(), ex["k_centroids"].clone()
        res["steps"].append(rec)
        print(json.dumps(rec), flush=True)
        del Q, K, V
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
