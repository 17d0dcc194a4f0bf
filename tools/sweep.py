"""BASELINE configs[4]: top-p sweep 0.5-1.0 and cluster-count sweep at the Wan 2.1 480p shape (N = 32,760,
H = 40, d = 128): accuracy vs dense and speed vs density.  Writes one JSON file (default profiles/sweep_r01.json).

Per point: density, ms per fused call (warm, 2 Lloyd iterations), attention-kernel ms, effective / executed TFLOPS,
accuracy of the sparse output against dense attention of the same inputs (max-abs, mean-abs, relative L2, PSNR as
in SPEC.md:530-545 on attention outputs), and the tile-work multiplier = MMA area actually executed (Q tiles of 128
rows, key streams rounded up to 16) / algorithmic area, next to the static 128x128-block alternative (each selected
key cluster padded to 128 keys, the FlashInfer analogue of PAPER.md:330-331, 444).
"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402


def to_dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def tile_work(q_off, k_off, mask):
    """Executed vs algorithmic MMA area from the selection (per head, summed)."""
    q_off = q_off.cpu().numpy().astype(np.int64)
    k_off = k_off.cpu().numpy().astype(np.int64)
    mask = mask.cpu().numpy().astype(bool)
    B, H, Cq, Ck = mask.shape
    alg = exe = static = 0
    for b in range(B):
        for h in range(H):
            sq = np.diff(q_off[b, h])
            sk = np.diff(k_off[b, h])
            keys = mask[b, h] @ sk
            alg += int((sq * keys).sum())
            qt = np.ceil(sq / 128) * 128
            exe += int((qt * (np.ceil(keys / 16) * 16)).sum())
            static += int((qt * (mask[b, h] @ (np.ceil(sk / 128) * 128))).sum())
    return alg, exe, static


def accuracy(O, ref):
    diff = (O.float() - ref.float())
    mse = float((diff ** 2).mean())
    peak = float(ref.float().abs().max())
    return {"max_abs": float(diff.abs().max()), "mean_abs": float(diff.abs().mean()),
            "rel_l2": float(diff.norm() / ref.float().norm()),
            "psnr_db": 10 * math.log10(peak * peak / mse) if mse > 0 else float("inf")}


def run_point(Q, K, V, ref, wl, Cq, Ck, p, reps=5):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    O, pairs, ex = svg2.sparse_attention(Q, K, V, Cq, Ck, wl.iters, p)
    cq, ck = ex["q_centroids"], ex["k_centroids"]
    svg2.sparse_attention(Q, K, V, Cq, Ck, 2, p, cq, ck, warm=True)
    torch.cuda.synchronize()
    names = ["kmeans_k_fork", "kmeans_q_join", "permute_fp8", "select_topp", "worklist", "attention", "end"]
    calls, attns, per_stage = [], [], {n: [] for n in names}
    for _ in range(reps):  # medians over the repetitions (a host stall in one call does not move the result)
        O, pairs, ex = svg2.sparse_attention(Q, K, V, Cq, Ck, 2, p, cq, ck, warm=True, events=ev, debug=True)
        torch.cuda.synchronize()
        calls.append(ev[0].elapsed_time(ev[7]))
        attns.append(ev[5].elapsed_time(ev[6]))
        for i, n in enumerate(names):
            per_stage[n].append(ev[i].elapsed_time(ev[i + 1]))
    med = lambda a: sorted(a)[len(a) // 2]  # noqa: E731
    t_call, t_attn = med(calls), med(attns)
    stages = {n: med(v) for n, v in per_stage.items()}
    B, H, N, d = Q.shape
    dens = float(pairs.double().sum()) / (B * H * N * N)
    alg, exe, static = tile_work(ex["q_offsets"], ex["k_offsets"], ex["mask"])
    return {"Cq": Cq, "Ck": Ck, "top_p": p, "density": dens, "ms_call": t_call, "ms_attention": t_attn,
            "eff_tflops": 4.0 * N * N * d * B * H / (t_call * 1e-3) / 1e12,
            "attn_executed_tflops": 4.0 * d * float(pairs.double().sum()) / (t_attn * 1e-3) / 1e12,
            "tile_work_multiplier": exe / alg, "static128_multiplier": static / alg,
            "static_over_packed": static / exe, "stages_ms": stages, **accuracy(O, ref)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="wan480p")
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--out", default="profiles/sweep_r02.json")
    ap.add_argument("--points", default=None, help="only these Cq:Ck pairs at p = 0.9, e.g. 200:4000,400:500")
    args = ap.parse_args()
    wl = svg2_synth.WORKLOADS[args.workload]
    q, k, v = svg2_synth.generate(wl, heads=range(args.heads))
    Q, K, V = to_dev(q), to_dev(k), to_dev(v)
    del q, k, v
    from torch.nn.attention import SDPBackend, sdpa_kernel
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION]):
        ref = torch.nn.functional.scaled_dot_product_attention(Q, K, V)
        times = []
        for _ in range(5):  # median of 5 timed calls
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            ref = torch.nn.functional.scaled_dot_product_attention(Q, K, V)
            e.record()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e))
        t_dense = sorted(times)[2]
    res = {"workload": wl.name, "heads": args.heads, "N": wl.N, "dense_ms_sdpa": t_dense, "topp_sweep": [],
           "cluster_sweep": []}
    if args.points:
        for pt in args.points.split(","):
            Cq, Ck = (int(x) for x in pt.split(":"))
            r = run_point(Q, K, V, ref, wl, Cq, Ck, 0.9)
            r["speedup_vs_dense"] = t_dense / r["ms_call"]
            print(json.dumps(r), flush=True)
        return
    for p in [0.5, 0.6, 0.7, 0.8, 0.9, 0.95, 1.0]:
        r = run_point(Q, K, V, ref, wl, 100, 500, p)
        r["speedup_vs_dense"] = t_dense / r["ms_call"]
        res["topp_sweep"].append(r)
        print(json.dumps(r), flush=True)
    for Cq, Ck in [(100, 250), (100, 1000), (50, 500), (200, 500), (400, 500), (100, 500), (50, 1000), (200, 1000),
                   (400, 1000), (200, 250), (200, 2000), (200, 4000)]:
        r = run_point(Q, K, V, ref, wl, Cq, Ck, 0.9)
        r["speedup_vs_dense"] = t_dense / r["ms_call"]
        res["cluster_sweep"].append(r)
        print(json.dumps(r), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
