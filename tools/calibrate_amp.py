"""Calibrate the svg2-synth group amplitude `a` so the fused warm call's density at top-p 0.9, (Cq, Ck) = (100, 500)
hits a target (HunyuanVideo 0.25 +- 0.02, cf. 25.45% at PAPER.md:416).  For each a: generate all heads,
cold 5-iteration call, then the warm 2-iteration call bench.py times; print the density (selected pairs / N^2).
    python tools/calibrate_amp.py --workload hunyuan720p --amps 8.0 8.02 8.05 8.1
"""
import argparse
import dataclasses
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="hunyuan720p")
    ap.add_argument("--amps", type=float, nargs="+", required=True)
    args = ap.parse_args()
    wl0 = svg2_synth.WORKLOADS[args.workload]
    for a in args.amps:
        wl = dataclasses.replace(wl0, amp=a)
        q, k, v = svg2_synth.generate(wl)
        Q, K, V = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda() for x in (q, k, v))
        del q, k, v
        _, _, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, wl.iters, wl.top_p)
        _, pairs, _ = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 2, wl.top_p, ex["q_centroids"], ex["k_centroids"],
                                            warm=True)
        dens = (pairs.double() / (wl.N * wl.N)).cpu().numpy()
        print(json.dumps({"workload": wl.name, "amp": a, "density": float(dens.mean()),
                          "density_min": float(dens.min()), "density_max": float(dens.max())}), flush=True)
        del Q, K, V
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
