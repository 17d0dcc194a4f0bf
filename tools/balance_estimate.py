"""Head-parallel load balance, estimated on one GPU (measurement tool).

Each head of the workload is run alone (warm start, as in a denoising step) and timed; the makespan of P ranks is
then max over ranks of the summed per-head times, for the fixed contiguous split (dist.head_range) and for the
balanced assignment (dist.balanced_assignment) built from (a) the measured times and (b) the per-head selected
pairs, which a real run has after its first sparse step.  Writes profiles/balance_r01.json.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402
from paper_2505_18875_b200.dist import balanced_assignment, head_range, makespan  # noqa: E402


def main():
    wl = svg2_synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "hunyuan720p"]
    q, k, v = svg2_synth.generate(wl)
    to = lambda a: torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda()  # noqa: E731
    Q, K, V = to(q), to(k), to(v)
    del q, k, v
    times, pairs = [], []
    for h in range(wl.H):
        Qh, Kh, Vh = (t[:, h:h + 1].contiguous() for t in (Q, K, V))
        _, _, ex = svg2.sparse_attention(Qh, Kh, Vh, wl.Cq, wl.Ck, wl.iters, wl.top_p)
        cq, ck = ex["q_centroids"], ex["k_centroids"]
        for _ in range(2):
            svg2.sparse_attention(Qh, Kh, Vh, wl.Cq, wl.Ck, 2, wl.top_p, cq.clone(), ck.clone(), warm=True)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            _, pr, _ = svg2.sparse_attention(Qh, Kh, Vh, wl.Cq, wl.Ck, 2, wl.top_p, cq.clone(), ck.clone(), warm=True)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) / 5)
        pairs.append(float(pr.sum()))
        del Qh, Kh, Vh
    res = {"workload": wl.name, "per_head_ms": times, "per_head_pairs": pairs,
           "corr_time_pairs": float(np.corrcoef(times, pairs)[0, 1]), "P": {}}
    for P in (2, 4, 8):
        fixed = [list(range(*head_range(wl.H, r, P))) for r in range(P)]
        by_time = balanced_assignment(times, P)
        by_pairs = balanced_assignment(pairs, P)
        mean = sum(times) / P
        res["P"][str(P)] = {"fixed_ms": makespan(times, fixed), "balanced_by_time_ms": makespan(times, by_time),
                            "balanced_by_pairs_ms": makespan(times, by_pairs), "mean_ms": mean,
                            "fixed_imbalance": makespan(times, fixed) / mean,
                            "balanced_imbalance": makespan(times, by_pairs) / mean, "assignment": by_pairs}
        print(P, json.dumps({k_: v_ for k_, v_ in res["P"][str(P)].items() if k_ != "assignment"}), flush=True)
    print("corr(time, pairs) =", res["corr_time_pairs"])
    os.makedirs("profiles", exist_ok=True)
    json.dump(res, open("profiles/balance_r01.json", "w"), indent=1)


if __name__ == "__main__":
    main()
