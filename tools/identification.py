"""Identification quality of the selection on synthetic workloads (the paper's §3.1-3.2 analyses,
PAPER.md:11, 213-216, 239, 468-473; metric definitions).

On sampled query rows of a few heads, against the exact dense attention distribution P (torch fp32 on the GPU):
  * oracle top-p policy (token level): per row the smallest set of keys holding a fraction p of P -> recall-vs-density
    curve;
  * SVG2: the selection of the fused call (k-means on Q and K, centroid top-p), read back through
    its debug outputs;
  * position-block baselines: 128-query x 64-key blocks of consecutive tokens, block scores from
    mean-pooled Q and mean- or max-pooled K, the same top-p rule; also cut AFTER the semantic permutation.
Metrics per method at each p: density, recall (selected P mass, averaged over rows), critical-token miss rate and
waste against the oracle set at the same p.  Writes profiles/identification_r02.json.  Uses no oracle/ code; tests/test_identification.py reproduces its metric
and position-block functions with oracle/identification.py on the tiny config.
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


def oracle_sets(P, p):
    """Boolean [R, N]: per row the minimal descending-order prefix with mass >= p (ties by index)."""
    vals, idx = torch.sort(P, dim=1, descending=True, stable=True)
    cum = torch.cumsum(vals, dim=1)
    keep_sorted = (cum - vals) < p  # include the element that crosses p
    keep = torch.zeros_like(P, dtype=torch.bool)
    keep.scatter_(1, idx, keep_sorted)
    return keep


def metrics(sel, P, orc):
    sel_n = sel.sum().item()
    orc_n = orc.sum().item()
    both = (sel & orc).sum().item()
    return {"density": sel.float().mean().item(), "recall": (P * sel).sum(1).mean().item(),
            "miss_rate": 1.0 - both / orc_n if orc_n else 0.0, "waste": 1.0 - both / sel_n if sel_n else 0.0}


def block_topp(q_rep, k_rep, k_sizes, scale, p):
    """Eq.1/Eq.2-style block scores and the same top-p rule as the clusters: [Bq, Bk] bool."""
    S = (q_rep.double() @ k_rep.double().T) * scale
    S = S - S.max(dim=1, keepdim=True).values
    w = k_sizes.double()[None, :] * torch.exp(S)
    vals, idx = torch.sort(w, dim=1, descending=True, stable=True)
    cum = torch.cumsum(vals, dim=1)
    keep_sorted = (cum - vals) < p * w.sum(1, keepdim=True)
    keep = torch.zeros_like(w, dtype=torch.bool)
    keep.scatter_(1, idx, keep_sorted)
    return keep


def position_blocks(Qh, Kh, rows_pos, scale, p, bq=128, bk=64, pool="mean", perm_q=None, perm_k=None):
    """Selection of position-block sparse attention for the sampled rows (tokens in original order unless a
    permutation is given: then blocks are cut in permuted order).  Returns bool [R, N] over original key order."""
    N, d = Kh.shape
    qo = Qh if perm_q is None else Qh[perm_q]
    ko = Kh if perm_k is None else Kh[perm_k]
    nq, nk = math.ceil(N / bq), math.ceil(N / bk)
    qpad = torch.zeros(nq * bq, d, device=Qh.device)
    qpad[:N] = qo.float()
    q_rep = qpad.view(nq, bq, d).sum(1) / torch.tensor([min(bq, N - i * bq) for i in range(nq)], device=Qh.device)[:, None]
    k_sizes = torch.tensor([min(bk, N - j * bk) for j in range(nk)], device=Qh.device)
    kpad = torch.full((nk * bk, d), float("-inf") if pool == "max" else 0.0, device=Qh.device)
    kpad[:N] = ko.float()
    if pool == "max":
        k_rep = kpad.view(nk, bk, d).max(1).values
    else:
        k_rep = kpad.view(nk, bk, d).sum(1) / k_sizes[:, None]
    blk = block_topp(q_rep, k_rep, k_sizes, scale, p)  # [nq, nk]
    # position of each sampled row / each key in the (possibly permuted) order
    if perm_q is None:
        qpos = rows_pos
    else:
        inv_q = torch.empty_like(perm_q)
        inv_q[perm_q] = torch.arange(N, device=Qh.device)
        qpos = inv_q[rows_pos]
    if perm_k is None:
        kblock = torch.arange(N, device=Qh.device) // bk
    else:
        inv_k = torch.empty_like(perm_k)
        inv_k[perm_k] = torch.arange(N, device=Qh.device)
        kblock = inv_k // bk
    return blk[qpos // bq][:, kblock]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="wan480p")
    ap.add_argument("--heads", type=int, default=4)
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--out", default="profiles/identification_r02.json")
    args = ap.parse_args()
    wl = svg2_synth.WORKLOADS[args.workload]
    heads = list(range(args.heads))
    q, k, v = svg2_synth.generate(wl, heads=heads)
    Q, K, V = to_dev(q), to_dev(k), to_dev(v)
    N, d = wl.N, wl.d
    scale = 1.0 / math.sqrt(d)
    grid = [0.5, 0.7, 0.8, 0.9, 0.95]
    res = {"workload": wl.name, "heads": args.heads, "rows_per_head": args.rows, "p_grid": grid,
           "oracle_curve": [], "methods": {}}
    cq = ck = None
    rng = np.random.default_rng(7)
    acc = {}
    curve = {p: [0.0, 0.0] for p in grid}
    for p in grid:
        O, pairs, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 5, p, debug=True)
        for h in heads:
            rows = torch.from_numpy(np.sort(rng.choice(N, args.rows, replace=False))).cuda()
            Qh, Kh = Q[0, h], K[0, h]
            P = torch.softmax((Qh[rows].float() @ Kh.float().T) * scale, dim=1)
            orc = oracle_sets(P, p)
            curve[p][0] += orc.float().mean().item() / len(heads)
            curve[p][1] += (P * orc).sum(1).mean().item() / len(heads)
            lq = ex["q_labels"][0, h].long()
            lk = ex["k_labels"][0, h].long()
            mask = ex["mask"][0, h].bool()
            sel = {"svg2": mask[lq[rows]][:, lk]}
            pq, pk = ex["q_perm"][0, h].long(), ex["k_perm"][0, h].long()
            sel["block_mean"] = position_blocks(Qh, Kh, rows, scale, p, pool="mean")
            sel["block_max"] = position_blocks(Qh, Kh, rows, scale, p, pool="max")
            sel["block_mean_permuted"] = position_blocks(Qh, Kh, rows, scale, p, pool="mean", perm_q=pq, perm_k=pk)
            for name, s in sel.items():
                m = metrics(s, P, orc)
                a = acc.setdefault(name, {}).setdefault(p, {k_: 0.0 for k_ in m})
                for k_, v_ in m.items():
                    a[k_] += v_ / len(heads)
            del P, orc, sel
        torch.cuda.empty_cache()
        print(json.dumps({"p": p, **{n: acc[n][p] for n in acc}}), flush=True)
    res["oracle_curve"] = [{"p": p, "density": curve[p][0], "recall": curve[p][1]} for p in grid]
    res["methods"] = {n: [{"p": p, **acc[n][p]} for p in grid] for n in acc}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)
    print(json.dumps(res["oracle_curve"]))


if __name__ == "__main__":
    main()
