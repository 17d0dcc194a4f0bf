"""Why does attention time depend on how well k-means converged?  Structure statistics of the attention work list for
one denoising step, cold (k-means++, 5 Lloyd iterations) vs warm (2 iterations from the previous step's centroids),
at the same inputs (measurement tool).

Per configuration: density, attention ms, selected key clusters per query-cluster row, runs per key stream (adjacent
selected clusters merge), 8-row padding, one-tile items, executed / algorithmic MMA area, and the spread of query-
and key-cluster sizes.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402


def to_dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def stats(ex, wl, heads):
    q_off = ex["q_offsets"].cpu().numpy().astype(np.int64).reshape(-1, wl.Cq + 1)
    k_off = ex["k_offsets"].cpu().numpy().astype(np.int64).reshape(-1, wl.Ck + 1)
    msk = ex["mask"].cpu().numpy().astype(bool).reshape(-1, wl.Cq, wl.Ck)
    sel, runs, pad, single, items, alg, exe = [], [], 0, 0, 0, 0, 0
    for hh in range(len(heads)):
        sq, sk = np.diff(q_off[hh]), np.diff(k_off[hh])
        for i in range(wl.Cq):
            if sq[i] == 0:
                continue
            m = msk[hh, i] & (sk > 0)
            sel.append(int(m.sum()))
            starts = m & ~np.concatenate(([False], m[:-1]))
            run_id = np.cumsum(starts) * m
            run_len = np.bincount(run_id, weights=sk * m)[1:]
            runs.append(len(run_len))
            pad += int((np.ceil(run_len / 8) * 8 - run_len).sum())
            tiles = int(np.ceil(sq[i] / 128))
            items += (tiles + 1) // 2
            single += tiles % 2
            keys = int((sk * m).sum())
            alg += int(sq[i]) * keys
            exe += int(np.ceil(sq[i] / 128) * 128) * int(np.ceil(np.ceil(run_len / 8).sum() * 8 / 16) * 16)
    sizes_q = np.diff(q_off, axis=1).ravel()
    sizes_k = np.diff(k_off, axis=1).ravel()
    return {"sel_clusters_per_row": float(np.mean(sel)), "runs_per_stream": float(np.mean(runs)),
            "pad_rows_frac": pad / max(1, sum(runs)) / 8, "one_tile_items_frac": single / max(1, items),
            "tile_work": exe / alg, "q_size_cv": float(sizes_q.std() / sizes_q.mean()),
            "k_size_cv": float(sizes_k.std() / sizes_k.mean()), "k_empty": int((sizes_k == 0).sum()),
            "q_empty": int((sizes_q == 0).sum())}


def timed(Q, K, V, wl, iters, cq=None, ck=None, init="strided"):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    O, pairs, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, iters, wl.top_p, cq, ck, warm=cq is not None,
                                         events=ev, debug=True, init=init, seed=2025)
    torch.cuda.synchronize()
    return ex, {"ms_attention": ev[5].elapsed_time(ev[6]), "density": float(pairs.double().sum()) /
                (wl.B * Q.shape[1] * wl.N * wl.N)}


def main():
    wl = svg2_synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "hunyuan720p"]
    heads = list(range(int(sys.argv[2]) if len(sys.argv) > 2 else 8))
    q, k, v = svg2_synth.generate(wl, heads=heads, drift_step=1)
    Q, K, V = to_dev(q), to_dev(k), to_dev(v)
    ex1, _ = timed(Q, K, V, wl, 5, init="kmeans++")
    cq, ck = ex1["q_centroids"].clone(), ex1["k_centroids"].clone()
    q, k, v = svg2_synth.generate(wl, heads=heads, drift_step=2)
    Q, K, V = to_dev(q), to_dev(k), to_dev(v)
    out = {}
    for name, kw in (("warm2", dict(iters=2, cq=cq.clone(), ck=ck.clone())), ("cold_pp5", dict(iters=5, init="kmeans++")),
                     ("cold_strided5", dict(iters=5)), ("warm8", dict(iters=8, cq=cq.clone(), ck=ck.clone()))):
        timed(Q, K, V, wl, **kw)  # warm-up of the same configuration
        ex, t = timed(Q, K, V, wl, **kw)
        t.update(stats(ex, wl, heads))
        out[name] = t
        print(name, json.dumps(t), flush=True)


if __name__ == "__main__":
    main()
