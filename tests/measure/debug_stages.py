"""Stage-by-stage GPU debug run (not a test): each ABI call synchronised and checked against the oracle."""
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2505_18875_b200 as svg2  # noqa: E402
import svg2_synth  # noqa: E402


def to_dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def stage(name, fn):
    t = time.time()
    out = fn()
    torch.cuda.synchronize()
    print(f"[ok] {name} {1e3 * (time.time() - t):.1f} ms", flush=True)
    return out


def main(name="tiny", heads=None):
    wl = svg2_synth.WORKLOADS[name]
    q, k, v = svg2_synth.generate(wl, heads=heads)
    Q, K, V = to_dev(q), to_dev(k), to_dev(v)
    d = wl.d
    lq, sq, cq, pq, oq = stage("kmeans Q", lambda: svg2.kmeans(Q, wl.Cq, wl.iters, return_perm=True))
    lk, sk, ck, pk, ok = stage("kmeans K", lambda: svg2.kmeans(K, wl.Ck, wl.iters, return_perm=True))
    _, _, Qp, _ = stage("permute Q", lambda: svg2.permute(lq, wl.Cq, Q))
    _, _, Kp, Vp = stage("permute K,V", lambda: svg2.permute(lk, wl.Ck, K, V))
    mask, pairs = stage("select", lambda: svg2.select_topp(cq, ck, sq, sk, wl.top_p))
    print("density", (pairs.double() / (wl.N * wl.N)).cpu().numpy().ravel()[:4])
    O = stage("varblock attention", lambda: svg2.varblock_attention(Qp, Kp, Vp, oq, ok, mask, q_perm=pq))
    Q64, K64, V64 = f64(Q)[0, 0], f64(K)[0, 0], f64(V)[0, 0]
    rows = svg2_synth.sample_rows(wl.N, 512, 0)
    ref = oracle.attention_rows(Q64, K64, V64, float(np.float32(1 / math.sqrt(d))), rows=rows,
                                lq=lq.cpu().numpy()[0, 0], lk=lk.cpu().numpy()[0, 0], mask=mask.cpu().numpy()[0, 0])
    got = f64(O)[0, 0][rows]
    err = np.abs(got - ref)
    print(f"attention vs oracle: max {err.max():.3e} mean {err.mean():.3e}")
    if err.max() > 2e-2:
        bad = np.argsort(-err.max(1))[:5]
        for b in bad:
            print("row", rows[b], "err", err[b].max(), "got", got[b][:4], "ref", ref[b][:4])
    Of, pf, _ = stage("fused", lambda: svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, wl.iters, wl.top_p))
    print("fused == staged:", torch.equal(Of, O))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "tiny", heads=[0] if len(sys.argv) > 1 else None)
