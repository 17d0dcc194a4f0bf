"""Helpers for the -m gpu parity tests: seeded inputs as torch bf16 on cuda:0 plus their exact fp64 copies for
the oracle, and the tie-band classifiers of DESIGN.md R16 / R17."""
import numpy as np
import torch

import svg2_synth


def to_dev(bits: np.ndarray) -> torch.Tensor:
    """uint16 bf16 bit patterns -> bf16 CUDA tensor (bit-exact)."""
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def to_f64(t: torch.Tensor) -> np.ndarray:
    """bf16 CUDA tensor -> exact float64 numpy."""
    return t.float().cpu().numpy().astype(np.float64)


def random_qkv(B, H, Nq, Nk, d, seed, amp=3.0, groups=8):
    """Clustered random inputs (not the synth recipe): useful for ragged / odd shapes."""
    rng = np.random.default_rng(seed)
    out = []
    for N in (Nq, Nk):  # clustered Q and K
        mu = rng.standard_normal((groups, d)).astype(np.float32)
        g = rng.integers(0, groups, (B, H, N))
        x = mu[g] * amp + rng.standard_normal((B, H, N, d)).astype(np.float32)
        out.append(svg2_synth.f32_to_bf16_bits(x))
    # V ~ N(0, I) as in the svg2-synth recipe: O(1) outputs, the scale the 2e-2 / 2e-3 tolerances are written for
    out.append(svg2_synth.f32_to_bf16_bits(rng.standard_normal((B, H, Nk, d)).astype(np.float32)))
    return out


def label_mismatches_are_ties(X64, cent64, gpu_labels, band=1e-5):
    """Rows whose GPU label differs from the exact argmin must be near-ties (DESIGN R16):
    d(x, c_gpu) - d(x, c_min) <= band * (|x|^2 + |c_min|^2), exact fp64 distances to the centroids the GPU used.
    The denominator is the magnitude the GPU's fp32 ||c||^2 - 2 x.c cancels (SURVEY 8(c) #16's stated fallback: on
    clustered data the flips sit at 1.2-1.9e-5 of d_min but <= 7.1e-7 of |x|^2 + |c|^2, profiles/r02_label_ties.txt).
    Returns (#mismatch, #non-tie)."""
    import oracle
    lab, d1, _ = oracle.assign(X64, cent64)
    bad = np.nonzero(lab != gpu_labels)[0]
    non_tie = 0
    for n in bad:
        dg = float(((X64[n] - cent64[gpu_labels[n]]) ** 2).sum())
        scale = float((X64[n] ** 2).sum()) + float((cent64[lab[n]] ** 2).sum())
        if dg - d1[n] > band * scale:
            non_tie += 1
    return len(bad), non_tie


def mask_mismatch_rows_are_ties(W, Z, sk, p, gpu_mask, or_mask, band=1e-9):
    """Rows where the GPU top-p mask differs from the oracle's must sit on a near-tie of the top-p boundary
    (DESIGN R17): either two w's straddling the boundary are equal within `band` (relative), or the cumulative
    mass before the boundary is within band*Z of p*Z.  Returns (#rows differing, #non-tie rows)."""
    rows = np.nonzero((gpu_mask != or_mask).any(axis=1))[0]
    non_tie = 0
    for i in rows:
        order = sorted(range(W.shape[1]), key=lambda j: (-W[i, j], j))
        order = [j for j in order if W[i, j] > 0]
        w = np.array([W[i, j] for j in order])
        cum = np.concatenate([[0.0], np.cumsum(w)])
        k = int(or_mask[i].sum())
        near = abs(cum[k - 1] - p * Z[i]) <= band * Z[i] or abs(cum[k] - p * Z[i]) <= band * Z[i]
        if k < len(w):
            near = near or abs(w[k] - w[k - 1]) <= band * w[k - 1]
        if not near:
            non_tie += 1
    return len(rows), non_tie
