"""Identification-quality metrics of a sparse-attention selection — TEST INFRASTRUCTURE ONLY.

Plain fp64 numpy, written from the paper's definitions (and SPEC.md's metric module where the paper leaves the
formula implicit); like the rest of ``oracle/`` it may only be imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` leg.  Every function works on one (b, h) head and a set of sampled query rows.

    attention_probs(Q, K, scale, rows)      the true attention distribution P
    oracle_topp_mask(P, p)                  per query, the minimal descending-order key set holding a fraction p of
                                            its attention mass (ties -> lower key index)
    oracle_curve(P, grid)                   (density, recall) of the oracle policy per p
    density(mask)                           selected pairs / all pairs
    recall(mask, P)                         mean over rows of the selected attention mass
    critical_miss_rate(mask, oracle)        oracle pairs the mask drops / oracle pairs
    waste(mask, oracle)                     mask pairs outside the oracle set / mask pairs
    psnr(reference, candidate)              10 log10(peak^2 / MSE), peak = max |reference|
    svg2_token_mask(lq, lk, cmask, rows)    token-level selection of a cluster-pair mask
    position_block_mask(...)                position-block sparse attention: blocks of consecutive
                                            tokens (128 queries x 64 keys), mean-pooled queries, mean- or max-pooled
                                            keys, and the same Eq. 1 / Eq. 2 / top-p rule SVG2 applies to clusters
                                            (oracle.select_topp on the block representatives);
                                            optionally with the blocks cut after a permutation.
"""
from __future__ import annotations

import math

import numpy as np


def attention_probs(Q, K, scale, rows=None):
    """P[r, m] = softmax_m(scale * q_r . k_m) for the sampled query rows, fp64 with a max shift."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    Qr = Q if rows is None else Q[np.asarray(rows)]
    S = (Qr @ K.T) * float(scale)
    S -= S.max(axis=1, keepdims=True)
    E = np.exp(S)
    return E / E.sum(axis=1, keepdims=True)


def oracle_topp_mask(P, p):
    """Per row: keys sorted by score descending (ties: lower index first), taken greedily until the cumulative score
    reaches p of the row's total — the crossing key included, so the set is the minimal such prefix (PAPER.md:11,
    213-214).  p = 1 selects every key with a nonzero score."""
    if not 0.0 < p <= 1.0:
        raise ValueError(f"target p must be in (0, 1], got {p}")
    P = np.asarray(P, dtype=np.float64)
    R, N = P.shape
    mask = np.zeros((R, N), dtype=bool)
    for r in range(R):
        row = P[r]
        if p == 1.0:
            mask[r] = row > 0
            continue
        order = np.lexsort((np.arange(N), -row))  # descending score, then ascending index
        target = p * row.sum()
        cum = 0.0
        for j in order:
            if cum >= target:
                break
            mask[r, j] = True
            cum += row[j]
    return mask


def density(mask):
    """Selected pairs / all pairs."""
    mask = np.asarray(mask, dtype=bool)
    return float(mask.sum()) / mask.size


def recall(mask, P):
    """Mean over query rows of (selected attention mass / total mass)."""
    P = np.asarray(P, dtype=np.float64)
    mask = np.asarray(mask, dtype=bool)
    return float(np.mean((P * mask).sum(axis=1) / P.sum(axis=1)))


def critical_miss_rate(mask, oracle):
    """|oracle pairs not in mask| / |oracle pairs| (0 for an empty oracle set)."""
    mask = np.asarray(mask, dtype=bool)
    oracle = np.asarray(oracle, dtype=bool)
    n = int(oracle.sum())
    return float((oracle & ~mask).sum()) / n if n else 0.0


def waste(mask, oracle):
    """|mask pairs not in the oracle set| / |mask pairs| (0 for an empty mask)."""
    mask = np.asarray(mask, dtype=bool)
    oracle = np.asarray(oracle, dtype=bool)
    n = int(mask.sum())
    return float((mask & ~oracle).sum()) / n if n else 0.0


def oracle_curve(P, grid):
    """[(p, density, recall)] of the oracle policy at each p of the grid."""
    if len(grid) == 0:
        raise ValueError("empty grid")
    out = []
    for p in grid:
        m = oracle_topp_mask(P, p)
        out.append((float(p), density(m), recall(m, P)))
    return out


def psnr(reference, candidate, cap=200.0):
    """10 log10(peak^2 / MSE), peak = max |reference|, MSE in fp64; `cap` dB when the tensors are equal."""
    ref = np.asarray(reference, dtype=np.float64)
    cand = np.asarray(candidate, dtype=np.float64)
    peak = float(np.abs(ref).max())
    if peak == 0.0:
        raise ValueError("reference is all zero")
    mse = float(np.mean((ref - cand) ** 2))
    if mse == 0.0:
        return cap
    return min(cap, 10.0 * math.log10(peak * peak / mse))


def svg2_token_mask(lq, lk, cmask, rows):
    """Token pairs selected by a cluster-pair mask: row r, key m selected iff cmask[lq[rows[r]], lk[m]]."""
    lq = np.asarray(lq)
    lk = np.asarray(lk)
    cmask = np.asarray(cmask, dtype=bool)
    return cmask[lq[np.asarray(rows)]][:, lk]


def position_block_mask(Q, K, rows, scale, p, bq=128, bk=64, pool="mean", perm_q=None, perm_k=None):
    """Position-block selection for the sampled rows: token order (or the order perm_* gives,
    perm[pos] = original index) cut into consecutive blocks of bq queries / bk keys (the last block ragged);
    representatives = mean of the query block, mean or max of the key block (per channel); block pairs chosen by
    Eq. 1 / Eq. 2 with block sizes as weights and top-p per query block.  Returns bool
    [len(rows), N] over ORIGINAL key order."""
    import oracle  # the Eq. 1 / Eq. 2 / top-p rule of the oracle, applied to blocks instead of clusters

    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    N, d = K.shape
    Nq = Q.shape[0]
    pq = np.arange(Nq) if perm_q is None else np.asarray(perm_q)
    pk = np.arange(N) if perm_k is None else np.asarray(perm_k)
    nqb, nkb = -(-Nq // bq), -(-N // bk)
    q_rep = np.empty((nqb, d))
    q_sz = np.empty(nqb, np.int64)
    for i in range(nqb):
        blk = Q[pq[i * bq:(i + 1) * bq]]
        q_rep[i] = blk.mean(axis=0)
        q_sz[i] = blk.shape[0]
    k_rep = np.empty((nkb, d))
    k_sz = np.empty(nkb, np.int64)
    for j in range(nkb):
        blk = K[pk[j * bk:(j + 1) * bk]]
        k_rep[j] = blk.max(axis=0) if pool == "max" else blk.mean(axis=0)
        k_sz[j] = blk.shape[0]
    bmask, _ = oracle.select_topp(q_rep, k_rep, q_sz, k_sz, d, scale, p)
    qpos = np.empty(Nq, np.int64)
    qpos[pq] = np.arange(Nq)  # position of each original query in the cut order
    kpos = np.empty(N, np.int64)
    kpos[pk] = np.arange(N)
    return bmask.astype(bool)[qpos[np.asarray(rows)] // bq][:, kpos // bk]
