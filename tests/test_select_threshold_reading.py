"""DESIGN R27 on the CPU: the GPU selects the top-p ranks without sorting, as the weights at or above
w* = max{v : B(v) >= p Z} with B(v) = sum of the w >= v (ties at w* taken in ascending j while the mass before them
stays below p Z).  This checks that reading against the oracle's sorted walk (R11) on rows where the
two can only differ by rounding: integer-valued weights (every sum exact in fp64), with and without ties at the
boundary.  Host logic only: no GPU, no library."""
import numpy as np
import pytest

import oracle as oracle_mod


def threshold_select(w, p):
    """The R27 decision, written out in numpy (exact sums: the test feeds integer-valued weights)."""
    pos = w > 0
    target = p * w[pos].sum()
    vals = np.unique(w[pos])[::-1]  # candidate thresholds, descending
    B = np.array([w[w >= v].sum() for v in vals])
    ok = vals[B >= target]
    wstar = ok.max() if ok.size else 0.0
    sel = pos & (w > wstar)
    above = w[w > wstar].sum()
    tied = np.nonzero(pos & (w == wstar))[0]  # ascending j
    for k, j in enumerate(tied):
        sel[j] = above + k * wstar < target
    return sel


def walk_select(w, p):
    """The oracle's rule (R11) on the same weights: sort by (w desc, j asc), take ranks whose preceding mass < p Z."""
    order = sorted(range(len(w)), key=lambda j: (-w[j], j))
    Z = w[w > 0].sum()
    sel = np.zeros(len(w), bool)
    mass = 0.0
    for j in order:
        if w[j] > 0 and mass < p * Z:
            sel[j] = True
        mass += max(w[j], 0.0)
    return sel


@pytest.mark.parametrize("seed", range(40))
def test_threshold_equals_sorted_walk(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    w = rng.integers(0, 12 if seed % 2 else 10_000, n).astype(np.float64)  # small ranges: many ties
    if not (w > 0).any():
        w[0] = 1.0
    for p in (0.1, 0.5, 0.9, 0.97):
        assert np.array_equal(threshold_select(w, p), walk_select(w, p)), (seed, p)


def test_walk_matches_the_oracle_selection():
    """walk_select is the oracle's rule: on single-row problems with equal centroids (S = 0, so every Eq. 2 weight is
    the integer cluster size), the oracle's mask equals walk_select and threshold_select."""
    rng = np.random.default_rng(7)
    for trial in range(20):
        Ck = int(rng.integers(2, 60))
        d = 8
        ck = np.zeros((Ck, d))  # equal centroids: S = 0, w_j = |K_j|
        cq = np.zeros((1, d))
        sk = rng.integers(0, 9, Ck)
        sk[0] = max(sk[0], 1)
        sq = np.array([3])
        for p in (0.3, 0.8):
            om, _ = oracle_mod.select_topp(cq, ck, sq, sk, d, 1.0, p)
            w = sk.astype(np.float64)
            assert np.array_equal(om[0].astype(bool), walk_select(w, p)), (trial, p)
            assert np.array_equal(om[0].astype(bool), threshold_select(w, p)), (trial, p)
