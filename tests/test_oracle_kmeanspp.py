"""Pins of the oracle's k-means++ cold start (generator and weights fixed by DESIGN R25).

What fixes it independently of the oracle's own code: the published Philox4x32-10 known-answer vectors, the defining
property of k-means++ sampling (pick n with probability proportional to D(x_n), checked statistically against the
exact distances of a tiny 1-D set), uniform first picks, and invariants that hold for any correct implementation
(chosen points never repeat while some weight is positive, C = N picks every point, well-separated blobs each get
one seed).
"""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _kat():
    rows = []
    for ln in open(os.path.join(HERE, "golden", "philox4x32_10_kat.txt")):
        if ln.strip() and not ln.startswith("#"):
            v = [int(x, 16) for x in ln.split()]
            rows.append((v[:4], v[4:6], v[6:]))
    return rows


@pytest.mark.parametrize("ctr,key,expect", _kat())
def test_philox_known_answers(oracle_mod, ctr, key, expect):
    assert list(oracle_mod.philox4x32_10(ctr, key)) == expect


def test_philox_counter_uniformity(oracle_mod):
    # 4096 counters x 4 words: every byte lane of a uniform generator is uniform over 256 values
    words = np.concatenate([oracle_mod.philox4x32_10([i, 0, 0, 0], [7, 3]) for i in range(4096)])
    top = (words >> 24).astype(np.int64)
    counts = np.bincount(top, minlength=256)
    exp = len(top) / 256
    chi2 = float(((counts - exp) ** 2 / exp).sum())
    assert chi2 < 255 + 6 * np.sqrt(2 * 255)  # 6 sigma of chi2(255)


def test_picks_are_distinct_rows(oracle_mod):
    rng = np.random.default_rng(1)
    X = rng.standard_normal((300, 8))
    idx = oracle_mod.kmeanspp_init(X, 50, seed=11, stream=3)
    assert idx.dtype == np.int64 and len(set(idx.tolist())) == 50
    assert idx.min() >= 0 and idx.max() < 300


def test_all_points_when_c_equals_n(oracle_mod):
    rng = np.random.default_rng(2)
    X = rng.standard_normal((40, 4))
    idx = oracle_mod.kmeanspp_init(X, 40, seed=5, stream=0)
    assert sorted(idx.tolist()) == list(range(40))


def test_duplicates_never_repicked(oracle_mod):
    # 10 distinct points, each repeated 30 times: a point at distance 0 from a chosen centroid has weight 0, so the
    # 10 picks land on the 10 distinct values, one each
    rng = np.random.default_rng(3)
    base = rng.standard_normal((10, 6))
    X = np.repeat(base, 30, axis=0)[rng.permutation(300)]
    for stream in range(5):
        idx = oracle_mod.kmeanspp_init(X, 10, seed=9, stream=stream)
        picked = {tuple(r) for r in X[idx]}
        assert picked == {tuple(r) for r in base}


def test_separated_blobs_get_one_seed_each(oracle_mod):
    # 8 blobs of radius ~1 at mutual distance >= ~1000: a second pick inside an already seeded blob has probability
    # < 20 * 4 / 1e6 per pick, so every blob receives exactly one seed
    rng = np.random.default_rng(4)
    centers = rng.standard_normal((8, 5)) * 1000
    X = np.concatenate([c + rng.standard_normal((20, 5)) for c in centers])[rng.permutation(160)]
    blob = np.argmin(((X[:, None, :] - centers[None]) ** 2).sum(-1), axis=1)
    for stream in range(6):
        idx = oracle_mod.kmeanspp_init(X, 8, seed=1, stream=stream)
        assert sorted(blob[idx].tolist()) == list(range(8))


def test_first_pick_uniform_and_second_pick_proportional_to_d(oracle_mod):
    # Points on a line at 0, 1, 2, 4, 8 (d = 1).  Over many independent streams the first pick is uniform and, given
    # the first pick a, the second pick is n with probability (x_n - x_a)^2 / sum_m (x_m - x_a)^2 -- the k-means++
    # rule with D = squared distance (Arthur & Vassilvitskii 2007).  Weight quantisation (2^-32) is far below the
    # statistical resolution.
    x = np.array([0.0, 1.0, 2.0, 4.0, 8.0])[:, None]
    runs = 12000
    first = np.empty(runs, np.int64)
    second = np.empty(runs, np.int64)
    for s in range(runs):
        idx = oracle_mod.kmeanspp_init(x, 2, seed=2024, stream=s)
        first[s], second[s] = idx
    counts = np.bincount(first, minlength=5)
    exp = runs / 5
    assert float(((counts - exp) ** 2 / exp).sum()) < 4 + 6 * np.sqrt(8)
    for a in range(5):
        sel = second[first == a]
        d = (x[:, 0] - x[a, 0]) ** 2
        p = d / d.sum()
        freq = np.bincount(sel, minlength=5) / len(sel)
        sigma = np.sqrt(p * (1 - p) / len(sel))
        assert np.all(np.abs(freq - p) <= 5 * sigma + 1e-12), (a, freq, p)
        assert freq[a] == 0.0  # the chosen point has D = 0


def test_kmeanspp_then_lloyd_objective_non_increasing(oracle_mod):
    rng = np.random.default_rng(5)
    X = rng.standard_normal((500, 8)) + np.repeat(rng.standard_normal((5, 8)) * 4, 100, axis=0)
    labels, cent, sizes, ja, jp, idx = oracle_mod.kmeanspp(X, 5, 4, seed=3, stream=1, return_objective=True)
    assert np.all(np.diff(ja) <= 1e-9 * ja[0])
    assert np.all(jp <= ja + 1e-9 * ja[0])
    assert sizes.sum() == 500
