"""CPU pins for the oracle's assignment step and the k-means tie rule (DESIGN R5: argmin ties -> lowest centroid index).

`oracle.assign` is the ground truth every GPU label-mismatch verdict (R16 tie band) rests on, so it is pinned here
against a brute force that shares nothing with it.  Inputs are small integers: every squared distance is then an
exact integer in fp64 whatever the summation order, so the brute force (numpy broadcasting + pairwise sums) and the
oracle's sequential loop must agree BIT FOR BIT — labels, best and second-best distances — and exact ties occur
often enough to exercise the tie rule on every draw.  A wrong tie comparison (<= for <), a second-best that is not
refreshed when a new best appears, a dropped coordinate or a transposed centroid index each fails one of these.
Paper: Lloyd assignment, PAPER.md:259 (argmin over centroids); the tie rule is DESIGN R5 (the paper is silent).
"""
import numpy as np
import pytest


def brute_assign(X, C):
    """Exhaustive argmin over every centroid: all distances, then the first index attaining the minimum."""
    D = ((X[:, None, :] - C[None, :, :]) ** 2).sum(-1)
    lab = np.empty(X.shape[0], np.int64)
    d1 = np.empty(X.shape[0])
    d2 = np.empty(X.shape[0])
    for n in range(X.shape[0]):
        row = D[n]
        m = row.min()
        lab[n] = int(np.flatnonzero(row == m)[0])  # ties -> lowest j
        srt = np.sort(row)
        d1[n] = srt[0]
        d2[n] = srt[1] if len(srt) > 1 else np.inf  # second-smallest WITH multiplicity (a tie gives d2 == d1)
    return lab, d1, d2


@pytest.mark.parametrize("seed", range(8))
def test_assign_matches_brute_force_exactly_on_integer_data(oracle_mod, seed):
    rng = np.random.default_rng(100 + seed)
    N, C, d = 400, 23, 6
    X = rng.integers(-3, 4, (N, d)).astype(np.float64)
    cent = rng.integers(-3, 4, (C, d)).astype(np.float64)
    cent[7] = cent[2]  # an exact duplicate centroid: every point nearest to it ties between j = 2 and 7
    lab, d1, d2 = oracle_mod.assign(X, cent)
    blab, bd1, bd2 = brute_assign(X, cent)
    assert np.array_equal(lab, blab)
    assert np.array_equal(d1, bd1) and np.array_equal(d2, bd2)
    ties = np.sum(bd1 == bd2)
    assert ties > 0  # the draw exercises the tie rule
    assert not np.any(lab == 7)  # the higher duplicate never wins


def test_assign_tie_goes_to_lowest_index(oracle_mod):
    # x = 0 is at squared distance 1 from c = -1 (j = 1) and +1 (j = 2), 4 from c = 2 (j = 0): tie -> 1;
    # x = 1.5 is at 0.25 from c = 2 (j = 0) and c = 1 (j = 2): tie -> 0;  x = -1 sits on c = -1 (j = 1)
    X = np.array([[0.0], [1.5], [-1.0]])
    cent = np.array([[2.0], [-1.0], [1.0]])
    lab, d1, d2 = oracle_mod.assign(X, cent)
    assert lab.tolist() == [1, 0, 1]
    assert d1.tolist() == [1.0, 0.25, 0.0] and d2.tolist() == [1.0, 0.25, 4.0]


def test_assign_second_best_refreshed_by_a_new_best(oracle_mod):
    # centroids visited in decreasing distance: each new best must push the previous best into d2
    X = np.zeros((1, 2))
    cent = np.array([[4.0, 0.0], [3.0, 0.0], [2.0, 0.0], [1.0, 0.0]])
    lab, d1, d2 = oracle_mod.assign(X, cent)
    assert lab[0] == 3 and d1[0] == 1.0 and d2[0] == 4.0


def test_assign_uses_every_coordinate(oracle_mod):
    # the points differ from the centroids only in the last coordinate
    X = np.array([[0.0, 0.0, 0.0, 5.0]])
    cent = np.array([[0.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 4.0]])
    lab, d1, d2 = oracle_mod.assign(X, cent)
    assert lab[0] == 1 and d1[0] == 1.0 and d2[0] == 25.0


@pytest.mark.parametrize("seed", range(4))
def test_kmeans_ties_go_to_lowest_index_every_iteration(oracle_mod, seed):
    """R5 inside Lloyd: on integer data with duplicated rows and duplicated initial centroids, every iteration's
    labels equal the brute-force first-minimum assignment against that iteration's centroids, and the update is
    the exact mean (checked against a test-local Lloyd that uses brute_assign)."""
    rng = np.random.default_rng(200 + seed)
    N, C, d = 300, 12, 4
    base = rng.integers(-2, 3, (40, d)).astype(np.float64)
    X = base[rng.integers(0, 40, N)]  # many duplicated rows
    init = X[rng.integers(0, N, C)].copy()
    init[5] = init[1]  # duplicate centroids: cluster 5 can only ever be empty while they coincide
    c = init.copy()
    for it in range(1, 5):
        lab, cent, sizes = oracle_mod.kmeans(X, C, it, init=init)
        # one more brute-force Lloyd step from the previous iteration's centroids
        blab, _, _ = brute_assign(X, c)
        assert np.array_equal(lab, blab), f"iteration {it}"
        nc = c.copy()
        for j in range(C):
            if np.any(blab == j):
                nc[j] = X[blab == j].sum(0) / np.sum(blab == j)
        assert np.array_equal(sizes, np.bincount(blab, minlength=C))
        assert np.max(np.abs(cent - nc)) <= 1e-12 * max(1.0, np.abs(nc).max())
        if it == 1:  # while the duplicates coincide the higher one never takes a point (R5) and keeps its centroid (R6)
            assert sizes[5] == 0 and np.array_equal(cent[5], init[5])
        c = nc


def test_kmeans_equidistant_point_goes_to_lower_cluster(oracle_mod):
    # 1-D: centroids at 0 and 2, the point 1 is equidistant; 0 and 2 are their own clusters' members
    X = np.array([[0.0], [1.0], [2.0]])
    lab, cent, sizes = oracle_mod.kmeans(X, 2, 1, init=np.array([[0.0], [2.0]]))
    assert lab.tolist() == [0, 0, 1] and sizes.tolist() == [2, 1]
    assert cent[:, 0].tolist() == [0.5, 2.0]
    # with the centroids listed the other way round the tie goes to the new lower index
    lab, cent, sizes = oracle_mod.kmeans(X, 2, 1, init=np.array([[2.0], [0.0]]))
    assert lab.tolist() == [1, 0, 0] and cent[:, 0].tolist() == [1.5, 0.0]
