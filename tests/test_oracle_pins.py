"""Pins for the fp64 oracle against what the paper and mathematics fix (CPU only, -m "not gpu").

Each test names the passage it pins.  None of them re-types the oracle's own formula: they use closed
forms, brute force on tiny inputs, numpy textbook routines, invariants and special cases.
"""
import math

import numpy as np
import pytest


def np_softmax_attention(Q, K, V, scale, allowed=None):
    """numpy textbook softmax(QK^T s)V (fp64); `allowed` is an optional [Nq, Nk] boolean token mask."""
    S = (Q @ K.T) * scale
    if allowed is not None:
        S = np.where(allowed, S, -np.inf)
    S = S - S.max(axis=1, keepdims=True)
    P = np.exp(S)
    P /= P.sum(axis=1, keepdims=True)
    return P @ V


# ------------------------------------------------------------------ dense attention
def test_dense_single_key_returns_v(oracle_mod):
    rng = np.random.default_rng(1)
    Q = rng.standard_normal((5, 8))
    K = rng.standard_normal((1, 8))
    V = rng.standard_normal((1, 8))
    O = oracle_mod.dense_rows(Q, K, V, 0.3)
    assert np.array_equal(O, np.repeat(V, 5, axis=0))


def test_dense_orthogonal_query_gives_mean_of_v(oracle_mod):
    rng = np.random.default_rng(2)
    K = rng.standard_normal((7, 4))
    V = rng.standard_normal((7, 4))
    Q = np.zeros((3, 4))  # q . k = 0 for every key -> uniform softmax
    O = oracle_mod.dense_rows(Q, K, V, 1.0)
    assert np.max(np.abs(O - V.mean(axis=0))) < 1e-15


def test_softmax_closed_form_quarter_three_quarters(oracle_mod):
    # scores [0, ln 3] -> weights [1/4, 3/4]; V = e_0, e_1 exposes the weights directly
    Q = np.array([[1.0]])
    K = np.array([[0.0], [math.log(3.0)]])
    V = np.array([[1.0, 0.0], [0.0, 1.0]])
    Q2 = np.concatenate([Q, np.zeros((1, 1))], axis=1)
    K2 = np.concatenate([K, np.zeros((2, 1))], axis=1)
    O = oracle_mod.dense_rows(Q2, K2, V, 1.0)
    assert abs(O[0, 0] - 0.25) < 1e-15 and abs(O[0, 1] - 0.75) < 1e-15


@pytest.mark.parametrize("seed", range(5))
def test_dense_matches_numpy_textbook(oracle_mod, seed):
    rng = np.random.default_rng(seed)
    Nq, Nk, d = 17, 23, 8
    Q, K, V = (rng.standard_normal((n, d)) * 2 for n in (Nq, Nk, Nk))
    s = 1 / math.sqrt(d)
    O, lse = oracle_mod.attention_rows(Q, K, V, s, return_lse=True)
    assert np.max(np.abs(O - np_softmax_attention(Q, K, V, s))) < 1e-12
    S = Q @ K.T * s
    ref_lse = S.max(1) + np.log(np.exp(S - S.max(1, keepdims=True)).sum(1))
    assert np.max(np.abs(lse - ref_lse)) < 1e-12


# ------------------------------------------------------------------ masked attention
@pytest.mark.parametrize("seed", range(6))
def test_masked_attention_brute_force(oracle_mod, seed):
    rng = np.random.default_rng(100 + seed)
    N, d, Cq, Ck = 48, 6, 4, 5
    Q, K, V = (rng.standard_normal((N, d)) for _ in range(3))
    lq = rng.integers(0, Cq, N).astype(np.int32)
    lk = rng.integers(0, Ck, N).astype(np.int32)
    lk[:Ck] = np.arange(Ck)  # every key cluster non-empty
    mask = (rng.random((Cq, Ck)) < 0.5).astype(np.uint8)
    mask[np.arange(Cq), rng.integers(0, Ck, Cq)] = 1  # >= 1 selected cluster per row
    allowed = mask[lq][:, lk].astype(bool)
    O = oracle_mod.attention_rows(Q, K, V, 0.4, lq=lq, lk=lk, mask=mask)
    assert np.max(np.abs(O - np_softmax_attention(Q, K, V, 0.4, allowed))) < 1e-12


def test_masked_attention_one_key_per_row_gives_v(oracle_mod):
    # each key its own cluster, each query cluster selects exactly one key cluster -> o = v_j
    rng = np.random.default_rng(7)
    N, d = 6, 4
    Q, K, V = (rng.standard_normal((N, d)) for _ in range(3))
    lq = np.arange(N, dtype=np.int32)
    lk = np.arange(N, dtype=np.int32)
    target = rng.permutation(N)
    mask = np.zeros((N, N), np.uint8)
    mask[np.arange(N), target] = 1
    O = oracle_mod.attention_rows(Q, K, V, 1.0, lq=lq, lk=lk, mask=mask)
    assert np.array_equal(O, V[target])


def test_masked_attention_empty_row_is_error(oracle_mod):
    Q = np.ones((2, 2))
    mask = np.zeros((1, 1), np.uint8)
    with pytest.raises(ValueError):
        oracle_mod.attention_rows(Q, Q, Q, 1.0, lq=np.zeros(2, np.int32), lk=np.zeros(2, np.int32), mask=mask)


# ------------------------------------------------------------------ permutation
def test_permutation_worked_example(oracle_mod):
    perm, off = oracle_mod.permute(np.array([1, 0, 1, 0]), 2)
    assert perm.tolist() == [1, 3, 0, 2] and off.tolist() == [0, 2, 4]


def test_permutation_single_cluster_is_identity(oracle_mod):
    perm, off = oracle_mod.permute(np.zeros(9, np.int32), 1)
    assert perm.tolist() == list(range(9)) and off.tolist() == [0, 9]


def test_permutation_stable_and_bijective(oracle_mod):
    rng = np.random.default_rng(3)
    labels = rng.integers(0, 13, 500).astype(np.int32)
    perm, off = oracle_mod.permute(labels, 13)
    assert sorted(perm.tolist()) == list(range(500))
    # numpy's stable argsort is the textbook stable counting order
    assert np.array_equal(perm, np.argsort(labels, kind="stable"))
    assert np.array_equal(np.diff(off), np.bincount(labels, minlength=13))


@pytest.mark.parametrize("seed", range(100))
def test_permutation_equivalence_identity(oracle_mod, seed):
    # pi_q^T Attn(pi_q Q, pi_k K, pi_k V) = Attn(Q, K, V)
    rng = np.random.default_rng(1000 + seed)
    Nq, Nk, d = rng.integers(2, 40), rng.integers(2, 40), 8
    Q, K, V = rng.standard_normal((Nq, d)), rng.standard_normal((Nk, d)), rng.standard_normal((Nk, d))
    pq = rng.permutation(Nq)
    pk = rng.permutation(Nk)
    Op = oracle_mod.dense_rows(Q[pq], K[pk], V[pk], 0.35)
    O = np.empty_like(Op)
    O[pq] = Op
    assert np.max(np.abs(O - oracle_mod.dense_rows(Q, K, V, 0.35))) < 1e-12


# ------------------------------------------------------------------ k-means
def np_lloyd(X, C, iters, init):
    """Test-local textbook Lloyd: same init, ties -> lowest index, empty cluster keeps its centroid."""
    c = init.copy()
    for _ in range(iters):
        D = ((X[:, None, :] - c[None, :, :]) ** 2).sum(-1)
        lab = np.argmin(D, axis=1)  # numpy argmin returns the first minimum
        for j in range(C):
            if np.any(lab == j):
                c[j] = X[lab == j].mean(axis=0)
    return lab, c


def test_kmeans_C_equals_N_has_zero_inertia(oracle_mod):
    rng = np.random.default_rng(4)
    X = rng.standard_normal((20, 5))
    lab, cent, sizes, ja, jp = oracle_mod.kmeans(X, 20, 2, return_objective=True)
    assert lab.tolist() == list(range(20)) and np.all(sizes == 1)
    assert jp[-1] == 0.0 and np.array_equal(cent, X)


def test_kmeans_C_equals_1_gives_mean(oracle_mod):
    rng = np.random.default_rng(5)
    X = rng.standard_normal((50, 7))
    lab, cent, sizes = oracle_mod.kmeans(X, 1, 3)
    assert np.all(lab == 0) and sizes[0] == 50
    assert np.max(np.abs(cent[0] - X.mean(axis=0))) < 1e-14


def test_kmeans_separated_blobs_recovered(oracle_mod):
    rng = np.random.default_rng(6)
    centres = rng.standard_normal((4, 16)) * 10.0  # >> unit noise (10 sigma)
    truth = np.repeat(np.arange(4), 25)
    X = centres[truth] + rng.standard_normal((100, 16)) * 0.1
    X = X[rng.permutation(100)]
    truth = None
    lab, cent, _ = oracle_mod.kmeans(X, 4, 10, init=X[[0, 30, 60, 90]] * 0 + np.array(
        [X[np.argmin(((X - c) ** 2).sum(1))] for c in centres]))
    # each true blob maps to exactly one cluster (partition equality up to relabeling)
    blob = np.argmin(((X[:, None, :] - centres[None]) ** 2).sum(-1), axis=1)
    pairs = set(zip(blob.tolist(), lab.tolist()))
    assert len(pairs) == 4 and len({b for b, _ in pairs}) == 4 and len({c for _, c in pairs}) == 4


@pytest.mark.parametrize("seed", range(4))
def test_kmeans_objective_non_increasing_and_argmin(oracle_mod, seed):
    rng = np.random.default_rng(10 + seed)
    X = rng.standard_normal((300, 8)) + rng.integers(0, 3, (300, 1)) * 2.0
    lab, cent, sizes, ja, jp = oracle_mod.kmeans(X, 9, 6, return_objective=True)
    for t in range(6):
        assert jp[t] <= ja[t] * (1 + 1e-12)
        if t + 1 < 6:
            assert ja[t + 1] <= jp[t] * (1 + 1e-12)
    assert sizes.sum() == 300 and np.array_equal(np.bincount(lab, minlength=9), sizes)
    # the returned centroids are the exact means of the returned clusters
    for j in range(9):
        if sizes[j]:
            assert np.max(np.abs(cent[j] - X[lab == j].mean(0))) < 1e-12


@pytest.mark.parametrize("seed", range(4))
def test_kmeans_matches_numpy_lloyd(oracle_mod, seed):
    rng = np.random.default_rng(20 + seed)
    N, C, d = 200, 7, 5
    X = rng.standard_normal((N, d)) + rng.integers(0, 4, (N, 1))
    init = X[(np.arange(C) * N) // C]  # the strided cold init (R2) written as numpy indexing
    lab, cent, _ = oracle_mod.kmeans(X, C, 5)
    lab2, cent2 = np_lloyd(X, C, 5, init)
    assert np.array_equal(lab, lab2)
    assert np.max(np.abs(cent - cent2)) < 1e-12


def test_kmeans_warm_start_fixed_point(oracle_mod):
    rng = np.random.default_rng(30)
    X = rng.standard_normal((400, 6)) + rng.integers(0, 5, (400, 1)) * 3.0
    lab, cent, _ = oracle_mod.kmeans(X, 5, 60)
    lab2, cent2, _ = oracle_mod.kmeans(X, 5, 1, init=cent)
    assert np.array_equal(lab, lab2) and np.max(np.abs(cent - cent2)) < 1e-12


def test_kmeans_row_permutation_equivariance(oracle_mod):
    rng = np.random.default_rng(31)
    X = rng.standard_normal((120, 4))
    init = rng.standard_normal((6, 4))
    lab, cent, _ = oracle_mod.kmeans(X, 6, 3, init=init)
    p = rng.permutation(120)
    labp, centp, _ = oracle_mod.kmeans(X[p], 6, 3, init=init)
    assert np.array_equal(labp, lab[p]) and np.max(np.abs(centp - cent)) < 1e-12


def test_kmeans_empty_cluster_keeps_centroid(oracle_mod):
    X = np.array([[0.0, 0.0], [0.1, 0.0], [0.0, 0.1]])
    init = np.array([[0.0, 0.0], [100.0, 100.0]])
    lab, cent, sizes = oracle_mod.kmeans(X, 2, 2, init=init)
    assert sizes.tolist() == [3, 0] and np.array_equal(cent[1], init[1])


def test_kmeans_invalid_arguments(oracle_mod):
    with pytest.raises(ValueError):
        oracle_mod.kmeans(np.ones((3, 2)), 4, 1)
    with pytest.raises(ValueError):
        oracle_mod.kmeans(np.ones((3, 2)), 0, 1)


# ------------------------------------------------------------------ Eq. 1 / Eq. 2 / top-p
def test_eq2_single_key_cluster(oracle_mod):
    rng = np.random.default_rng(40)
    mask, pairs, S, W, Z = oracle_mod.select_topp(rng.standard_normal((3, 4)), rng.standard_normal((1, 4)),
                                                  [2, 3, 4], [9], 4, 0.5, 0.5, return_tables=True)
    assert np.allclose(W / Z[:, None], 1.0, atol=0) and mask.ravel().tolist() == [1, 1, 1]
    assert pairs == 9 * 9


def test_eq2_equal_centroids_uniform(oracle_mod):
    cq = np.ones((2, 3))
    ck = np.ones((5, 3)) * 0.7
    _, _, S, W, Z = oracle_mod.select_topp(cq, ck, [1, 1], [4] * 5, 3, 0.5, 0.9, return_tables=True)
    assert np.all(W / Z[:, None] == 0.2)


def test_eq2_hand_evaluated_3x4(oracle_mod):
    # d = 2, scale = 1: S_0j = [ln 2, 0, 0, 0], sizes [1, 2, 1, 4] -> P'_0 = [2, 2, 1, 4] / 9;
    # S_1j = [0, ln 3, 0, 0] -> [1, 6, 1, 4] / 12;  S_2j = 0 -> sizes / 8
    cq = np.array([[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]])
    ck = np.array([[math.log(2.0), 0.0], [0.0, math.log(3.0)], [0.0, 0.0], [0.0, 0.0]])
    _, _, S, W, Z = oracle_mod.select_topp(cq, ck, [1, 1, 1], [1, 2, 1, 4], 2, 1.0, 0.5, return_tables=True)
    P = W / Z[:, None]
    expect = np.array([[2, 2, 1, 4], [1, 6, 1, 4], [1, 2, 1, 4]], float) / np.array([[9], [12], [8]])
    assert np.max(np.abs(P - expect)) < 1e-15


def test_topp_worked_example_060_030_010(oracle_mod):
    # equal centroids, sizes 6/3/1 -> P' = [0.6, 0.3, 0.1]; p = 0.85 selects {0, 1}
    mask, pairs = oracle_mod.select_topp(np.zeros((1, 2)), np.zeros((3, 2)), [5], [6, 3, 1], 2, 1.0, 0.85)
    assert mask.ravel().tolist() == [1, 1, 0] and pairs == 5 * 9


def test_topp_p1_selects_all_nonempty(oracle_mod):
    rng = np.random.default_rng(41)
    sk = np.array([3, 0, 5, 1, 0, 2])
    mask, pairs = oracle_mod.select_topp(rng.standard_normal((4, 3)), rng.standard_normal((6, 3)),
                                         [1, 2, 3, 4], sk, 3, 0.5, 1.0)
    assert np.array_equal(mask, np.tile((sk > 0).astype(np.uint8), (4, 1))) and pairs == 10 * 11


@pytest.mark.parametrize("seed", range(20))
def test_topp_is_minimal_descending_prefix(oracle_mod, seed):
    rng = np.random.default_rng(50 + seed)
    Cq, Ck, d = 5, 17, 4
    sk = rng.integers(0, 6, Ck)
    sk[0] = 3
    p = rng.uniform(0.05, 0.99)
    mask, _, S, W, Z = oracle_mod.select_topp(rng.standard_normal((Cq, d)) * 2, rng.standard_normal((Ck, d)) * 2,
                                              np.ones(Cq, np.int64), sk, d, 0.5, p, return_tables=True)
    for i in range(Cq):
        order = sorted(range(Ck), key=lambda j: (-W[i, j], j))
        # brute force: smallest k whose top-k mass reaches p (exact rational check in fp64 per prefix)
        best = None
        for k in range(1, Ck + 1):
            if sum(W[i, j] for j in order[:k]) >= p * Z[i] or W[i, order[k - 1]] == 0:
                best = k
                break
        chosen = {j for j in order[:best] if W[i, j] > 0}
        assert {j for j in range(Ck) if mask[i, j]} == chosen


def test_topp_nesting_in_p(oracle_mod):
    rng = np.random.default_rng(60)
    cq, ck = rng.standard_normal((6, 5)), rng.standard_normal((30, 5))
    sq, sk = rng.integers(1, 9, 6), rng.integers(0, 9, 30)
    prev = np.zeros((6, 30), np.uint8)
    for p in [0.1, 0.3, 0.5, 0.7, 0.9, 0.97, 1.0]:
        m, _ = oracle_mod.select_topp(cq, ck, sq, sk, 5, 0.6, p)
        assert np.all(m >= prev)
        prev = m


def test_topp_invalid_p(oracle_mod):
    for p in (0.0, -0.1, 1.0001):
        with pytest.raises(ValueError):
            oracle_mod.select_topp(np.ones((1, 1)), np.ones((1, 1)), [1], [1], 1, 1.0, p)


@pytest.mark.parametrize("seed", range(5))
def test_singleton_clusters_reduce_to_per_query_oracle_topp(oracle_mod, seed):
    # C = N, strided init = the tokens themselves, 1 iteration: P' is the true attention P, so the selection
    # equals the per-query oracle top-p policy of PAPER.md:11, 213 (ties by ascending key index)
    rng = np.random.default_rng(70 + seed)
    N, d, p = 24, 6, 0.8
    Q, K = rng.standard_normal((N, d)), rng.standard_normal((N, d))
    s = 1 / math.sqrt(d)
    lq, cq, sq = oracle_mod.kmeans(Q, N, 1)
    lk, ck, sk = oracle_mod.kmeans(K, N, 1)
    assert lq.tolist() == list(range(N)) and lk.tolist() == list(range(N))
    mask, pairs = oracle_mod.select_topp(cq, ck, sq, sk, d, s, p)
    S = Q @ K.T * s
    P = np.exp(S - S.max(1, keepdims=True))
    P /= P.sum(1, keepdims=True)
    for i in range(N):
        order = sorted(range(N), key=lambda j: (-P[i, j], j))
        cum, sel = 0.0, set()
        for j in order:
            if cum >= p:
                break
            sel.add(j)
            cum += P[i, j]
        assert {j for j in range(N) if mask[i, j]} == sel
        assert sum(P[i, j] for j in sel) >= p - 1e-12  # the true-mass guarantee
    assert pairs == int(mask.sum())


# ------------------------------------------------------------------ whole pipeline pins
@pytest.mark.parametrize("seed", range(3))
def test_sparse_p1_equals_dense(oracle_mod, seed):
    # north star: top-p = 1.0 reproduces dense softmax attention (<= 1e-12)
    rng = np.random.default_rng(80 + seed)
    N, d = 96, 8
    Q, K, V = (rng.standard_normal((N, d)) * 2 for _ in range(3))
    r = oracle_mod.sparse_attention_head(Q, K, V, 6, 9, 3, 1.0)
    dense = oracle_mod.dense_rows(Q, K, V, 1 / math.sqrt(d))
    assert np.max(np.abs(r["O"] - dense)) < 1e-12
    assert r["pairs"] == N * N


def test_pairs_equal_expanded_token_mask(oracle_mod):
    rng = np.random.default_rng(90)
    N, d = 128, 8
    Q, K, V = (rng.standard_normal((N, d)) for _ in range(3))
    r = oracle_mod.sparse_attention_head(Q, K, V, 5, 11, 4, 0.7)
    token_mask = r["mask"][r["labels_q"]][:, r["labels_k"]]
    assert r["pairs"] == int(token_mask.sum())
    assert oracle_mod.flops_from_pairs(r["pairs"], d) == 4 * d * int(token_mask.sum())


def test_density_accounting_reproduces_table1_flops(oracle_mod):
    """The paper's FLOP column equals L + A (w + (1-w) rho) with A = calls * 4 N^2 d H.
    Fit A, L from the dense row and one sparse row of each model; predict every other row to the printed
    precision.  Pins density = selected pairs / N^2 and FLOP = 4 d * pairs per head."""
    import csv
    import os
    rows = [r for r in csv.reader(open(os.path.join(os.path.dirname(__file__), "golden", "table1_flops.csv")))
            if r and not r[0].startswith("#")]
    shapes = {"wan_i2v": (75600, 40), "wan_t2v": (75600, 40), "hunyuan": (118800, 24)}
    for model, (N, H) in shapes.items():
        mr = [(t, float(w), float(rho), float(f)) for m, t, w, rho, f, _ in rows if m == model]
        dense = [x for x in mr if x[2] == 1.0][0][3]
        t, w, rho, f = [x for x in mr if x[0] == "main" and x[2] < 1.0][0]
        A = (dense - f) / ((1 - w) * (1 - rho))
        L = dense - A
        for t, w, rho, f in mr:
            assert abs(L + A * (w + (1 - w) * rho) - f) < 0.02, (model, t, rho)
        per_call = oracle_mod.flops_from_pairs(N * N, 128) * H / 1e15  # PF per attention call, all heads
        calls = A / per_call
        if model == "wan_t2v":
            assert abs(calls - 4000) < 2
        if model == "wan_i2v":
            assert abs(calls - 3200) < 2
