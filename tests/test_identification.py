"""Pins of oracle/identification.py (the identification-quality metrics of SURVEY 8(f) row 3) against values the
definitions fix: SPEC.md's worked examples, brute force on tiny instances, closed forms
and special cases; and the GPU-box tool (tools/identification.py, torch) reproduced by the oracle on the tiny config."""
import itertools
import math
import os
import sys

import numpy as np
import pytest

import oracle.identification as ident

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- oracle top-p policy
def test_topp_worked_example():
    # row [0.5, 0.3, 0.2], p = 0.7 -> keys {0, 1} (0.5 < 0.7 <= 0.8)
    m = ident.oracle_topp_mask(np.array([[0.5, 0.3, 0.2]]), 0.7)
    assert m.tolist() == [[True, True, False]]
    # the crossing key is included; exactly reaching p stops
    assert ident.oracle_topp_mask(np.array([[0.5, 0.3, 0.2]]), 0.8).tolist() == [[True, True, False]]
    assert ident.oracle_topp_mask(np.array([[0.5, 0.3, 0.2]]), 0.5).tolist() == [[True, False, False]]


def test_topp_p1_selects_nonzero_and_ties_by_index():
    P = np.array([[0.25, 0.0, 0.25, 0.5], [0.25, 0.25, 0.25, 0.25]])
    assert ident.oracle_topp_mask(P, 1.0).tolist() == [[True, False, True, True], [True] * 4]
    # equal scores: lower index first
    assert ident.oracle_topp_mask(P[1:], 0.5).tolist() == [[True, True, False, False]]
    with pytest.raises(ValueError):
        ident.oracle_topp_mask(P, 0.0)
    with pytest.raises(ValueError):
        ident.oracle_topp_mask(P, 1.5)


@pytest.mark.parametrize("seed", range(3))
def test_topp_is_the_minimal_prefix_by_brute_force(seed):
    """Random 16 x 16 P, p = 0.9: per row the smallest k whose top-k mass reaches p, found by trying
    every k on the descending order, and no set of fewer keys reaches p."""
    rng = np.random.default_rng(seed)
    P = rng.random((16, 16)) ** 3
    P /= P.sum(1, keepdims=True)
    m = ident.oracle_topp_mask(P, 0.9)
    for r in range(16):
        s = np.sort(P[r])[::-1]
        kmin = next(k for k in range(1, 17) if s[:k].sum() >= 0.9 * P[r].sum())
        assert m[r].sum() == kmin
        assert P[r][m[r]].sum() >= 0.9 * P[r].sum()
        assert s[:kmin - 1].sum() < 0.9 * P[r].sum()  # fewer keys cannot reach p


def test_oracle_dominance_exhaustive():
    """no per-row subset of the same size holds more mass than the oracle set (N_k <= 12, all subsets)."""
    rng = np.random.default_rng(4)
    P = rng.random((6, 10)) ** 2
    P /= P.sum(1, keepdims=True)
    for p in (0.3, 0.6, 0.9):
        m = ident.oracle_topp_mask(P, p)
        for r in range(6):
            k = int(m[r].sum())
            best = max(P[r, list(c)].sum() for c in itertools.combinations(range(10), k))
            assert P[r][m[r]].sum() >= best - 1e-12


def test_topp_nesting_and_recall_at_least_p():
    rng = np.random.default_rng(5)
    P = rng.random((20, 50)) ** 4
    P /= P.sum(1, keepdims=True)
    prev = None
    for p in (0.1, 0.3, 0.5, 0.7, 0.9, 0.95, 1.0):
        m = ident.oracle_topp_mask(P, p)
        assert np.all((P * m).sum(1) >= p * P.sum(1) - 1e-12)  # per row
        if prev is not None:
            assert np.all(prev <= m)  # greedy prefixes nest
        prev = m


def test_curve_special_cases():
    P = np.full((4, 10), 0.1)
    assert ident.oracle_curve(P, [1.0]) == [(1.0, 1.0, 1.0)]
    for p in (0.25, 0.5, 0.73):
        (_, dens, rec), = ident.oracle_curve(P, [p])
        expect = math.ceil(p * 10 - 1e-12) / 10  # uniform P: density == recall == ceil(p Nk) / Nk
        assert abs(dens - expect) < 1e-12 and abs(rec - expect) < 1e-12
    with pytest.raises(ValueError):
        ident.oracle_curve(P, [])


# ---------------------------------------------------------------- metrics
def test_density_recall_miss_waste_closed_forms():
    full = np.ones((5, 10), bool)
    one = np.zeros((5, 10), bool)
    one[np.arange(5), np.arange(5)] = True
    assert ident.density(full) == 1.0 and abs(ident.density(one) - 0.1) < 1e-15
    rng = np.random.default_rng(6)
    rnd = rng.random((7, 13)) < 0.3
    assert ident.density(rnd) == sum(bin(int("".join("1" if b else "0" for b in row), 2)).count("1")
                                     for row in rnd) / rnd.size  # popcount
    P = rng.random((5, 10))
    P /= P.sum(1, keepdims=True)
    assert abs(ident.recall(full, P) - 1.0) < 1e-12
    U = np.full((5, 10), 0.1)
    k3 = np.zeros((5, 10), bool)
    k3[:, :3] = True
    assert abs(ident.recall(k3, U) - 0.3) < 1e-12  # uniform P, k of n -> k / n
    # recall against a scalar double loop
    ref = np.mean([sum(P[r, m] for m in range(10) if rnd[r % 7, m]) for r in range(5)])
    assert abs(ident.recall(rnd[:5, :10], P) - ref) < 1e-12
    orc = ident.oracle_topp_mask(P, 0.7)
    assert ident.critical_miss_rate(full, orc) == 0.0 and ident.critical_miss_rate(~orc, orc) == 1.0
    assert ident.waste(orc, orc) == 0.0
    q = ident.density(orc)
    assert abs(ident.waste(full, orc) - (1 - q)) < 1e-12  # full mask, oracle density q -> 1 - q
    # critical-selected + wasted-selected == selected
    m = rnd[:5, :10]
    crit = (m & orc).sum()
    assert crit + round(ident.waste(m, orc) * m.sum()) == m.sum()
    assert abs(ident.critical_miss_rate(m, orc) - (orc & ~m).sum() / orc.sum()) < 1e-15


def test_psnr_closed_forms():
    assert ident.psnr([1.0, 0.0], [1.0, 0.0]) == 200.0
    assert abs(ident.psnr([1.0, 0.0], [0.0, 0.0]) - 10 * math.log10(2.0)) < 1e-12  # 3.0103 dB
    rng = np.random.default_rng(7)
    a, b = rng.standard_normal(100), rng.standard_normal(100)
    assert abs(ident.psnr(a, b) - ident.psnr(3.7 * a, 3.7 * b)) < 1e-9  # scale invariance


def test_nested_masks_are_monotone():
    rng = np.random.default_rng(8)
    P = rng.random((6, 30))
    m1 = rng.random((6, 30)) < 0.2
    m2 = m1 | (rng.random((6, 30)) < 0.2)
    assert ident.recall(m1, P) <= ident.recall(m2, P) and ident.density(m1) <= ident.density(m2)


# ---------------------------------------------------------------- position blocks
def test_singleton_blocks_reduce_to_the_oracle_policy():
    """bq = bk = 1: every block is one token with weight 1, so Eq. 2 is the true attention row and the block top-p
    is the per-query oracle policy exactly (the singleton special case)."""
    rng = np.random.default_rng(9)
    Q, K = rng.standard_normal((24, 16)), rng.standard_normal((24, 16))
    scale = 1 / 4.0
    rows = np.arange(24)
    P = ident.attention_probs(Q, K, scale, rows)
    for p in (0.5, 0.9):
        assert np.array_equal(ident.position_block_mask(Q, K, rows, scale, p, bq=1, bk=1), ident.oracle_topp_mask(P, p))


def test_block_mask_structure_and_permutation():
    """Whole-block structure: rows of one query block share their selection, keys of one key block are selected
    together; p = 1 selects everything; with permutations the blocks are cut in permuted order (a permutation that
    is the identity changes nothing; reversing the order reverses the key blocks)."""
    rng = np.random.default_rng(10)
    N, d = 300, 8
    Q, K = rng.standard_normal((N, d)), rng.standard_normal((N, d)) * 2
    rows = np.arange(N)
    m = ident.position_block_mask(Q, K, rows, 0.35, 0.6, bq=128, bk=64)
    for i0 in range(0, N, 128):
        assert np.all(m[i0:i0 + 128] == m[i0])
    for j0 in range(0, N, 64):
        assert np.all(m[:, j0:j0 + 64] == m[:, j0:j0 + 1])
    assert ident.position_block_mask(Q, K, rows, 0.35, 1.0).all()
    ident_perm = np.arange(N)
    assert np.array_equal(ident.position_block_mask(Q, K, rows, 0.35, 0.6, perm_q=ident_perm, perm_k=ident_perm), m)
    mx = ident.position_block_mask(Q, K, rows, 0.35, 0.6, pool="max")
    assert mx.shape == m.shape and mx.any()


def test_svg2_token_mask():
    lq = np.array([0, 1, 1, 0])
    lk = np.array([1, 0, 2])
    cm = np.array([[1, 0, 1], [0, 1, 0]], np.uint8)
    assert ident.svg2_token_mask(lq, lk, cm, [0, 2]).tolist() == [[False, True, True], [True, False, False]]


# ---------------------------------------------------------------- the tool, reproduced by the oracle
def _tool():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import identification as tool  # noqa: E402
    return tool


def test_tool_metrics_match_oracle_tiny():
    """tools/identification.py's torch metric path (run here on CPU in fp64) equals the oracle's on the tiny config:
    oracle sets, recall, miss rate, waste, and the position-block selections (mean / max pooling, and cut after a
    permutation)."""
    torch = pytest.importorskip("torch")
    import svg2_synth
    tool = _tool()
    wl = svg2_synth.WORKLOADS["tiny"]
    q, k, _ = svg2_synth.generate(wl)
    Q = svg2_synth.bf16_bits_to_f64(q)[0, 0]
    K = svg2_synth.bf16_bits_to_f64(k)[0, 0]
    scale = 1 / math.sqrt(wl.d)
    rows = np.sort(np.random.default_rng(0).choice(wl.N, 96, replace=False))
    P = ident.attention_probs(Q, K, scale, rows)
    Qt, Kt, Pt, rt = torch.from_numpy(Q), torch.from_numpy(K), torch.from_numpy(P), torch.from_numpy(rows)
    rng = np.random.default_rng(1)
    perm_q, perm_k = rng.permutation(wl.N), rng.permutation(wl.N)
    for p in (0.5, 0.9):
        orc = ident.oracle_topp_mask(P, p)
        assert np.array_equal(tool.oracle_sets(Pt, p).numpy(), orc)
        for pool in ("mean", "max"):
            ref = ident.position_block_mask(Q, K, rows, scale, p, pool=pool)
            got = tool.position_blocks(Qt, Kt, rt, scale, p, pool=pool).numpy()
            assert np.array_equal(got, ref), pool
        ref = ident.position_block_mask(Q, K, rows, scale, p, perm_q=perm_q, perm_k=perm_k)
        got = tool.position_blocks(Qt, Kt, rt, scale, p, perm_q=torch.from_numpy(perm_q),
                                   perm_k=torch.from_numpy(perm_k)).numpy()
        assert np.array_equal(got, ref)
        m = tool.metrics(torch.from_numpy(ref), Pt, torch.from_numpy(orc))
        assert abs(m["density"] - ident.density(ref)) < 1e-12
        assert abs(m["recall"] - ident.recall(ref, P)) < 1e-12
        assert abs(m["miss_rate"] - ident.critical_miss_rate(ref, orc)) < 1e-12
        assert abs(m["waste"] - ident.waste(ref, orc)) < 1e-12
