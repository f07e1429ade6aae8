"""Banded diagonal blocks (the executor's X_BAND sweep) vs the CPU oracle.

A diagonal block whose filled pattern stays within a band of <= 15 is
factored by one CTA sweeping the band instead of the 64x64 tile DAG.  The
pivot rule must be the reference's (factorize.py:38-78): ZeroPivot at the
same (block, column), a needed row swap detected (then the dense-scratch
re-run pivots), values within 1e-10.
"""

import numpy as np
import pytest

import paper_2512_04389_b200 as M
from oracle import numeric as ON
from oracle import structure as OS

pytestmark = pytest.mark.gpu


def banded(n, bl, bu, rng, diag_boost=4.0, zero_at=None, weak_at=None, keep=0.7):
    rows, cols, vals = [], [], []
    for c in range(n):
        for r in range(max(0, c - bu), min(n, c + bl + 1)):
            if r == c:
                continue
            if rng.random() < keep:
                rows += [r, c]
                cols += [c, r]
                vals += [rng.uniform(-1, 1), rng.uniform(-1, 1)]
    for k in range(n):
        rows.append(k)
        cols.append(k)
        v = diag_boost * (2 * bl + 2)
        if zero_at is not None and k == zero_at:
            v = 0.0
        if weak_at is not None and k == weak_at:
            v = 1e-3
        vals.append(v)
    return M.csc_from_triplets(n, (np.array(rows), np.array(cols), np.array(vals)))


def run_both(a, positions):
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    g = M.partition(f, a, M.BlockingPlan(a.n, np.asarray(positions, np.int64), "given"))
    t = M.dependency_levels(g)
    oa = OS.Csc(a.n, a.col_ptr, a.row_idx, a.values)
    og = OS.partition(a.n, *OS.symbolic(OS.symmetrize(oa)), oa, np.asarray(positions, np.int64))
    return g, t, og


@pytest.mark.parametrize("bl,bu,n,keep", [(1, 1, 700, 0.7), (4, 4, 1000, 0.7), (15, 15, 900, 0.7), (3, 9, 600, 0.7),
                                          (20, 20, 500, 0.7), (1, 1, 4000, 1.0), (2, 2, 3200, 1.0),
                                          (3, 3, 5000, 1.0), (4, 4, 4500, 1.0)])
def test_band_values_match_oracle(bl, bu, n, keep):
    """keep=1.0: a full band (no independent segments), so blocks longer than one
    shared-memory chunk of the register sweep (~1000-2600 columns) cross chunks."""
    rng = np.random.default_rng(bl * 100 + bu)
    a = banded(n, max(bl, bu), max(bl, bu), rng, keep=keep)
    positions = [0, n // 2, n]  # two banded diagonal blocks of > 128 rows
    g, t, og = run_both(a, positions)
    lu = M.factorize(g, t)
    state, _ = ON.factorize(og, OS.levels(og))
    lb, ub = ON.export(state)
    amax = float(np.abs(a.values).max())
    for got, want in ((lu.l_blocks, lb), (lu.u_blocks, ub)):
        assert set(got) == set(want)
        for k in want:
            assert np.array_equal(got[k].row_idx, want[k].row_idx), k
            np.testing.assert_allclose(got[k].values, want[k].values, rtol=0, atol=1e-10 * amax)


def test_band_zero_pivot_location():
    rng = np.random.default_rng(7)
    n = 600
    a = banded(n, 3, 3, rng, zero_at=None)
    # decouple row and column 417 and zero its diagonal: the column is exactly
    # zero at its elimination step (the symmetrized pattern keeps a 0.0 diagonal)
    d = a.to_scipy().tolil()
    for q in range(n):
        d[417, q] = 0.0
        d[q, 417] = 0.0
    d = d.tocsc()
    a = M.CscMatrix(n, d.indptr.astype(np.int64), d.indices.astype(np.int64), d.data)
    g, t, og = run_both(a, [0, 300, n])
    with pytest.raises(M.ZeroPivot) as ei:
        M.factorize(g, t)
    with pytest.raises(ON.OracleZeroPivot) as eo:
        ON.factorize(og, OS.levels(og))
    assert (ei.value.block, ei.value.col) == (eo.value.block, eo.value.col)


def test_band_needed_swap_reruns_dense():
    rng = np.random.default_rng(11)
    n = 500
    a = banded(n, 2, 2, rng, weak_at=260)  # a weak pivot: a row below dominates -> swap
    g, t, og = run_both(a, [0, 250, n])
    lu = M.factorize(g, t)
    state, perms = ON.factorize(og, OS.levels(og))
    assert any(not np.array_equal(p, np.arange(len(p))) for p in perms)
    lb, ub = ON.export(state)
    amax = float(np.abs(a.values).max())
    for got, want in ((lu.l_blocks, lb), (lu.u_blocks, ub)):
        for k in want:
            assert np.array_equal(got[k].row_idx, want[k].row_idx), k
            np.testing.assert_allclose(got[k].values, want[k].values, rtol=0, atol=1e-9 * amax)


def test_band_independent_segments_match_oracle():
    """A banded diagonal block made of independent bodies (BBD-like): the
    engine factors its segments as separate tasks; values must not change."""
    rng = np.random.default_rng(5)
    n = 1200
    a = banded(n, 4, 4, rng)
    d = a.to_scipy().tolil()
    for s in (150, 333, 334, 700, 1000):  # cut every coupling across these boundaries
        for r in range(max(0, s - 4), s):
            for c in range(s, min(n, s + 4)):
                d[r, c] = 0.0
                d[c, r] = 0.0
    d = d.tocsc()
    a = M.CscMatrix(n, d.indptr.astype(np.int64), d.indices.astype(np.int64), d.data)
    g, t, og = run_both(a, [0, 900, n])
    lu = M.factorize(g, t)
    state, _ = ON.factorize(og, OS.levels(og))
    lb, ub = ON.export(state)
    amax = float(np.abs(a.values).max())
    for got, want in ((lu.l_blocks, lb), (lu.u_blocks, ub)):
        for k in want:
            assert np.array_equal(got[k].row_idx, want[k].row_idx), k
            np.testing.assert_allclose(got[k].values, want[k].values, rtol=0, atol=1e-10 * amax)
