"""The drop-in against the UNMODIFIED reference, value for value.

Grids and trees are built by the reference itself (``lublock.partition`` /
``lublock.dependency_levels``, pkg/src/lublock/grid.py:85-148, 223-378, from
baseline/_ref, pip-installed by paper_2512_04389_b200.build) and handed
straight to this package's ``factorize`` — the reference's own objects crossing
the boundary, as INTEGRATION.md advertises.  The result is compared with
``lublock.factorize`` on the same objects (factorize.py:245-384): identical
block keys and L/U structure per block, perms equal, every value within 1e-10
of the block's scale, ZeroPivot at the same (block, column), residual and solve
no worse.  Sizes are those the reference factors in seconds.
"""

import numpy as np
import pytest

import paper_2512_04389_b200 as M
from oracle import ref_timing as RT

pytestmark = pytest.mark.gpu

try:
    L = RT.import_reference()
except ImportError:  # pragma: no cover - the reference install travels with the repo snapshot
    L = None


def ref_objects(family, size, seed=0, values=None, plan=None):
    n, r, c, v = RT.family_triplets(family, size, seed)
    a = L.csc_from_triplets(n, (r, c, v))
    if values is not None:
        a = L.CscMatrix(a.n, a.col_ptr, a.row_idx, values(a))
    filled = L.symbolic_factorize(L.symmetrize_pattern(a))
    if plan is None:
        pl = L.irregular_plan(L.percentage_curve(L.diag_block_pointer(filled)), a.n)
    else:
        pl = L.regular_plan(a.n, plan)
    grid = L.partition(filled, a, pl)
    return a, grid, L.dependency_levels(grid)


def compare(ref, ours, scale):
    assert set(ours.l_blocks) == set(ref.l_blocks) and set(ours.u_blocks) == set(ref.u_blocks)
    for i in range(len(ref.perms)):
        assert np.array_equal(np.asarray(ours.perms[i]), np.asarray(ref.perms[i])), i
    worst = 0.0
    for got_d, want_d in ((ours.l_blocks, ref.l_blocks), (ours.u_blocks, ref.u_blocks)):
        for k, want in want_d.items():
            got = got_d[k]
            assert np.array_equal(got.col_ptr, want.col_ptr) and np.array_equal(got.row_idx, want.row_idx), k
            s = max(float(np.abs(want.values).max(initial=0.0)), scale)
            err = float(np.abs(got.values - want.values).max(initial=0.0))
            assert err <= 1e-10 * s, (k, err, s)
            worst = max(worst, err / s)
    return worst


CASES = [
    ("poisson2d", 48, None),
    ("poisson3d", 12, None),
    ("poisson3d", 16, None),
    ("bbd", 20000, None),
    ("bbd2", 25000, None),
    ("poisson2d", 40, 300),
]


@pytest.mark.skipif(L is None, reason="baseline/_ref (the reference install) is not present")
@pytest.mark.parametrize("family,size,plan", CASES)
def test_reference_built_grid_all_values(family, size, plan):
    a, grid, tree = ref_objects(family, size, plan=plan)
    ref = L.factorize(grid, tree, workers=1)
    ours = M.factorize(grid, tree)
    compare(ref, ours, 1e-3 * float(np.abs(a.values).max()))
    assert M.residual(a, ours) <= max(2 * L.residual(a, ref), 1e-15)
    b = a.to_scipy() @ np.ones(a.n)
    x_ref = L.solve(ref, b)
    x = M.solve(ours, b)
    rr = np.linalg.norm(a.to_scipy() @ x_ref - b) / np.linalg.norm(b)
    r = np.linalg.norm(a.to_scipy() @ x - b) / np.linalg.norm(b)
    assert r <= max(2 * rr, 1e-15), (r, rr)


@pytest.mark.skipif(L is None, reason="baseline/_ref (the reference install) is not present")
def test_dense_blas_flag_matches_reference_lapack_path():
    """dense_blas=True (LAPACK getrf / trsm on >= 50 % dense blocks, factorize.py:271-275, 331-343):
    same factors within rounding as the reference's own dense_blas run."""
    a, grid, tree = ref_objects("poisson2d", 24, plan=48)
    ref = L.factorize(grid, tree, dense_blas=True)
    ours = M.factorize(grid, tree, dense_blas=True)
    compare(ref, ours, 1e-3 * float(np.abs(a.values).max()))


@pytest.mark.skipif(L is None, reason="baseline/_ref (the reference install) is not present")
def test_reference_built_grid_with_row_swaps():
    """Non-dominant values: block-local pivoting swaps rows (the reference's quirk of
    leaving L blocks unpermuted, factorize.py:326-331, reproduced)."""
    rng = np.random.default_rng(7)
    a, grid, tree = ref_objects("poisson2d", 20, values=lambda a: rng.uniform(-1.0, 1.0, a.nnz), plan=50)
    ref = L.factorize(grid, tree)
    assert any(not np.array_equal(p, np.arange(len(p))) for p in ref.perms)
    ours = M.factorize(grid, tree)
    compare(ref, ours, 1e-3)


@pytest.mark.skipif(L is None, reason="baseline/_ref (the reference install) is not present")
def test_reference_built_grid_zero_pivot_and_static_pivot():
    def zero_col(a):
        v = np.array(a.values, dtype=np.float64)
        cols = np.repeat(np.arange(a.n), np.diff(a.col_ptr))
        v[cols == 37] = 0.0
        return v

    a, grid, tree = ref_objects("poisson2d", 16, values=zero_col, plan=32)
    with pytest.raises(L.ZeroPivot) as want:
        L.factorize(grid, tree)
    with pytest.raises(M.ZeroPivot) as got:
        M.factorize(grid, tree)
    assert (got.value.block, got.value.col) == (want.value.block, want.value.col)
    # dense_blas=True: the reference's LAPACK path (factorize.py:81-95) checks the same |u_kk| against
    # tol * colmax-at-entry after the fact and raises the lowest failing column
    with pytest.raises(L.ZeroPivot) as want_b:
        L.factorize(grid, tree, dense_blas=True)
    with pytest.raises(M.ZeroPivot) as got_b:
        M.factorize(grid, tree, dense_blas=True)
    assert (got_b.value.block, got_b.value.col) == (want_b.value.block, want_b.value.col)
    ref = L.factorize(grid, tree, static_pivot=1e-8)
    ours = M.factorize(grid, tree, static_pivot=1e-8)
    compare(ref, ours, 1e-3)
