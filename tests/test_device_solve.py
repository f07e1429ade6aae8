"""Device triangular solve (lbk_solve) vs the reference's host solve.

solve(f, b) runs on the device while the factors produced by factorize are
still resident (factorize.py:451-457 semantics: x = U^-1 L^-1 b[perm_global]
on the exported blocks).  Bar: same solution as the host solve within 1e-10
relative, and ||Ax - b||/||b|| no worse than the host solve's (x10 slack for
the different summation order, floor 1e-14).
"""

import numpy as np
import pytest

import paper_2512_04389_b200 as M
from conftest import load_small
from paper_2512_04389_b200 import generators as G
from paper_2512_04389_b200.matrix_io import generate
from paper_2512_04389_b200.numeric import solve_host

pytestmark = pytest.mark.gpu


def pipeline(a, bs=None):
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    pl = (M.irregular_plan(M.percentage_curve(M.diag_block_pointer(f)), a.n) if bs is None
          else M.regular_plan(a.n, bs))
    g = M.partition(f, a, pl)
    return g, M.dependency_levels(g)


CASES = {
    "C1": (lambda: G.poisson2d(64), None, {}),
    "C1_reg200": (lambda: G.poisson2d(64), 200, {}),
    "p3d16": (lambda: G.poisson3d(16, "nd"), None, {}),
    "bbd20k": (lambda: G.bbd(20000, 400, 20, seed=1), None, {}),
    "arrow": (lambda: generate("arrowhead", 1000, b=100), None, {}),
    "randspd": (lambda: generate("random_spd", 3000, bandwidth=20, density=0.3), None, {}),
    "p3d12_csc": (lambda: G.poisson3d(12, "nd"), None, {"dense_threshold": None}),
    # banded diagonal blocks solved per segment (solve_band_kernel), bodies longer than one
    # 1,024-row staging chunk, and one 2,500-row segment per block
    "bbd_bigbody": (lambda: G.bbd(30000, 600, 10, seed=2), None, {}),
    "tridiag_reg": (lambda: generate("tridiagonal", 5000), 2500, {}),
}


def check(a, lu, b):
    xd = M.solve(lu, b)
    xh = solve_host(lu, b)
    A = a.to_scipy()
    rd = float(np.linalg.norm(A @ xd - b) / np.linalg.norm(b))
    rh = float(np.linalg.norm(A @ xh - b) / np.linalg.norm(b))
    assert np.linalg.norm(xd - xh) <= 1e-10 * np.linalg.norm(xh), (rd, rh)
    assert rd <= max(10 * rh, 1e-14), (rd, rh)
    return rd


@pytest.mark.parametrize("name", sorted(CASES))
def test_device_solve_matches_host(name):
    mk, bs, kw = CASES[name]
    a = mk()
    g, t = pipeline(a, bs)
    lu = M.factorize(g, t, **kw)
    assert lu._device is not None
    rng = np.random.default_rng(3)
    check(a, lu, a.to_scipy() @ np.ones(a.n))
    check(a, lu, rng.standard_normal(a.n))


@pytest.mark.parametrize("idx", [14, 15, 16, 18, 21])
def test_device_solve_with_pivot_swaps(idx):
    """Golden small cases whose diagonal blocks pivot (dense-scratch re-run):
    the solve must apply perm_global and the unpermuted-L quirk like the host."""
    d = load_small(idx)
    a = M.CscMatrix(int(d["n"]), d["a_col_ptr"], d["a_row_idx"], d["a_values"])
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    g = M.partition(f, a, M.BlockingPlan(a.n, np.asarray(d["positions"], np.int64), "given"))
    t = M.dependency_levels(g)
    sp = float(d["static_pivot"][0])
    lu = M.factorize(g, t, static_pivot=None if np.isnan(sp) else sp)
    b = np.arange(1, a.n + 1, dtype=np.float64)
    xd = M.solve(lu, b)
    xh = solve_host(lu, b)
    np.testing.assert_allclose(xd, xh, rtol=1e-9, atol=1e-12 * np.abs(xh).max())


def test_stale_factors_fall_back_to_host():
    a = G.poisson2d(24)
    g, t = pipeline(a)
    lu1 = M.factorize(g, t)
    eng, gen = lu1._device
    lu2 = M.factorize(g, t)  # same cached engine: lu1's device copy is overwritten
    assert lu2._device[0] is eng and eng.generation != gen
    b = a.to_scipy() @ np.ones(a.n)
    np.testing.assert_allclose(M.solve(lu1, b), solve_host(lu1, b), rtol=0, atol=0)
    check(a, lu2, b)


@pytest.mark.parametrize("name", ["p3d16", "bbd20k"])
def test_streamed_output_matches_plain_download(name):
    """lbk_factorize_host with a pinned output buffer copies each block to the host
    as soon as its level finishes; the result must equal the plain download."""
    from paper_2512_04389_b200.numeric import Engine, pinned_empty

    mk, bs, kw = CASES[name]
    a = mk()
    g, t = pipeline(a, bs)
    eng = Engine(g, t)
    vin = pinned_empty(eng.nnz)
    vin[:] = eng.pool.values
    plain = np.empty(eng.nnz)
    streamed = pinned_empty(eng.nnz)
    streamed[:] = np.nan
    perms = np.empty(max(eng.n_diag_rows, 1), np.int32)
    assert eng.run_host(vin, plain, perms).code == 0
    for _ in range(2):  # second call reuses the cached streamed graph
        assert eng.run_host(vin, streamed, perms).code == 0
        assert np.asarray(streamed).tobytes() == plain.tobytes()
    eng.close()


def test_refactor_from_matrix_values():
    """lbk_refactor_host: A's own values in (bound pool positions) == the pooled path;
    new values on the same pattern give the factors of the new matrix."""
    from paper_2512_04389_b200.grid import pool_positions
    from paper_2512_04389_b200.numeric import Engine, pinned_empty

    a = G.poisson3d(12, "nd")
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    plan = M.irregular_plan(M.percentage_curve(M.diag_block_pointer(f)), a.n)
    g = M.partition(f, a, plan)
    t = M.dependency_levels(g)
    eng = Engine(g, t)
    eng.bind_matrix(pool_positions(f, a, plan))
    perms = np.empty(max(eng.n_diag_rows, 1), np.int32)
    plain = np.empty(eng.nnz)
    assert eng.run_host(np.ascontiguousarray(g.pool.values), plain, perms).code == 0
    out = pinned_empty(eng.nnz)
    assert eng.refactor_host(np.ascontiguousarray(a.values), out, perms).code == 0
    assert np.asarray(out).tobytes() == plain.tobytes()
    # new values, same pattern
    a2 = M.CscMatrix(a.n, a.col_ptr, a.row_idx, a.values * 1.5 + (a.row_idx == np.repeat(
        np.arange(a.n), np.diff(a.col_ptr))) * 0.25)
    g2 = M.partition(f, a2, plan)
    assert eng.refactor_host(np.ascontiguousarray(a2.values), out, perms).code == 0
    ref = np.empty(eng.nnz)
    assert eng.run_host(np.ascontiguousarray(g2.pool.values), ref, perms).code == 0
    assert np.asarray(out).tobytes() == ref.tobytes()
    eng.close()
