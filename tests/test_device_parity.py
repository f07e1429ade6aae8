"""GPU parity: the sm_100a engine vs the reference's own outputs and the oracle.

Bar (BASELINE.json north_star): identical L/U structure and block
boundaries, values within 1e-10 relative in FP64, ||Ax-b||/||b|| no worse
than the reference's.  GETRF/GESSM/TSTRF reproduce the reference's operation
order with separately rounded mul/sub, so the remaining difference is the
SSSSM summation order (the reference's dgemm order is itself unpinned).
"""

import json
import os

import numpy as np
import pytest

import paper_2512_04389_b200 as M
from conftest import GOLDEN, SMALL_IDS, load_small
from oracle import numeric as ON
from oracle import structure as OS
from paper_2512_04389_b200 import generators as G
from paper_2512_04389_b200.matrix_io import generate

pytestmark = pytest.mark.gpu
CASES = json.load(open(os.path.join(GOLDEN, "cases.json")))


def grid_tree(a, positions):
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    g = M.partition(f, a, M.BlockingPlan(a.n, np.asarray(positions, np.int64), "given"))
    return g, M.dependency_levels(g)


def stacked(blocks, keys):
    return (np.concatenate([blocks[k].col_ptr for k in keys]), np.concatenate([blocks[k].row_idx for k in keys]),
            np.concatenate([blocks[k].values for k in keys]))


@pytest.mark.parametrize("dt", [0.1, None], ids=["dmma", "csc"])
@pytest.mark.parametrize("idx", SMALL_IDS)
def test_small_cases_vs_reference(idx, dt):
    """dt=None: every block stays CSC, so the sparse kernels (ssssm/gessm/tstrf/getrf_item,
    lbk_sparse.cuh) run every task."""
    d = load_small(idx)
    n = int(d["n"])
    a = M.CscMatrix(n, d["a_col_ptr"], d["a_row_idx"], d["a_values"]).check()
    g, t = grid_tree(a, d["positions"])
    sp_ = float(d["static_pivot"][0])
    sp_ = None if np.isnan(sp_) else sp_
    zp = d["zero_pivot"].tolist()
    if zp != [-1, -1]:
        with pytest.raises(M.ZeroPivot) as ei:
            M.factorize(g, t, static_pivot=sp_, dense_threshold=dt)
        assert [ei.value.block, ei.value.col] == zp
        return
    f = M.factorize(g, t, static_pivot=sp_, dense_threshold=dt)
    assert np.array_equal(f.perm_global(), d["perm_global"])
    amax = max(np.abs(d["a_values"]).max(), 1.0)
    for tag, blocks in (("L", f.l_blocks), ("U", f.u_blocks)):
        keys = sorted(blocks)
        assert np.array_equal(np.array(keys).reshape(-1, 2), d[tag + "_keys"])
        cp, ri, vv = stacked(blocks, keys)
        assert np.array_equal(cp, d[tag + "_col_ptr"]) and np.array_equal(ri, d[tag + "_row_idx"])
        np.testing.assert_allclose(vv, d[tag + "_values"], rtol=0, atol=1e-12 * amax)
    r = M.residual(a, f)
    assert r <= float(d["residual"][0]) * 1.5 + 1e-14


NAMED = {
    "C1": (lambda: G.poisson2d(64), None),
    "C1_reg200": (lambda: G.poisson2d(64), 200),
    "C1_reg500": (lambda: G.poisson2d(64), 500),
    "arrow1000": (lambda: generate("arrowhead", 1000, b=100), None),
    "tridiag2000": (lambda: generate("tridiagonal", 2000), None),
    "randspd3000": (lambda: generate("random_spd", 3000, bandwidth=20, density=0.3), None),
    "poisson3d16nd": (lambda: G.poisson3d(16, "nd"), None),
    "bbd20k": (lambda: G.bbd(20000, 400, 20, seed=1), None),
    "bbd20k_reg500": (lambda: G.bbd(20000, 400, 20, seed=1), 500),
}


def pipeline(a, bs=None):
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    c = M.percentage_curve(M.diag_block_pointer(f))
    pl = M.irregular_plan(c, a.n) if bs is None else M.regular_plan(a.n, bs)
    g = M.partition(f, a, pl)
    return g, M.dependency_levels(g)


_ORACLE = {}


def oracle_export(name, a, g, t):
    """Every factor value of the oracle's serial run on the same grid (pinned to the reference in
    tests/test_oracle_golden.py), cached per case."""
    if name not in _ORACLE:
        og = OS.Grid(a.n, g.p, g.plan.positions, g.blocks, g.block_nnz, g.value_max)
        state, _ = ON.factorize(og, t)
        _ORACLE[name] = ON.export(state)
    return _ORACLE[name]


@pytest.mark.parametrize("dt", [0.1, None], ids=["dmma", "csc"])
@pytest.mark.parametrize("name", sorted(NAMED))
def test_named_cases_vs_reference(name, dt):
    rec = CASES[name]
    mk, bs = NAMED[name]
    a = mk()
    g, t = pipeline(a, bs)
    f = M.factorize(g, t, dense_threshold=dt)
    z = np.load(os.path.join(GOLDEN, f"case_{name}.npz"))
    amax = float(np.abs(a.values).max())
    for tag, blocks in (("L", f.l_blocks), ("U", f.u_blocks)):
        keys = z[tag + "_samples_key"]
        got = np.array([blocks[(int(bi), int(bj))].values[int(e)] for bi, bj, e in keys])
        want = z[tag + "_samples_val"]
        np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-10 * amax)
        bk = z[tag + "_blocks_key"]
        nnz = np.array([blocks[(int(bi), int(bj))].nnz for bi, bj, _ in bk])
        assert np.array_equal(nnz, bk[:, 2])  # identical exported structure per block
        sums = np.array([np.abs(blocks[(int(bi), int(bj))].values).sum() for bi, bj, _ in bk])
        np.testing.assert_allclose(sums, z[tag + "_blocks_abssum"], rtol=1e-10)
        if tag + "_blocks_proj" in z:  # a +-1 projection of every value of the reference's block
            w = [np.where(((np.arange(len(blocks[(int(bi), int(bj))].values), dtype=np.uint64)
                            * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(40)) & np.uint64(1), 1.0, -1.0)
                 for bi, bj, _ in bk]
            proj = np.array([np.dot(wq, blocks[(int(bi), int(bj))].values) for wq, (bi, bj, _) in zip(w, bk)])
            np.testing.assert_allclose(proj, z[tag + "_blocks_proj"], rtol=1e-9, atol=1e-10 * amax)
    # all values against the oracle's run on the same grid
    lb, ub = oracle_export(name, a, g, t)
    for blocks, ob in ((f.l_blocks, lb), (f.u_blocks, ub)):
        assert set(blocks) == set(ob)
        for k, want in ob.items():
            got = blocks[k]
            assert np.array_equal(got.row_idx, want.row_idx) and np.array_equal(got.col_ptr, want.col_ptr), k
            scale = max(float(np.abs(want.values).max(initial=0.0)), 1e-3 * amax)
            assert float(np.abs(got.values - want.values).max(initial=0.0)) <= 1e-10 * scale, k
    b = a.to_scipy() @ np.ones(a.n)
    x = M.solve(f, b)
    relres = float(np.linalg.norm(a.to_scipy() @ x - b) / np.linalg.norm(b))
    assert relres <= max(2 * rec["relres"], 1e-15), (relres, rec["relres"])
    assert M.residual(a, f) <= max(2 * rec["residual"], 1e-15)


def test_deterministic_bits():
    a = G.poisson3d(16, "nd")
    g, t = pipeline(a)
    f1 = M.factorize(g, t)
    f2 = M.factorize(g, t)
    for k in f1.l_blocks:
        assert f1.l_blocks[k].values.tobytes() == f2.l_blocks[k].values.tobytes()
    for k in f1.u_blocks:
        assert f1.u_blocks[k].values.tobytes() == f2.u_blocks[k].values.tobytes()


def test_oracle_agreement_random():
    """Random patterns and plans (incl. single-block and scalar blocking) vs the CPU oracle."""
    rng = np.random.default_rng(5)
    from oracle import brute
    for trial in range(12):
        n = int(rng.integers(3, 60))
        pat = brute.random_symmetric_pattern(n, rng, fill=float(rng.uniform(0.03, 0.35)))
        r, c, v = brute.pattern_triplets(n, pat, rng)
        a = M.csc_from_triplets(n, (r, c, v))
        bs = [1, 2, max(1, n // 3), n][trial % 4]
        g, t = grid_tree(a, M.regular_plan(n, bs).positions)
        f = M.factorize(g, t)
        og = OS.partition(n, *OS.symbolic(OS.symmetrize(OS.Csc(n, a.col_ptr, a.row_idx, a.values))),
                          OS.Csc(n, a.col_ptr, a.row_idx, a.values), g.plan.positions)
        state, perms = ON.factorize(og, OS.levels(og))
        lb, ub = ON.export(state)
        for blocks, ob in ((f.l_blocks, lb), (f.u_blocks, ub)):
            assert set(blocks) == set(ob)
            for k in ob:
                assert np.array_equal(blocks[k].row_idx, ob[k].row_idx)
                np.testing.assert_allclose(blocks[k].values, ob[k].values, rtol=0, atol=1e-13 * np.abs(v).max())


def test_kernel_level_entries_match_oracle():
    rng = np.random.default_rng(3)
    m = 13
    d = rng.uniform(-1, 1, (m, m)) + np.diag(rng.uniform(3, 5, m))
    lo, up, perm = M.factor_diagonal(d)
    w = d.copy()
    operm, _ = ON.getrf(w)
    assert np.array_equal(perm, operm)
    np.testing.assert_array_equal(up, np.triu(w))  # same op order -> same bits
    np.testing.assert_array_equal(lo, np.tril(w, -1) + np.eye(m))
    # pivoting block: swaps happen on device in full-rectangle storage
    dp = rng.uniform(-1, 1, (m, m))
    lo2, up2, perm2 = M.factor_diagonal(dp)
    w2 = dp.copy()
    operm2, swapped = ON.getrf(w2)
    assert swapped and np.array_equal(perm2, operm2)
    np.testing.assert_allclose(up2, np.triu(w2), rtol=0, atol=1e-13)
    x = rng.uniform(-1, 1, (m, 7))
    got = M.factor_u_panel(lo2, perm2, x)
    want = x[perm2].copy()
    ON.gessm(lo2, want)
    np.testing.assert_array_equal(got, want)
    y = rng.uniform(-1, 1, (5, m))
    got = M.factor_l_panel(y, up)
    want = y.copy()
    ON.tstrf(want, up)
    np.testing.assert_array_equal(got, want)
    lk = rng.uniform(-1, 1, (6, m))
    uj = rng.uniform(-1, 1, (m, 9))
    bk = rng.uniform(-1, 1, (6, 9))
    np.testing.assert_allclose(M.schur_update(bk, lk, uj), bk - lk @ uj, rtol=0, atol=1e-13)
    with pytest.raises(M.ZeroPivot):
        M.factor_diagonal(np.zeros((3, 3)), block_index=4)


def test_static_pivot_and_zero_pivot_lowest_block():
    n = 40
    a = generate("tridiagonal", n)
    vals = a.values.copy()
    cols = np.repeat(np.arange(n), np.diff(a.col_ptr))
    # zero out two diagonal entries' columns in different blocks -> lowest block wins
    for col in (25, 12):
        vals[(cols == col)] = 0.0
    a2 = M.CscMatrix(n, a.col_ptr, a.row_idx, vals)
    g, t = grid_tree(a2, M.regular_plan(n, 5).positions)
    with pytest.raises(M.ZeroPivot) as ei:
        M.factorize(g, t)
    assert (ei.value.block, ei.value.col) == (2, 2)
    f = M.factorize(g, t, static_pivot=1e-8)
    og = OS.partition(n, *OS.symbolic(OS.symmetrize(OS.Csc(n, a2.col_ptr, a2.row_idx, a2.values))),
                      OS.Csc(n, a2.col_ptr, a2.row_idx, a2.values), g.plan.positions)
    state, _ = ON.factorize(og, OS.levels(og), static_pivot=1e-8)
    lb, ub = ON.export(state)
    for k in ub:
        np.testing.assert_allclose(f.u_blocks[k].values, ub[k].values, rtol=1e-12, atol=0)


@pytest.mark.slow
def test_c2_full_size_properties():
    """C2 (3D Poisson 64^3, ND): structure == reference golden, solve residual gate."""
    rec = CASES.get("C2")
    a = G.poisson3d(64, "nd")
    g, t = pipeline(a)
    if rec:
        assert t.task_count == rec["tasks"] and g.p == rec["p"]
    f = M.factorize(g, t)
    b = a.to_scipy() @ np.ones(a.n)
    x = M.solve(f, b)
    relres = float(np.linalg.norm(a.to_scipy() @ x - b) / np.linalg.norm(b))
    assert relres < 1e-12


@pytest.mark.parametrize("kind,n,bs", [("dense", 300, 150), ("random_spd", 2400, 400), ("arrowhead", 1500, 500)])
def test_large_blocks_tile_dag_vs_oracle(kind, n, bs):
    """Diagonal blocks of several 64-tiles and compressed panels: tile-DAG executor
    (tiled GETRF with verified no-swap speculation, panel solves, DMMA SSSSM)."""
    kw = {"random_spd": {"bandwidth": 60, "density": 0.3}, "arrowhead": {"b": 200}}.get(kind, {})
    a = generate(kind, n, **kw)
    g, t = grid_tree(a, M.regular_plan(n, bs).positions)
    f = M.factorize(g, t)
    oa = OS.Csc(n, a.col_ptr, a.row_idx, a.values)
    og = OS.partition(n, *OS.symbolic(OS.symmetrize(oa)), oa, g.plan.positions)
    state, perms = ON.factorize(og, OS.levels(og))
    lb, ub = ON.export(state)
    amax = np.abs(a.values).max()
    for blocks, ob in ((f.l_blocks, lb), (f.u_blocks, ub)):
        assert set(blocks) == set(ob)
        for k in ob:
            assert np.array_equal(blocks[k].row_idx, ob[k].row_idx), k
            np.testing.assert_allclose(blocks[k].values, ob[k].values, rtol=0, atol=1e-11 * amax)


@pytest.mark.parametrize("n,border,bodies,seed", [(20000, 400, 20, 1), (30000, 600, 40, 2), (12000, 480, 8, 3)])
def test_segment_refined_schedule_is_bitwise_identical(n, border, bodies, seed):
    """Segment-refined levels (lbk_plan flags bit 2: banded diagonal blocks swept per body,
    updates / panels waiting only for the segments they touch) reorder launches, never the
    per-entry operations: the factors equal the block-level schedule's bit for bit."""
    from paper_2512_04389_b200.numeric import Engine

    a = G.bbd(n, border, bodies, seed=seed)
    g, t = pipeline(a)
    out = []
    for refine in (True, False):
        e = Engine(g, t, refine=refine)
        e.upload()
        e.run_device()
        out.append((e.download(), e.n_launch_levels))
        e.close()
    (v1, p1), l1 = out[0]
    (v0, p0), l0 = out[1]
    assert v1.tobytes() == v0.tobytes() and p1.tobytes() == p0.tobytes()
    print(f"launch levels: refined {l1}, block-level {l0}")


@pytest.mark.parametrize("n,bs", [(16, None), (16, 1024), (20, 2000)])
def test_subtree_aligned_tiles_vs_uniform_and_oracle(monkeypatch, n, bs):
    """Executor tiling (lbk_device.cu subtree_tiles / tile_cp_model): diagonal blocks tiled along
    their elimination subtrees and panel chains cut at the same subtree regions give the same
    factors as uniform 64-column tiles (LBK_UNIFORM_TILES=1) within the FP64 tolerance, every
    value checked against the oracle; the task DAGs differ (the aligned tiling was chosen)."""
    from paper_2512_04389_b200.numeric import Engine

    a = G.poisson3d(n, "nd")
    g, t = pipeline(a, bs)
    res = {}
    for mode in ("uniform", "aligned"):  # (the drop-in factorize below then plans aligned tiles)
        if mode == "uniform":
            monkeypatch.setenv("LBK_UNIFORM_TILES", "1")
        else:
            monkeypatch.delenv("LBK_UNIFORM_TILES", raising=False)
        e = Engine(g, t)
        e.upload()
        e.run_device()
        vals, perms = e.download()
        e.run_device()
        assert e.download()[0].tobytes() == vals.tobytes()  # deterministic under either tiling
        _, info = e.exec_trace()
        res[mode] = (vals, perms, info)
        e.close()
    (va, pa, ia), (vu, pu, iu) = res["aligned"], res["uniform"]
    assert np.array_equal(pa, pu)
    amax = np.abs(a.values).max()
    np.testing.assert_allclose(va, vu, rtol=0, atol=1e-11 * amax)
    if bs is not None:  # blocks of several subtrees: the aligned tiling differs from the uniform one
        assert len(ia) != len(iu) or not np.array_equal(ia, iu)
    f = M.factorize(g, t)
    oa = OS.Csc(a.n, a.col_ptr, a.row_idx, a.values)
    og = OS.partition(a.n, *OS.symbolic(OS.symmetrize(oa)), oa, g.plan.positions)
    state, _ = ON.factorize(og, OS.levels(og))
    lb, ub = ON.export(state)
    for blocks, ob in ((f.l_blocks, lb), (f.u_blocks, ub)):
        assert set(blocks) == set(ob)
        for k in ob:
            np.testing.assert_allclose(blocks[k].values, ob[k].values, rtol=0, atol=1e-11 * amax)


@pytest.mark.parametrize("kind", ["p3d", "bbd", "dense"])
def test_aggregated_panel_updates_are_bitwise_identical(monkeypatch, kind):
    """Panel tile updates from consecutive steps aggregated into one executor task
    (LBK_PANEL_AGG, default 4; XTask::pad1) apply the same operations in the same order as
    one task per step (LBK_PANEL_AGG=1): the factors are equal bit for bit."""
    from paper_2512_04389_b200.numeric import Engine

    if kind == "p3d":
        a = G.poisson3d(16, "nd")
        g, t = pipeline(a, 1024)
    elif kind == "bbd":
        a = G.bbd(20000, 800, 10, seed=5)
        g, t = pipeline(a)
    else:
        a = generate("dense", 900)
        g, t = grid_tree(a, M.regular_plan(900, 450).positions)
    out, ntasks = [], []
    for agg in ("1", "4"):
        monkeypatch.setenv("LBK_PANEL_AGG", agg)
        e = Engine(g, t)
        e.upload()
        e.run_device()
        out.append(e.download())
        ntasks.append(len(e.exec_trace()[1]))
        e.close()
    assert out[0][0].tobytes() == out[1][0].tobytes() and out[0][1].tobytes() == out[1][1].tobytes()
    if kind == "dense":  # dense panels: updates from consecutive steps were actually aggregated
        assert ntasks[1] < ntasks[0], ntasks
