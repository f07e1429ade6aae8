"""Product host structure path == reference, bit for bit (golden fixtures + oracle)."""

import ctypes
import hashlib
import json
import os
import re

import numpy as np
import pytest

import paper_2512_04389_b200 as M
from conftest import GOLDEN, REPO, SMALL_IDS, load_small
from oracle import structure as S
from paper_2512_04389_b200 import _native, generators as G
from paper_2512_04389_b200.matrix_io import generate

CASES = json.load(open(os.path.join(GOLDEN, "cases.json")))
SPEC = json.load(open(os.path.join(GOLDEN, "spec.json")))


def sha(a):
    a = np.ascontiguousarray(a)
    if a.dtype.kind in "iu":
        a = a.astype(np.int64)
    return hashlib.sha256(a.tobytes()).hexdigest()


MAKERS = {
    "C1": (lambda: G.poisson2d(64), None),
    "C1_reg200": (lambda: G.poisson2d(64), 200),
    "C1_reg500": (lambda: G.poisson2d(64), 500),
    "arrow1000": (lambda: generate("arrowhead", 1000, b=100), None),
    "tridiag2000": (lambda: generate("tridiagonal", 2000), None),
    "randspd3000": (lambda: generate("random_spd", 3000, bandwidth=20, density=0.3), None),
    "poisson3d16nd": (lambda: G.poisson3d(16, "nd"), None),
    "bbd20k": (lambda: G.bbd(20000, 400, 20, seed=1), None),
    "bbd20k_reg500": (lambda: G.bbd(20000, 400, 20, seed=1), 500),
    # full BASELINE configs (records: make_golden.py --c2 / --c3 / --c5, the reference run here)
    "C2": (G.CONFIGS["C2"], None),
    "C3": (G.CONFIGS["C3"], None),
    "C5": (G.CONFIGS["C5"], None),
}


def structure(a, bs=None):
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    bp = M.diag_block_pointer(f)
    c = M.percentage_curve(bp)
    pl = M.irregular_plan(c, a.n) if bs is None else M.regular_plan(a.n, bs)
    g = M.partition(f, a, pl)
    return f, bp, c, pl, g, M.dependency_levels(g)


@pytest.mark.parametrize("name", sorted(MAKERS))
def test_case_structure_matches_reference(name):
    if name not in CASES:
        pytest.skip(f"no reference record for {name}")
    rec = CASES[name]
    mk, bs = MAKERS[name]
    a = mk()
    assert [sha(a.col_ptr), sha(a.row_idx), sha(a.values)] == rec["a_sha"]
    f, bp, c, pl, g, t = structure(a, bs)
    assert f.nnz_filled == rec["nnz_filled"] and pl.p == rec["p"]
    assert sha(f.col_ptr) == rec["filled_col_ptr"] and sha(f.row_idx) == rec["filled_row_idx"]
    assert sha(bp.blockptr) == rec["blockptr"] and sha(c.pct) == rec["pct"]
    assert sha(pl.positions) == rec["positions"]
    keys = list(g.blocks)
    assert sha(np.array(keys, dtype=np.int64).ravel()) == rec["block_keys"]
    assert sha(np.concatenate([g.blocks[k].col_ptr for k in keys])) == rec["block_col_ptr"]
    assert sha(np.concatenate([g.blocks[k].row_idx for k in keys])) == rec["block_row_idx"]
    assert sha(np.concatenate([g.blocks[k].values for k in keys])) == rec["block_values"]
    assert sha(g.block_nnz) == rec["block_nnz"] and g.value_max == rec["value_max"]
    for fld in ("kinds", "steps", "rows", "cols", "weights", "costs", "levels_of", "pred_ptr", "pred_idx"):
        assert sha(getattr(t, fld)) == rec["tree_" + fld], fld
    assert t.task_count == rec["tasks"] and t.n_levels == rec["levels"]


@pytest.mark.parametrize("idx", SMALL_IDS)
def test_small_structure_matches_reference(idx):
    d = load_small(idx)
    n = int(d["n"])
    a = M.CscMatrix(n, d["a_col_ptr"], d["a_row_idx"], d["a_values"]).check()
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    assert np.array_equal(f.col_ptr, d["filled_col_ptr"]) and np.array_equal(f.row_idx, d["filled_row_idx"])
    assert np.array_equal(M.diag_block_pointer(f).blockptr, d["blockptr"])
    g = M.partition(f, a, M.BlockingPlan(n, d["positions"], "given"))
    t = M.dependency_levels(g)
    for fld in ("kinds", "steps", "rows", "cols", "weights", "costs", "levels_of", "pred_ptr", "pred_idx"):
        x = getattr(t, fld)
        assert x.dtype == d["tree_" + fld].dtype and np.array_equal(x, d["tree_" + fld]), fld


def test_spec_plans_and_selector():
    for name in ("ex1", "ex2", "ex3"):
        c = M.PercentCurve(1000, 10, np.array(SPEC[f"curve_{name}"], dtype=np.float64))
        assert M.irregular_plan(c, 1000, 2, 3, 0.2).positions.tolist() == SPEC[f"plan_{name}"]
        assert M.irregular_plan(c, 1000, 2, 3, 0.2, True).positions.tolist() == SPEC[f"plan_{name}_overlap"]
    for key, want in SPEC["regular"].items():
        n, bs = map(int, key.split("_"))
        assert M.regular_plan(n, bs).positions.tolist() == want
    for key, want in SPEC["select"].items():
        n, nnz = map(int, key.split("_"))
        assert M.pangulu_size_select(n, nnz) == want
    assert M.generate("arrowhead", 100, b=10).nnz == SPEC["arrowhead_100_10_nnz"] == 1990


def test_random_patterns_vs_oracle():
    rng = np.random.default_rng(11)
    from oracle import brute
    for _ in range(25):
        n = int(rng.integers(2, 70))
        pat = brute.random_symmetric_pattern(n, rng, fill=float(rng.uniform(0.02, 0.4)))
        r, c, v = brute.pattern_triplets(n, pat, rng)
        a = M.csc_from_triplets(n, (r, c, v))
        (fcp, fri), pct, pos, og, ot = S.pipeline(S.Csc(n, a.col_ptr, a.row_idx, a.values),
                                                   sample_points=int(rng.integers(2, 50)))
        f = M.symbolic_factorize(M.symmetrize_pattern(a))
        assert np.array_equal(f.col_ptr, fcp) and np.array_equal(f.row_idx, fri)
        g = M.partition(f, a, M.BlockingPlan(n, pos, "given"))
        t = M.dependency_levels(g)
        for fld in ("kinds", "levels_of", "pred_ptr", "pred_idx", "costs", "weights"):
            assert np.array_equal(getattr(t, fld), getattr(ot, fld))


def test_errors_follow_reference():
    with pytest.raises(M.BadParams):
        M.regular_plan(10, 0)
    c = M.PercentCurve(10, 10, np.linspace(0, 1, 11))
    with pytest.raises(M.BadParams):
        M.irregular_plan(c, 10, step=0)
    with pytest.raises(M.BadParams):
        M.irregular_plan(c, 10, max_num=0)
    with pytest.raises(M.BadParams):
        M.irregular_plan(c, 10, threshold=1.5)
    with pytest.raises(M.DegenerateCurve):
        M.irregular_plan(M.PercentCurve(10, 10, np.zeros(11)), 10)
    with pytest.raises(M.IndexOutOfRange):
        M.csc_from_triplets(2, [(0, 2, 1.0)])
    with pytest.raises(M.EmptyMatrix):
        M.csc_from_triplets(0, [])
    a = M.csc_from_triplets(3, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0), (2, 0, 1.0)])
    with pytest.raises(M.NotSymmetric):
        M.symbolic_factorize(a)
    with pytest.raises(M.MissingDiagonal):
        M.symbolic_factorize(M.csc_from_triplets(2, [(0, 0, 1.0)]))
    x = M.csc_from_triplets(2, [(1, 0, 4.0), (0, 0, 1.0), (1, 0, -4.0)])
    assert x.nnz == 2 and x.values[1] == 0.0  # explicit zero kept


def test_matrix_market_roundtrip(tmp_path):
    p = tmp_path / "a.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 3\n1 1 2.0\n2 1 5.0\n3 3 1.5\n")
    a = M.read_matrix_market(str(p))
    assert a.col_ptr.tolist() == [0, 2, 3, 4] and a.row_idx.tolist() == [0, 1, 0, 2]
    assert a.values.tolist() == [2.0, 5.0, 5.0, 1.5]
    p.write_text("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n")
    with pytest.raises(M.UnsupportedField):
        M.read_matrix_market(str(p))


def test_host_library_exports_every_declared_symbol():
    hdr = open(os.path.join(REPO, "include", "lbk.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void\s*\*?)\s*(lbk_\w+)\s*\(", hdr, re.M))
    host = ctypes.CDLL(_native.HOST_LIB)
    dev_syms = {s for s in declared if not s.startswith(("lbk_symbolic", "lbk_partition", "lbk_levels",
                                                         "lbk_check", "lbk_blockptr"))}
    for s in declared - dev_syms:
        assert hasattr(host, s), s
    if dev_syms:
        assert os.path.exists(_native.DEV_LIB), "device library not built"
        # the device library links libcudart; loading it needs no GPU
        dev = ctypes.CDLL(_native.DEV_LIB)
        for s in dev_syms:
            assert hasattr(dev, s), s


def test_pool_positions_place_every_entry_of_a():
    """grid.pool_positions (the refactorization input map): the pooled grid values
    are exactly A's values at those positions and zero elsewhere (fill)."""
    from paper_2512_04389_b200 import generators as G
    from paper_2512_04389_b200.grid import pool_positions

    for a in (G.poisson3d(8, "nd"), G.bbd(3000, 60, 10, seed=3)):
        f = M.symbolic_factorize(M.symmetrize_pattern(a))
        plan = M.irregular_plan(M.percentage_curve(M.diag_block_pointer(f)), a.n)
        vals = M.partition(f, a, plan).pool.values
        pmap = pool_positions(f, a, plan)
        assert len(np.unique(pmap)) == a.nnz
        assert np.array_equal(vals[pmap], a.values)
        rest = np.ones(len(vals), bool)
        rest[pmap] = False
        assert not np.any(vals[rest])
