"""Full-size BASELINE configurations on the device, value by value.

* structure: the product's structure path on C2 / C3 / C5 is pinned to the
  reference's own records (tests/golden/cases.json, produced by
  tests/golden/make_golden.py running lublock) in tests/test_structure.py;
  here the same hashes are re-asserted on the grid the device factorizes;
* values, C2 / C3 / C5: every value of every block that is FINAL after the
  oracle's prefix of steps 0..s (oracle.numeric.factorize_prefix, a serial
  restatement of factorize.py:245-384 pinned to the reference in
  tests/test_oracle_golden.py) is compared with the device factors, at the
  north-star tolerance 1e-10 relative (per block: max|d| <= 1e-10 * max(|block|max,
  1e-3 |A|max));
* values, C5 whole: per-block checksums of the reference's own factors
  (lublock.factorize run to completion here: abs-sum, max, a +-1 projection of
  every value, 32 sampled values per block, exported nnz per block);
* solve: ||Ax - b|| / ||b|| with b = A 1 (the north-star gate).
"""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2512_04389_b200 as M
from conftest import GOLDEN
from oracle import numeric as ON
from oracle import structure as OS
from paper_2512_04389_b200 import generators as G

pytestmark = pytest.mark.gpu
CASES = json.load(open(os.path.join(GOLDEN, "cases.json")))
BUDGET_S = float(os.environ.get("LBK_ORACLE_BUDGET_S", "45"))


def sha(a):
    a = np.ascontiguousarray(a)
    if a.dtype.kind in "iu":
        a = a.astype(np.int64)
    return hashlib.sha256(a.tobytes()).hexdigest()


def pipeline(a):
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    pl = M.irregular_plan(M.percentage_curve(M.diag_block_pointer(f)), a.n)
    g = M.partition(f, a, pl)
    return f, g, M.dependency_levels(g)


def proj_weights(m):
    """Same +-1 weights as tests/golden/make_golden.py:proj_weights."""
    e = np.arange(m, dtype=np.uint64)
    h = (e * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(40)
    return np.where(h & np.uint64(1), 1.0, -1.0)


def factored(name):
    """(a, grid, tree, device LUFactors) of a config, structure re-checked against the reference."""
    a = G.CONFIGS[name]()
    f, g, t = pipeline(a)
    rec = CASES.get(name)
    if rec:
        assert [sha(a.col_ptr), sha(a.row_idx), sha(a.values)] == rec["a_sha"]
        assert f.nnz_filled == rec["nnz_filled"] and g.p == rec["p"]
        assert sha(g.plan.positions) == rec["positions"]
        for fld in ("kinds", "levels_of", "pred_ptr", "pred_idx", "costs"):
            assert sha(getattr(t, fld)) == rec["tree_" + fld], fld
    return a, g, t, M.factorize(g, t)


def final_blocks_vs_oracle(name, a, g, t, lu):
    og = OS.Grid(a.n, g.p, g.plan.positions, g.blocks, g.block_nnz, g.value_max)
    s, final = ON.factorize_prefix(og, t, budget_s=BUDGET_S)
    lb, ub = ON.export(final)
    amax = float(np.abs(a.values).max())
    compared = 0
    worst = 0.0
    for blocks, ob in ((lu.l_blocks, lb), (lu.u_blocks, ub)):
        for k, want in ob.items():
            got = blocks[k]
            assert np.array_equal(got.col_ptr, want.col_ptr) and np.array_equal(got.row_idx, want.row_idx), k
            scale = max(float(np.abs(want.values).max(initial=0.0)), 1e-3 * amax)
            err = float(np.abs(got.values - want.values).max(initial=0.0))
            assert err <= 1e-10 * scale, (k, err, scale)
            worst = max(worst, err / scale)
            compared += len(want.values)
    total = sum(b.nnz for b in lu.l_blocks.values()) + sum(b.nnz for b in lu.u_blocks.values())
    print(f"{name}: steps 0..{s} of {g.p}: {compared}/{total} factor values compared, worst rel {worst:.2e}")
    assert compared > 0


def whole_factor_checksums_vs_reference(a, lu, z):
    amax = float(np.abs(a.values).max())
    for tag, blocks in (("L", lu.l_blocks), ("U", lu.u_blocks)):
        bk = z[tag + "_blocks_key"]
        assert len(bk) == len(blocks)
        got_nnz = np.array([blocks[(int(bi), int(bj))].nnz for bi, bj, _ in bk])
        assert np.array_equal(got_nnz, bk[:, 2])  # identical exported structure per block
        for q, (bi, bj, nz) in enumerate(bk):
            v = blocks[(int(bi), int(bj))].values
            absmax = float(z[tag + "_blocks_absmax"][q])
            tol = 1e-10 * max(absmax, 1e-3 * amax)
            assert abs(float(np.abs(v).max(initial=0.0)) - absmax) <= tol
            # every value enters the abs-sum and the +-1 projection; independent rounding-level
            # deviations grow like sqrt(nnz)
            slack = tol * max(1.0, float(nz) ** 0.5)
            assert abs(float(np.abs(v).sum()) - float(z[tag + "_blocks_abssum"][q])) <= slack
            assert abs(float(np.dot(proj_weights(len(v)), v)) - float(z[tag + "_blocks_proj"][q])) <= slack
        keys = z[tag + "_samples_key"]
        got = np.array([blocks[(int(bi), int(bj))].values[int(e)] for bi, bj, e in keys])
        np.testing.assert_allclose(got, z[tag + "_samples_val"], rtol=1e-10, atol=1e-10 * amax)


@pytest.mark.parametrize("name", ["C5", "C3", "C2"])
def test_full_config_vs_oracle_and_reference(name):
    a, g, t, lu = factored(name)
    final_blocks_vs_oracle(name, a, g, t, lu)
    path = os.path.join(GOLDEN, f"case_{name}.npz")
    z = np.load(path) if os.path.exists(path) else None
    if z is not None and "L_blocks_proj" in z:
        whole_factor_checksums_vs_reference(a, lu, z)
    A = a.to_scipy()
    b = A @ np.ones(a.n)
    x = M.solve(lu, b)
    relres = float(np.linalg.norm(A @ x - b) / np.linalg.norm(b))
    rec = CASES.get(name, {})
    bound = max(2 * rec["relres"], 1e-14) if "relres" in rec else 1e-12
    assert relres <= bound, (relres, bound)
