"""SupportViolation semantics (factorize.py:277-324) for grids this package did not build.

A grid whose block patterns are not elimination-closed makes the reference raise
SupportViolation at the first SSSSM whose product leaves the target's filled
support.  The drop-in checks the same thing structurally before any device work
(numeric.check_support), so these tests run on the CPU: a reference-built grid
with one fill entry removed from a block must raise the reference's exception
class with the reference's message, and a closed reference-built grid must pass.
"""

import os
import sys

import numpy as np
import pytest

import paper_2512_04389_b200 as M
from oracle import ref_timing as RT
from paper_2512_04389_b200.numeric import check_support


def _reference():
    try:
        return RT.import_reference()
    except ImportError:
        src = "/root/reference/pkg/src"
        if not os.path.isdir(src):
            return None
        sys.path.insert(0, src)
        import lublock

        return lublock


L = _reference()
pytestmark = pytest.mark.skipif(L is None, reason="the reference is not importable here")


def ref_grid(k=8, bs=16):
    n, r, c, v = RT.family_triplets("poisson2d", k)
    a = L.csc_from_triplets(n, (r, c, v))
    f = L.symbolic_factorize(L.symmetrize_pattern(a))
    g = L.partition(f, a, L.regular_plan(a.n, bs))
    return a, g, L.dependency_levels(g)


def drop_product_entry(grid, tree):
    """Remove from the target of the first SSSSM one position its product structurally hits
    (a fill entry, value 0.0): that update then writes outside the stored support."""
    import scipy.sparse as sp

    def pat(key):
        b = grid.blocks[key]
        return sp.csc_matrix((np.ones(b.nnz), b.row_idx, b.col_ptr), shape=(b.nrows, b.ncols)).toarray() > 0

    q = int(np.flatnonzero(np.asarray(tree.kinds) == L.SSSSM)[0])
    i, r, c = int(tree.steps[q]), int(tree.rows[q]), int(tree.cols[q])
    hit = (pat((r, i)).astype(int) @ pat((i, c)).astype(int)) > 0
    b = grid.blocks[(r, c)]
    cols = np.repeat(np.arange(b.ncols), np.diff(b.col_ptr))
    cand = [e for e in range(b.nnz) if hit[b.row_idx[e], cols[e]] and b.values[e] == 0.0]
    e = cand[0]
    keep = np.ones(b.nnz, bool)
    keep[e] = False
    cp = np.concatenate([[0], np.cumsum(np.bincount(cols[keep], minlength=b.ncols))]).astype(np.int64)
    grid.blocks[(r, c)] = L.SparseBlock(b.nrows, b.ncols, cp, b.row_idx[keep], b.values[keep])
    grid.block_nnz[r, c] -= 1


def test_closed_reference_grid_passes():
    a, g, t = ref_grid()
    check_support(g, t)
    assert getattr(g, "_lbk_support_ok", False)


def test_broken_support_raises_like_the_reference():
    a, g, t = ref_grid()
    drop_product_entry(g, t)
    with pytest.raises(L.SupportViolation) as want:
        L.factorize(g, t)
    with pytest.raises(M.SupportViolation) as got:
        check_support(g, t)
    assert str(got.value) == str(want.value)
