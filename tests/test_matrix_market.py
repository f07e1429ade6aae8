"""Matrix Market input: the product reader vs the reference's own reader.

``read_matrix_market`` (pkg/src/lublock/matrix_io.py:156-227) is the entry the
paper's SuiteSparse matrices (not downloadable here: no
network) come through.  Files covering the format's variants — real / integer /
pattern fields, general / symmetric storage, duplicates (summed, zero sums
kept), comments and blank lines, 1-based indices — are written to a temp dir
and read by both; the CSC arrays must be identical and the same exception
classes must be raised on malformed input.  A generated BASELINE matrix written
as .mtx and read back then runs the whole structure path bit-exactly.
"""

import os
import sys

import numpy as np
import pytest

import paper_2512_04389_b200 as M
from oracle import ref_timing as RT
from paper_2512_04389_b200 import generators as G


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

FILES = {
    "real_general": "%%MatrixMarket matrix coordinate real general\n% a comment\n\n4 4 7\n1 1 4.0\n2 1 -1.5\n"
                    "1 2 -1.0\n2 2 4.0\n3 3 2.5e-1\n4 4 1e3\n3 4 -0.0\n",
    "duplicates": "%%MatrixMarket matrix coordinate real general\n3 3 6\n1 1 1.0\n1 1 2.0\n2 2 1.0\n3 3 1.0\n"
                  "3 1 1.0\n3 1 -1.0\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n5 5 7\n1 1 2\n2 1 -1\n2 2 2\n3 2 -1\n3 3 2\n"
                 "5 1 0.5\n5 5 2\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n3 3 4\n1 1\n2 2\n3 3\n1 3\n",
    "pattern_symmetric": "%%MatrixMarket matrix coordinate pattern symmetric\n4 4 5\n1 1\n2 2\n3 3\n4 4\n4 2\n",
    "integer": "%%MatrixMarket matrix coordinate integer general\n2 2 3\n1 1 3\n2 2 -7\n1 2 1\n",
}

BAD = {
    "non_square": "%%MatrixMarket matrix coordinate real general\n3 4 1\n1 1 1.0\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1.0 0.0\n",
    "array": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "short_entry": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "too_many": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n",
    "too_few": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n",
    "empty": "%%MatrixMarket matrix coordinate real general\n0 0 0\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n2 2\n",
}


def write(tmp_path, name, text):
    p = tmp_path / f"{name}.mtx"
    p.write_text(text)
    return str(p)


@pytest.mark.parametrize("name", sorted(FILES))
def test_reader_matches_reference(tmp_path, name):
    path = write(tmp_path, name, FILES[name])
    want = L.read_matrix_market(path)
    got = M.read_matrix_market(path)
    assert got.n == want.n
    for fld in ("col_ptr", "row_idx", "values"):
        a, b = np.asarray(getattr(got, fld)), np.asarray(getattr(want, fld))
        assert a.dtype == b.dtype and a.tobytes() == b.tobytes(), fld


@pytest.mark.parametrize("name", sorted(BAD))
def test_reader_errors_match_reference(tmp_path, name):
    path = write(tmp_path, name, BAD[name])
    with pytest.raises(Exception) as want:
        L.read_matrix_market(path)
    with pytest.raises(Exception) as got:
        M.read_matrix_market(path)
    assert type(got.value).__name__ == type(want.value).__name__


def test_generated_matrix_roundtrip_through_mtx(tmp_path):
    """A BBD matrix (the circuit-like family of configs 3 / 5) written as symmetric-pattern-free
    general .mtx and read back: same matrix, then the same plan and task tree as the reference."""
    a = G.bbd(6000, 120, 12, seed=4)
    cols = np.repeat(np.arange(a.n), np.diff(a.col_ptr))
    lines = ["%%MatrixMarket matrix coordinate real general", f"{a.n} {a.n} {a.nnz}"]
    lines += [f"{r + 1} {c + 1} {float(v)!r}" for r, c, v in zip(a.row_idx, cols, a.values)]
    path = write(tmp_path, "bbd6000", "\n".join(lines) + "\n")
    got = M.read_matrix_market(path)
    want = L.read_matrix_market(path)
    assert np.array_equal(got.values, a.values) and np.array_equal(got.row_idx, a.row_idx)
    f = M.symbolic_factorize(M.symmetrize_pattern(got))
    plan = M.irregular_plan(M.percentage_curve(M.diag_block_pointer(f)), got.n)
    t = M.dependency_levels(M.partition(f, got, plan))
    rf = L.symbolic_factorize(L.symmetrize_pattern(want))
    rplan = L.irregular_plan(L.percentage_curve(L.diag_block_pointer(rf)), want.n)
    rt = L.dependency_levels(L.partition(rf, want, rplan))
    assert np.array_equal(plan.positions, rplan.positions)
    for fld in ("kinds", "steps", "rows", "cols", "levels_of", "costs", "weights", "pred_ptr", "pred_idx"):
        assert np.array_equal(getattr(t, fld), getattr(rt, fld)), fld
