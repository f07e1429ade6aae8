"""Symbolic factorization (pkg/src/lublock/symbolic.py) with a native core.

``symbolic_factorize`` runs the elimination-tree row-subtree walk in C++
(csrc/lbk_host.cpp, ``lbk_symbolic_run``); output arrays equal the
reference's element for element.  The reference's Python loop takes 210 s at
C2; the native walk takes seconds.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes as C
import numpy as np

from . import _native
from .errors import DimensionMismatch, MissingDiagonal, NotSymmetric
from .matrix_io import CscMatrix, csc_from_triplets


@dataclass
class FilledPattern:
    """Structurally symmetric CSC pattern of L+U with full diagonal (symbolic.py:21-34)."""

    n: int
    col_ptr: np.ndarray
    row_idx: np.ndarray

    @property
    def nnz_filled(self) -> int:
        return int(self.col_ptr[-1])

    def entry_cols(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.col_ptr))


def symmetrize_pattern(a: CscMatrix) -> CscMatrix:
    """Pattern of A + A^T + I; A's values kept, added entries 0.0 (symbolic.py:37-43)."""
    n = a.n
    cols = a.entry_cols()
    diag = np.arange(n, dtype=np.int64)
    r = np.concatenate([a.row_idx, cols, diag])
    c = np.concatenate([cols, a.row_idx, diag])
    v = np.zeros(len(r))
    v[: a.nnz] = a.values
    return csc_from_triplets(n, (r, c, v))


def require_symmetric_full_diag(col_ptr, row_idx, n) -> None:
    """Reject patterns without a full diagonal or not structurally symmetric (symbolic.py:46-54)."""
    cp = np.ascontiguousarray(col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(row_idx, dtype=np.int64)
    nd = C.c_int64(0)
    rc = _native.host_lib().lbk_check_symmetric(
        n, _native.ptr(cp, _native.c_i64p), _native.ptr(ri, _native.c_i64p), C.byref(nd))
    if rc == 3:
        # unsorted input: fall back to the sort-based statement of the same rule
        cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
        ndiag = int(np.count_nonzero(ri == cols))
        if ndiag != n:
            raise MissingDiagonal(f"pattern has {ndiag} of {n} diagonal entries")
        if not np.array_equal(np.sort(cols * n + ri), np.sort(ri * n + cols)):
            raise NotSymmetric("pattern is not structurally symmetric")
        return
    if rc == 1:
        raise MissingDiagonal(f"pattern has {nd.value} of {n} diagonal entries")
    if rc == 2:
        raise NotSymmetric("pattern is not structurally symmetric")


def symbolic_factorize(a_sym: CscMatrix, *, validate: bool = True) -> FilledPattern:
    """Fill pattern of symmetric elimination in natural order (symbolic.py:57-108)."""
    n = a_sym.n
    cp = np.ascontiguousarray(a_sym.col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(a_sym.row_idx, dtype=np.int64)
    if validate:
        require_symmetric_full_diag(cp, ri, n)
    lib = _native.host_lib()
    nnz = C.c_int64()
    P, i64 = _native.ptr, _native.c_i64p
    _native.check_host(lib.lbk_symbolic_nnz(n, P(cp, i64), P(ri, i64), C.byref(nnz)), "symbolic_factorize")
    out_cp = np.empty(n + 1, np.int64)
    out_ri = np.empty(nnz.value, np.int64)
    _native.check_host(lib.lbk_symbolic_fill(n, P(cp, i64), P(ri, i64), P(out_cp, i64), P(out_ri, i64), None),
                       "symbolic_factorize")
    f = FilledPattern(n=n, col_ptr=out_cp, row_idx=out_ri)
    f._verified = True  # symmetric with a full diagonal by construction
    return f


def fill_ratio(a: CscMatrix, f: FilledPattern) -> float:
    """nnz(L+U) / nnz(symmetrized A) (symbolic.py:111-115)."""
    if a.n != f.n:
        raise DimensionMismatch(f"order mismatch: {a.n} vs {f.n}")
    return f.nnz_filled / symmetrize_pattern(a).nnz
