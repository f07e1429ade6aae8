"""Oracle restatement of the reference numerical factorization (TEST INFRASTRUCTURE ONLY).

Serial topological execution of the task DAG over a dense scratch copy of
every stored block, like pkg/src/lublock/factorize.py:245-384 with
workers=1.  Kernels (dense loops, rank-1 updates over the full trailing
block — the reference restricts to structural nonzeros, which only skips
exact-zero products, factorize.py:72-73):

* GETRF  factorize.py:38-78   block-local partial pivoting, first argmax,
  ZeroPivot test ``piv == 0 or piv < tol * colmax_at_entry``, static pivot
  replacement keeps the sign;
* GESSM  factorize.py:326-337 + 98-109  perm applied to the U panel, unit
  lower forward substitution;
* TSTRF  factorize.py:338-345 + 112-130 right upper solve;
* SSSSM  factorize.py:307-325  tgt -= L @ U with the support checks.

Returns dense blocks + perms, and ``export`` turns them into per-block CSC
with exact zeros dropped (factorize.py:179-192, 370-381).
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular

from .structure import GESSM, GETRF, SSSSM, TSTRF, Block


class OracleZeroPivot(Exception):
    def __init__(self, block, col):
        self.block, self.col = block, col
        super().__init__(f"zero pivot in block {block} col {col}")


class OracleSupportViolation(Exception):
    pass


def dense(b: Block) -> np.ndarray:
    d = np.zeros((b.nrows, b.ncols))
    d[b.row_idx, np.repeat(np.arange(b.ncols), np.diff(b.col_ptr))] = b.values
    return d


def getrf(d, pivot_tol=1e-12, static_eps=None, block=0):
    """In-place LU with pivoting confined to the block; returns (perm, swapped)."""
    m = d.shape[0]
    perm = np.arange(m)
    swapped = False
    colmax = np.abs(d).max(axis=0) if m else np.zeros(0)
    for k in range(m):
        mags = np.abs(d[k:, k])
        off = int(np.argmax(mags))
        piv = mags[off]
        if piv == 0.0 or piv < pivot_tol * colmax[k]:
            if static_eps is None:
                raise OracleZeroPivot(block, k)
            d[k, k] = static_eps if d[k, k] == 0.0 else math.copysign(static_eps, d[k, k])
        elif off:
            d[[k, k + off]] = d[[k + off, k]]
            perm[[k, k + off]] = perm[[k + off, k]]
            swapped = True
        if k + 1 < m:
            d[k + 1:, k] /= d[k, k]
            # rank-1 update on the nonzero rows x nonzero columns only: the
            # skipped terms are exact-zero products (same bits, far less work
            # on sparse blocks — this is also what the reference does)
            rows = k + 1 + np.flatnonzero(d[k + 1:, k])
            cols = k + 1 + np.flatnonzero(d[k, k + 1:])
            if len(rows) and len(cols):
                d[np.ix_(rows, cols)] -= np.outer(d[rows, k], d[k, cols])
    return perm, swapped


def gessm(lsrc, x):
    """x <- L^-1 x, L = unit lower part of lsrc."""
    for k in range(lsrc.shape[0] - 1):
        rows = k + 1 + np.flatnonzero(lsrc[k + 1:, k])
        if len(rows):
            x[rows] -= np.outer(lsrc[rows, k], x[k])


def tstrf(x, usrc):
    """x <- x U^-1, U = upper part (with diagonal) of usrc."""
    m = usrc.shape[1]
    for k in range(m):
        x[:, k] /= usrc[k, k]
        if k + 1 < m:
            rows = np.flatnonzero(x[:, k])
            cols = k + 1 + np.flatnonzero(usrc[k, k + 1:])
            if len(rows) and len(cols):
                x[np.ix_(rows, cols)] -= np.outer(x[rows, k], usrc[k, cols])


def factorize(grid, tree, pivot_tol=1e-12, static_pivot=None):
    """Serial DAG execution; returns (state: {(bi,bj): dense}, perms: list)."""
    state = {k: dense(b) for k, b in grid.blocks.items()}
    perms = [None] * grid.p
    static_eps = None if static_pivot is None else float(static_pivot) * (grid.value_max or 1.0)
    checking = True
    outside = {}
    for t in range(len(tree.kinds)):
        kind, i, r, c = int(tree.kinds[t]), int(tree.steps[t]), int(tree.rows[t]), int(tree.cols[t])
        if kind == SSSSM:
            prod = state[(r, i)] @ state[(i, c)]
            tgt = state.get((r, c))
            if tgt is None:
                if prod.any():
                    raise OracleSupportViolation(f"step {i} hits empty block ({r},{c})")
                continue
            if checking:
                if (r, c) not in outside:
                    b = grid.blocks[(r, c)]
                    mask = np.ones((b.nrows, b.ncols), bool)
                    mask[b.row_idx, np.repeat(np.arange(b.ncols), np.diff(b.col_ptr))] = False
                    outside[(r, c)] = mask
                if prod[outside[(r, c)]].any():
                    raise OracleSupportViolation(f"step {i} writes outside support of ({r},{c})")
            tgt -= prod
        elif kind == GESSM:
            x = state[(i, c)]
            if perms[i] is not None:
                x[:] = x[perms[i]]
            gessm(state[(i, i)], x)
        elif kind == TSTRF:
            tstrf(state[(r, i)], state[(i, i)])
        else:
            perm, swapped = getrf(state[(i, i)], pivot_tol, static_eps, i)
            perms[i] = perm if swapped else None
            if swapped:
                checking = False
    for i in range(grid.p):
        if perms[i] is None:
            perms[i] = np.arange(int(grid.positions[i + 1] - grid.positions[i]))
    return state, perms


def factorize_prefix(grid, tree, max_step=None, budget_s=None, pivot_tol=1e-12):
    """The serial execution of ``factorize`` restricted to the task-list prefix of steps
    0..s (construction order puts every task of step i before any task of step i+1,
    grid.py:223-378), densifying blocks on first touch.  Stops after step ``max_step``
    or, with ``budget_s``, after the first step that ends past the budget.

    Blocks (bi, bj) with min(bi, bj) <= s are FINAL after step s (their GETRF / GESSM /
    TSTRF at step min(bi, bj) and every SSSSM into them, steps < min(bi, bj), are in the
    prefix), so a full-size device factorization can be checked value by value on them.
    No-swap inputs only (the row-swap quirk needs the whole dense scratch).
    Returns (s, {(bi, bj): dense} of the final blocks).
    """
    import time

    state = {}

    def blk(key):
        d = state.get(key)
        if d is None:
            d = dense(grid.blocks[key])
            state[key] = d
        return d

    t0 = time.perf_counter()
    nt = len(tree.kinds)
    last = -1
    t = 0
    while t < nt:
        step = int(tree.steps[t])
        if max_step is not None and step > max_step:
            break
        if budget_s is not None and last >= 0 and time.perf_counter() - t0 > budget_s:
            break
        while t < nt and int(tree.steps[t]) == step:
            kind, i, r, c = int(tree.kinds[t]), step, int(tree.rows[t]), int(tree.cols[t])
            if kind == SSSSM:
                if (r, c) in grid.blocks:
                    blk((r, c))[...] -= blk((r, i)) @ blk((i, c))
            elif kind == GESSM:
                gessm(blk((i, i)), blk((i, c)))
            elif kind == TSTRF:
                tstrf(blk((r, i)), blk((i, i)))
            else:
                _, swapped = getrf(blk((i, i)), pivot_tol, None, i)
                if swapped:
                    raise ValueError("factorize_prefix: row swap in block %d (no-swap inputs only)" % i)
            t += 1
        last = step
    final = {k: d for k, d in state.items() if min(k) <= last}
    return last, final


def to_block(d) -> Block:
    """Dense -> CSC dropping exact zeros (factorize.py:179-192)."""
    cols, rows = np.nonzero(d.T)
    cp = np.concatenate([[0], np.cumsum(np.bincount(cols, minlength=d.shape[1]))]).astype(np.int64)
    return Block(d.shape[0], d.shape[1], cp, rows.astype(np.int64), d.T[cols, rows])


def export(state):
    """(l_blocks, u_blocks): strictly lower -> L, strictly upper -> U, diagonal split."""
    lb, ub = {}, {}
    for (bi, bj), d in state.items():
        if bi > bj:
            lb[(bi, bj)] = to_block(d)
        elif bi < bj:
            ub[(bi, bj)] = to_block(d)
        else:
            lb[(bi, bj)] = to_block(np.tril(d, -1) + np.eye(d.shape[0]))
            ub[(bi, bj)] = to_block(np.triu(d))
    return lb, ub


def assemble(n, positions, blocks):
    rows, cols, vals = [], [], []
    for (bi, bj), b in blocks.items():
        rows.append(b.row_idx + positions[bi])
        cols.append(np.repeat(np.arange(b.ncols), np.diff(b.col_ptr)) + positions[bj])
        vals.append(b.values)
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n, n)).tocsr()


def perm_global(positions, perms):
    return np.concatenate([positions[i] + perms[i] for i in range(len(perms))])


def residual(a, n, positions, lb, ub, perms):
    """||P A - L U||_F / ||A||_F (factorize.py:438-448)."""
    A = sp.csc_matrix((a.values, a.row_idx, a.col_ptr), shape=(n, n)).tocsr()
    diff = (A[perm_global(positions, perms), :] - assemble(n, positions, lb) @ assemble(n, positions, ub)).tocoo()
    num = math.sqrt(float(np.sum(diff.data ** 2)))
    den = math.sqrt(float(np.sum(a.values ** 2)))
    return 0.0 if den == 0 and num == 0 else (math.inf if den == 0 else num / den)


def solve(n, positions, lb, ub, perms, b):
    """x = U^-1 L^-1 b[perm] (factorize.py:451-457)."""
    y = spsolve_triangular(assemble(n, positions, lb), np.asarray(b, float)[perm_global(positions, perms)],
                           lower=True)
    return spsolve_triangular(assemble(n, positions, ub), y, lower=False)
