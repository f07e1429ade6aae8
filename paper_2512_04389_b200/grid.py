"""Block grid and task dependency tree — pkg/src/lublock/grid.py, native core.

``partition`` and ``dependency_levels`` run in C++ (csrc/lbk_host.cpp) and
return the reference's exact types and arrays.  A grid built here also keeps
its pooled arrays (``BlockGrid.pool``): every ``SparseBlock`` is a view into
them, so packing the grid for the device is a no-op; a grid built by the
reference (dict of independent blocks) is pooled on first use instead.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from . import _native
from .blocking import BlockingPlan
from .errors import DimensionMismatch
from .matrix_io import CscMatrix
from .symbolic import FilledPattern

GETRF, GESSM, TSTRF, SSSSM = 0, 1, 2, 3
KIND_NAMES = ("GETRF", "GESSM", "TSTRF", "SSSSM")


@dataclass
class SparseBlock:
    """Local-index CSC block, possibly rectangular (grid.py:28-59)."""

    nrows: int
    ncols: int
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])

    @property
    def col_counts(self) -> np.ndarray:
        return np.diff(self.col_ptr)

    @property
    def row_counts(self) -> np.ndarray:
        return np.bincount(self.row_idx, minlength=self.nrows)

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols))
        d[self.row_idx, np.repeat(np.arange(self.ncols), self.col_counts)] = self.values
        return d

    def support_flat(self) -> np.ndarray:
        """Row-major flat indices of the stored support."""
        return self.row_idx * self.ncols + np.repeat(np.arange(self.ncols), self.col_counts)


@dataclass
class GridPool:
    """Pooled storage of all blocks: the host image of the device layout.

    table: int64[7, nblocks] = bi, bj, nrows, ncols, nnz, colptr_off, entry_off
    col_ptr: local col pointers, concatenated; row_idx/values: entries, concatenated.
    """

    table: np.ndarray
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray

    @property
    def nblocks(self) -> int:
        return self.table.shape[1]


@dataclass
class BlockGrid:
    """Sparse map of nonempty blocks plus per-block nnz counts (grid.py:62-82)."""

    n: int
    p: int
    plan: BlockingPlan
    blocks: dict
    block_nnz: np.ndarray
    nnz_filled: int
    value_max: float
    pool: GridPool | None = field(default=None, repr=False, compare=False)
    # pool position of every entry of A (CSC order) when built by ``partition``: the
    # remaining pool entries are the fill (exactly 0.0, grid.py:85-148), so the device
    # factorization only needs A's nnz values (numeric.factorize)
    a_pos: np.ndarray | None = field(default=None, repr=False, compare=False)

    def lower_blocks(self, i: int) -> np.ndarray:
        return i + 1 + np.flatnonzero(self.block_nnz[i + 1:, i])

    def upper_blocks(self, i: int) -> np.ndarray:
        return i + 1 + np.flatnonzero(self.block_nnz[i, i + 1:])


def pool_grid(grid) -> GridPool:
    """Pooled view of any BlockGrid-like object (ours or the reference's)."""
    pool = getattr(grid, "pool", None)
    if pool is not None:
        return pool
    keys = sorted(grid.blocks, key=lambda k: (k[1], k[0]))  # column-major block order
    nb = len(keys)
    table = np.zeros((7, nb), dtype=np.int64)
    cps, ris, vals = [], [], []
    cpo = 0
    ento = 0
    for b, (bi, bj) in enumerate(keys):
        blk = grid.blocks[(bi, bj)]
        table[:, b] = (bi, bj, blk.nrows, blk.ncols, blk.nnz, cpo, ento)
        cps.append(np.asarray(blk.col_ptr, dtype=np.int64))
        ris.append(np.asarray(blk.row_idx, dtype=np.int64))
        vals.append(np.asarray(blk.values, dtype=np.float64))
        cpo += blk.ncols + 1
        ento += blk.nnz
    cat = lambda xs, dt: np.concatenate(xs) if xs else np.empty(0, dt)  # noqa: E731
    pool = GridPool(table=table, col_ptr=cat(cps, np.int64), row_idx=cat(ris, np.int64),
                    values=cat(vals, np.float64))
    try:
        grid.pool = pool
    except AttributeError:  # frozen / slotted foreign grid
        pass
    return pool


def pool_positions(f: FilledPattern, a: CscMatrix, plan: BlockingPlan) -> np.ndarray:
    """Position in the pooled grid values (reference pool order) of every entry
    of A (CSC order), as recorded by ``partition`` (``BlockGrid.a_pos``).
    Refactorizations with new values on A's pattern then only move A's entries
    to the device (Engine.bind_matrix / refactor_host)."""
    return partition(f, a, plan).a_pos


def partition(f: FilledPattern, a: CscMatrix, plan: BlockingPlan) -> BlockGrid:
    """Cut the filled pattern into blocks, scattering A's values (grid.py:85-148)."""
    n = f.n
    if not plan.n == n == a.n:
        raise DimensionMismatch(f"plan n={plan.n}, pattern n={f.n}, matrix n={a.n} must agree")
    fcp = np.ascontiguousarray(f.col_ptr, dtype=np.int64)
    fri = np.ascontiguousarray(f.row_idx, dtype=np.int64)
    acp = np.ascontiguousarray(a.col_ptr, dtype=np.int64)
    ari = np.ascontiguousarray(a.row_idx, dtype=np.int64)
    av = np.ascontiguousarray(a.values, dtype=np.float64)
    pos = np.ascontiguousarray(plan.positions, dtype=np.int64)
    p = plan.p
    lib = _native.host_lib()
    nb = C.c_int64()
    cpl = C.c_int64()
    P = _native.ptr
    i64 = _native.c_i64p
    rc = lib.lbk_partition_count(n, P(fcp, i64), P(fri, i64), p, P(pos, i64), C.byref(nb), C.byref(cpl))
    _native.check_host(rc, "partition")
    nblocks = nb.value
    table = np.empty((7, nblocks), np.int64)
    col_ptr = np.empty(cpl.value, np.int64)
    nnzf = int(fcp[-1])
    row_idx = np.empty(nnzf, np.int64)
    values = np.empty(nnzf, np.float64)
    block_nnz = np.empty((p, p), np.int64)
    a_pos = np.empty(len(ari), np.int64)
    rc = lib.lbk_partition_fill(n, P(fcp, i64), P(fri, i64), P(acp, i64), P(ari, i64), P(av, _native.c_f64p),
                                p, P(pos, i64), nblocks, P(table, i64), P(col_ptr, i64), P(row_idx, i64),
                                P(values, _native.c_f64p), P(block_nnz, i64), P(a_pos, i64))
    _native.check_host(rc, "partition")
    # the grid is an input (factorize never mutates it, factorize.py:265); read-only
    # pooled values guarantee that the fill entries stay 0.0, which lets the device
    # path upload only A's values (a_pos)
    values.flags.writeable = False
    pool = GridPool(table=table, col_ptr=col_ptr, row_idx=row_idx, values=values)
    blocks = {}
    for b in range(nblocks):
        bi, bj, nr, nc, nz, cpo, eo = (int(x) for x in table[:, b])
        blocks[(bi, bj)] = SparseBlock(nrows=nr, ncols=nc, col_ptr=col_ptr[cpo:cpo + nc + 1],
                                       row_idx=row_idx[eo:eo + nz], values=values[eo:eo + nz])
    value_max = float(np.max(np.abs(av))) if a.nnz else 0.0
    return BlockGrid(n=n, p=p, plan=plan, blocks=blocks, block_nnz=block_nnz,
                     nnz_filled=f.nnz_filled, value_max=value_max, pool=pool, a_pos=a_pos)


class TaskView(NamedTuple):
    kind: int
    step: int
    row: int
    col: int
    weight: int
    cost: int
    level: int


@dataclass
class DependencyTree:
    """Level-ordered task DAG of blocked right-looking LU (grid.py:161-220)."""

    p: int
    kinds: np.ndarray
    steps: np.ndarray
    rows: np.ndarray
    cols: np.ndarray
    weights: np.ndarray
    costs: np.ndarray
    levels_of: np.ndarray
    pred_ptr: np.ndarray
    pred_idx: np.ndarray

    @property
    def task_count(self) -> int:
        return len(self.kinds)

    @property
    def n_levels(self) -> int:
        return int(self.levels_of.max()) + 1 if self.task_count else 0

    @property
    def levels(self) -> list[np.ndarray]:
        """Task ids per level, construction order inside a level."""
        order = np.argsort(self.levels_of, kind="stable")
        bounds = np.cumsum(np.bincount(self.levels_of, minlength=self.n_levels))[:-1]
        return np.split(order, bounds)

    def task(self, t: int) -> TaskView:
        return TaskView(int(self.kinds[t]), int(self.steps[t]), int(self.rows[t]), int(self.cols[t]),
                        int(self.weights[t]), int(self.costs[t]), int(self.levels_of[t]))

    def successors(self) -> tuple[np.ndarray, np.ndarray]:
        nt = self.task_count
        dst = np.repeat(np.arange(nt, dtype=np.int64), np.diff(self.pred_ptr).astype(np.int64))
        order = np.argsort(self.pred_idx, kind="stable")
        ptr = np.zeros(nt + 1, dtype=np.int64)
        np.cumsum(np.bincount(self.pred_idx, minlength=nt), out=ptr[1:])
        return ptr, dst[order]


def dependency_levels(grid: BlockGrid) -> DependencyTree:
    """Static task DAG with ASAP levels, construction order of grid.py:223-378."""
    pool = pool_grid(grid)
    p = grid.p
    lib = _native.host_lib()
    h = C.c_void_p()
    nt = C.c_int64()
    npred = C.c_int64()
    P = _native.ptr
    i64 = _native.c_i64p
    table = np.ascontiguousarray(pool.table)
    rc = lib.lbk_levels_run(p, pool.nblocks, P(table, i64), P(pool.col_ptr, i64),
                            P(pool.row_idx, i64), C.byref(h), C.byref(nt), C.byref(npred))
    _native.check_host(rc, "dependency_levels")
    try:
        t = nt.value
        kinds = np.empty(t, np.int8)
        steps = np.empty(t, np.int32)
        rows = np.empty(t, np.int32)
        cols = np.empty(t, np.int32)
        weights = np.empty(t, np.int64)
        costs = np.empty(t, np.int64)
        levels = np.empty(t, np.int32)
        pred_ptr = np.empty(t + 1, np.int64)
        pred_idx = np.empty(npred.value, np.int32)
        i32 = _native.c_i32p
        lib.lbk_levels_fetch(h, P(kinds, _native.c_i8p), P(steps, i32), P(rows, i32), P(cols, i32),
                             P(weights, i64), P(costs, i64), P(levels, i32), P(pred_ptr, i64),
                             P(pred_idx, i32))
    finally:
        lib.lbk_levels_free(h)
    return DependencyTree(p=p, kinds=kinds, steps=steps, rows=rows, cols=cols, weights=weights,
                          costs=costs, levels_of=levels, pred_ptr=pred_ptr, pred_idx=pred_idx)
