"""Algorithmic work per task, used for GFLOP/s and the roofline.

Flops F_t (lc/uc = strictly-lower column / strictly-upper row counts inside
the diagonal block; colcnt/rowcnt = per-column / per-row counts of a panel):
  GETRF(i)     sum_c lc_c (1 + 2 uc_c)
  GESSM(i,j)   2 sum_k lc_ii[k] rowcnt_ij[k]
  TSTRF(k,i)   sum_c colcnt_ki[c] (1 + 2 uc_ii[c])
  SSSSM(k,j,i) 2 tree.costs[t]                       (grid.py:334)
sum_t F_t == sum_k c_k (1 + 2 c_k) over the filled pattern (checked in tests).

Bytes B_t (8 B per value, 4 B per index; read+write of outputs):
  GETRF 20 nnz_ii;  panels 12 nnz_ii + 20 nnz_panel;
  SSSSM 12 nnz_ki + 12 nnz_ij + 20 nnz_kj.
"""

from __future__ import annotations

import numpy as np

from .grid import GESSM, GETRF, SSSSM, TSTRF, pool_grid


def _block_counts(pool):
    """Per block: (col counts, row counts, strictly-lower col counts, strictly-upper row counts)."""
    t = pool.table
    out = {}
    for b in range(pool.nblocks):
        bi, bj, nr, nc, nz, cpo, eo = (int(x) for x in t[:, b])
        cp = pool.col_ptr[cpo:cpo + nc + 1]
        ri = pool.row_idx[eo:eo + nz]
        colcnt = np.diff(cp)
        rowcnt = np.bincount(ri, minlength=nr)
        if bi == bj:
            cols = np.repeat(np.arange(nc), colcnt)
            lc = np.bincount(cols[ri > cols], minlength=nc)
            uc = np.bincount(ri[ri < cols], minlength=nr)
        else:
            lc = uc = None
        out[(bi, bj)] = (colcnt, rowcnt, lc, uc, nz)
    return out


def task_work(grid, tree):
    """(flops[t], bytes[t]) as float64 arrays."""
    pool = pool_grid(grid)
    bc = _block_counts(pool)
    nt = tree.task_count
    flops = np.zeros(nt)
    byts = np.zeros(nt)
    for t in range(nt):
        k = int(tree.kinds[t])
        i, r, c = int(tree.steps[t]), int(tree.rows[t]), int(tree.cols[t])
        _, _, lc, uc, nzd = bc[(i, i)]
        if k == GETRF:
            flops[t] = float(np.dot(lc, 1 + 2 * uc))
            byts[t] = 20.0 * nzd
        elif k == GESSM:
            _, rowcnt, _, _, nzp = bc[(i, c)]
            flops[t] = 2.0 * float(np.dot(lc, rowcnt))
            byts[t] = 12.0 * nzd + 20.0 * nzp
        elif k == TSTRF:
            colcnt, _, _, _, nzp = bc[(r, i)]
            flops[t] = float(np.dot(colcnt, 1 + 2 * uc))
            byts[t] = 12.0 * nzd + 20.0 * nzp
        else:
            flops[t] = 2.0 * float(tree.costs[t])
            nl = bc[(r, i)][4]
            nu = bc[(i, c)][4]
            nk = bc[(r, c)][4] if (r, c) in bc else 0
            byts[t] = 12.0 * nl + 12.0 * nu + 20.0 * nk
    return flops, byts


def scalar_flops(f) -> float:
    """sum_k c_k (1 + 2 c_k), c_k = strictly-lower count of column k of the filled pattern."""
    cols = f.entry_cols()
    ck = np.bincount(cols[f.row_idx > cols], minlength=f.n).astype(np.float64)
    return float(np.sum(ck * (1 + 2 * ck)))
