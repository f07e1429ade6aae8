"""Oracle restatement of the reference structure path (TEST INFRASTRUCTURE ONLY).

Plain numpy / Python, written from the reference's documented behaviour with
deliberately different formulations where the result is integer-exact:

* symbolic: column-merge over the elimination tree (struct L(:,j) = A's
  lower column j  U  children's structures minus j) instead of the
  reference's row-subtree walk (symbolic.py:57-108);
* blockptr: bincount of max(row, col) instead of Alg. 2's row counts
  (features.py:44-54) — equal on symmetric full-diagonal patterns;
* plan / partition / levels: direct transcriptions of blocking.py:49-151,
  grid.py:85-148 and grid.py:223-378.

Matrices are plain tuples (n, col_ptr, row_idx, values) of numpy arrays.
"""

from __future__ import annotations

from collections import namedtuple

import numpy as np
import scipy.sparse as sp

Csc = namedtuple("Csc", "n col_ptr row_idx values")
Block = namedtuple("Block", "nrows ncols col_ptr row_idx values")
Grid = namedtuple("Grid", "n p positions blocks block_nnz value_max")
Tree = namedtuple("Tree", "kinds steps rows cols weights costs levels_of pred_ptr pred_idx")

GETRF, GESSM, TSTRF, SSSSM = 0, 1, 2, 3


def triplets_to_csc(n, rows, cols, vals) -> Csc:
    """COO -> CSC, duplicates summed, zeros kept (matrix_io.py:99-139 semantics)."""
    m = sp.coo_matrix((np.asarray(vals, np.float64), (np.asarray(rows, np.int64),
                                                       np.asarray(cols, np.int64))),
                      shape=(n, n)).tocsc()
    m.sort_indices()
    return Csc(n, m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data.astype(np.float64))


def entry_cols(col_ptr) -> np.ndarray:
    return np.repeat(np.arange(len(col_ptr) - 1, dtype=np.int64), np.diff(col_ptr))


def symmetrize(a: Csc) -> Csc:
    """A + A^T + I pattern, A's values kept, new entries +0.0 (symbolic.py:37-43)."""
    n = a.n
    c = entry_cols(a.col_ptr)
    d = np.arange(n)
    r = np.concatenate([a.row_idx, c, d])
    cc = np.concatenate([c, a.row_idx, d])
    v = np.concatenate([a.values, np.zeros(len(c) + n)])
    return triplets_to_csc(n, r, cc, v)


def symbolic(a_sym: Csc):
    """Filled pattern (col_ptr, row_idx) of L+L^T+I by elimination-tree column merging."""
    n = a_sym.n
    cp, ri = a_sym.col_ptr, a_sym.row_idx
    children = [[] for _ in range(n)]
    lstruct = [None] * n
    for j in range(n):
        parts = [ri[cp[j]:cp[j + 1]]]
        parts += [lstruct[c] for c in children[j]]
        s = np.unique(np.concatenate(parts)) if parts else np.empty(0, np.int64)
        s = s[s > j]
        lstruct[j] = s
        if len(s):
            children[int(s[0])].append(j)
    lr = np.concatenate([lstruct[j] for j in range(n)]) if n else np.empty(0, np.int64)
    lc = np.repeat(np.arange(n), [len(lstruct[j]) for j in range(n)])
    d = np.arange(n)
    rows = np.concatenate([lr, lc, d]).astype(np.int64)
    cols = np.concatenate([lc, lr, d]).astype(np.int64)
    order = np.lexsort((rows, cols))
    rows = rows[order]
    cols = cols[order]
    col_ptr = np.concatenate([[0], np.cumsum(np.bincount(cols, minlength=n))]).astype(np.int64)
    return col_ptr, rows


def blockptr(n, col_ptr, row_idx) -> np.ndarray:
    """blockptr[k] = #entries in the leading k x k block (Alg. 2 result, features.py:44-54)."""
    m = np.maximum(row_idx, entry_cols(col_ptr))
    out = np.zeros(n + 1, np.int64)
    out[1:] = np.cumsum(np.bincount(m, minlength=n))
    return out


def curve(n, bptr, sample_points=1000):
    """(sp, pct): pct[k] = blockptr[(2kn+sp)//(2sp)] / blockptr[n] (features.py:57-68)."""
    sp_ = min(sample_points, n)
    k = np.arange(sp_ + 1, dtype=np.int64)
    idx = (2 * k * n + sp_) // (2 * sp_)
    return sp_, bptr[idx] / int(bptr[n])


def irregular_positions(pct, n, step=2, max_num=3, threshold="linear", overlapping=False):
    """Alg. 3 disjoint-window scan (blocking.py:49-114)."""
    sp_ = len(pct) - 1
    thr = float(step / sp_ if threshold == "linear" else threshold)
    emitted = []
    skipped = 0
    i = 0
    while i < sp_:
        if pct[min(i + step, sp_)] - pct[i] >= thr:
            emitted.append((2 * (i + step) * n + sp_) // (2 * sp_))
            skipped = 0
        elif skipped >= max_num:
            emitted.append((2 * (i + step) * n + sp_) // (2 * sp_))
            skipped = 0
        else:
            skipped += 1
        i += 1 if overlapping else step
    pos = [0]
    for e in emitted:
        if e >= n:
            break
        if e > pos[-1]:
            pos.append(e)
    return np.array(pos + [n], dtype=np.int64)


def regular_positions(n, bs):
    return np.array(list(range(0, n, bs)) + [n], dtype=np.int64)


def pangulu_select(n, nnz_filled):
    """blocking.py:130-151."""
    sizes = (200, 300, 500, 1000, 2000, 5000)
    dens = nnz_filled / float(n) / float(n)
    base = len(sizes) - 1
    for i, s in enumerate(sizes):
        if 10 * s >= n:
            base = i
            break
    down = 0
    if dens < 1e-4:
        down = 1
    if dens < 1e-6:
        down = 2
    return sizes[max(0, base - down)]


def partition(n, fcp, fri, a: Csc, positions) -> Grid:
    """Blocks of the filled pattern with A's values scattered in (grid.py:85-148)."""
    fcols = entry_cols(fcp)
    fkey = fcols * n + fri
    akey = entry_cols(a.col_ptr) * n + a.row_idx
    where = np.searchsorted(fkey, akey)
    assert np.array_equal(fkey[where], akey), "filled pattern must cover A"
    fvals = np.zeros(len(fkey))
    fvals[where] = a.values
    p = len(positions) - 1
    br = np.searchsorted(positions, fri, side="right") - 1
    bc = np.searchsorted(positions, fcols, side="right") - 1
    order = np.lexsort((np.arange(len(fkey)), bc * p + br))
    blocks = {}
    bnnz = np.zeros((p, p), np.int64)
    keys = (bc * p + br)[order]
    bounds = np.flatnonzero(np.diff(keys)) + 1
    for seg in np.split(order, bounds):
        if not len(seg):
            continue
        bi, bj = int(br[seg[0]]), int(bc[seg[0]])
        nr = int(positions[bi + 1] - positions[bi])
        nc = int(positions[bj + 1] - positions[bj])
        lc = fcols[seg] - positions[bj]
        cp = np.concatenate([[0], np.cumsum(np.bincount(lc, minlength=nc))]).astype(np.int64)
        blocks[(bi, bj)] = Block(nr, nc, cp, (fri[seg] - positions[bi]).astype(np.int64), fvals[seg])
        bnnz[bi, bj] = len(seg)
    vmax = float(np.abs(a.values).max()) if len(a.values) else 0.0
    return Grid(n, p, np.asarray(positions, np.int64), blocks, bnnz, vmax)


def levels(g: Grid) -> Tree:
    """Task DAG in construction order with ASAP levels (grid.py:223-378)."""
    p = g.p
    bn = g.block_nnz
    tasks = []  # (kind, step, row, col, weight, cost, level, preds)
    last = {}   # (r, c) -> (task id, level) of the latest SSSSM into that block

    def emit(kind, i, r, c, w, cost, lvl, preds):
        tasks.append((kind, i, r, c, w, cost, lvl, preds))
        return len(tasks) - 1

    for i in range(p):
        ups = [j for j in range(i + 1, p) if bn[i, j]]
        lows = [k for k in range(i + 1, p) if bn[k, i]]
        pid, plv = last.get((i, i), (-1, -1))
        g_lv = plv + 1
        g_id = emit(GETRF, i, i, i, int(bn[i, i]), int(bn[i, i]), g_lv, [pid] if pid >= 0 else [])
        u = {}
        for j in ups:
            pid, plv = last.get((i, j), (-1, -1))
            lv = max(g_lv, plv) + 1
            u[j] = (emit(GESSM, i, i, j, int(bn[i, j]), int(bn[i, j]), lv,
                         [g_id] + ([pid] if pid >= 0 else [])), lv)
        l_ = {}
        for k in lows:
            pid, plv = last.get((k, i), (-1, -1))
            lv = max(g_lv, plv) + 1
            l_[k] = (emit(TSTRF, i, k, i, int(bn[k, i]), int(bn[k, i]), lv,
                          [g_id] + ([pid] if pid >= 0 else [])), lv)
        for k in lows:
            colcnt = np.diff(g.blocks[(k, i)].col_ptr)
            for j in ups:
                rowcnt = np.bincount(g.blocks[(i, j)].row_idx, minlength=g.blocks[(i, j)].nrows)
                madds = int(np.dot(colcnt, rowcnt))
                pid, plv = last.get((k, j), (-1, -1))
                lv = max(l_[k][1], u[j][1], plv) + 1
                w = min(int(bn[k, i]), int(bn[i, j]))
                if 0 < bn[k, j] < w:
                    w = int(bn[k, j])
                t = emit(SSSSM, i, k, j, w, madds, lv,
                         [l_[k][0], u[j][0]] + ([pid] if pid >= 0 else []))
                last[(k, j)] = (t, lv)
    cnt = [len(t[7]) for t in tasks]
    return Tree(
        kinds=np.array([t[0] for t in tasks], np.int8),
        steps=np.array([t[1] for t in tasks], np.int32),
        rows=np.array([t[2] for t in tasks], np.int32),
        cols=np.array([t[3] for t in tasks], np.int32),
        weights=np.array([t[4] for t in tasks], np.int64),
        costs=np.array([t[5] for t in tasks], np.int64),
        levels_of=np.array([t[6] for t in tasks], np.int32),
        pred_ptr=np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64),
        pred_idx=np.array([q for t in tasks for q in t[7]], np.int32),
    )


def pipeline(a: Csc, *, sample_points=1000, plan="irregular", block_size=None, step=2, max_num=3):
    """A -> (filled pattern, pct, positions, grid, tree), the reference's default chain."""
    s = symmetrize(a)
    fcp, fri = symbolic(s)
    sp_, pct = curve(a.n, blockptr(a.n, fcp, fri), sample_points)
    if plan == "irregular":
        pos = irregular_positions(pct, a.n, step, max_num)
    else:
        pos = regular_positions(a.n, block_size)
    g = partition(a.n, fcp, fri, a, pos)
    return (fcp, fri), pct, pos, g, levels(g)
