"""Deterministic generators for the five BASELINE configurations.

The reference has no Poisson or BBD generator and no reordering
(pkg/src/lublock/matrix_io.py:27), so these build the inputs that
both engines consume through ``csc_from_triplets`` (matrix_io.py:99).

* C1  ``poisson2d(64)``                      5-point, natural order
* C2  ``poisson3d(64, order="nd")``          7-point + geometric nested dissection
* C3  ``bbd(1_000_000, border=10_000, ...)``  bordered block diagonal, row+column dominant
* C4  ``poisson3d(96, order="nd")``
* C5  ``bbd(200_000, border=4_000, blocks=200, seed=s)``
"""

from __future__ import annotations

import numpy as np

from .matrix_io import CscMatrix, csc_from_triplets


def _stencil_triplets(shape, diag):
    """Lexicographic (last axis fastest) grid Laplacian triplets."""
    dims = tuple(int(s) for s in shape)
    n = int(np.prod(dims))
    idx = np.arange(n, dtype=np.int64).reshape(dims)
    rows = [idx.ravel()]
    cols = [idx.ravel()]
    vals = [np.full(n, float(diag))]
    for ax in range(len(dims)):
        lo = [slice(None)] * len(dims)
        hi = [slice(None)] * len(dims)
        lo[ax] = slice(0, dims[ax] - 1)
        hi[ax] = slice(1, dims[ax])
        a = idx[tuple(lo)].ravel()
        b = idx[tuple(hi)].ravel()
        rows += [a, b]
        cols += [b, a]
        vals += [np.full(len(a), -1.0), np.full(len(a), -1.0)]
    return n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def poisson2d_triplets(k: int = 64):
    """(n, rows, cols, values) of ``poisson2d``."""
    return _stencil_triplets((k, k), 4.0)


def poisson2d(k: int = 64) -> CscMatrix:
    """C1: 5-point Laplacian on a k x k grid, Dirichlet; diag 4, neighbours -1; index r*k+c."""
    n, r, c, v = poisson2d_triplets(k)
    return csc_from_triplets(n, (r, c, v))


def nested_dissection_3d(k: int, leaf: int = 8) -> np.ndarray:
    """Geometric nested dissection of a k^3 grid; returns perm new->old.

    Recursively split the box's longest axis (first axis on ties) at
    m = size//2 and order [left box, right box, separator plane]; boxes whose
    every side is <= ``leaf`` are emitted lexicographically.
    """
    grid = np.arange(k ** 3, dtype=np.int64).reshape(k, k, k)
    out = []
    stack = [(0, k, 0, k, 0, k, False)]  # (x0,x1,y0,y1,z0,z1, emit-only)
    # explicit recursion order: left, right, separator -> push in reverse
    while stack:
        x0, x1, y0, y1, z0, z1, emit = stack.pop()
        if x1 <= x0 or y1 <= y0 or z1 <= z0:
            continue
        sz = (x1 - x0, y1 - y0, z1 - z0)
        if emit or max(sz) <= leaf:
            out.append(grid[x0:x1, y0:y1, z0:z1].ravel())
            continue
        ax = int(np.argmax(sz))
        lo = (x0, y0, z0)[ax]
        m = lo + sz[ax] // 2
        box = [x0, x1, y0, y1, z0, z1]
        left = list(box); left[2 * ax + 1] = m
        sep = list(box); sep[2 * ax] = m; sep[2 * ax + 1] = m + 1
        right = list(box); right[2 * ax] = m + 1
        stack.append((*sep, True))
        stack.append((*right, False))
        stack.append((*left, False))
    perm = np.concatenate(out)
    assert len(perm) == k ** 3
    return perm


def permute_symmetric(a: CscMatrix, perm: np.ndarray) -> CscMatrix:
    """B = A[perm, perm] with perm new->old."""
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm), dtype=perm.dtype)
    r = inv[a.row_idx]
    c = inv[a.entry_cols()]
    return csc_from_triplets(a.n, (r, c, a.values.copy()))


def poisson3d_triplets(k: int = 64, order: str = "nd", leaf: int = 8):
    """(n, rows, cols, values) of ``poisson3d`` before COO->CSC (also fed to the reference's own
    ``csc_from_triplets`` by the CPU-reference timing, oracle/ref_timing.py)."""
    n, r, c, v = _stencil_triplets((k, k, k), 6.0)
    if order == "natural":
        return n, r, c, v
    if order != "nd":
        raise ValueError(f"unknown order {order!r}")
    perm = nested_dissection_3d(k, leaf)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(n, dtype=np.int64)
    return n, inv[r], inv[c], v


def poisson3d(k: int = 64, order: str = "nd", leaf: int = 8) -> CscMatrix:
    """C2/C4: 7-point Laplacian on k^3 (diag 6, neighbours -1), ND-ordered by default."""
    n, r, c, v = poisson3d_triplets(k, order, leaf)
    return csc_from_triplets(n, (r, c, v))


def bbd(n: int, border: int, blocks: int, *, seed: int = 0, band: int = 4, keep: float = 0.5,
        ports: int = 4, port_links: int = 8, border_density: float = 0.001) -> CscMatrix:
    """CSC of ``bbd_triplets`` (same arguments)."""
    return csc_from_triplets(n, bbd_triplets(n, border, blocks, seed=seed, band=band, keep=keep, ports=ports,
                                             port_links=port_links, border_density=border_density))


def bbd_triplets(n: int, border: int, blocks: int, *, seed: int = 0, band: int = 4, keep: float = 0.5,
                 ports: int = 4, port_links: int = 8, border_density: float = 0.001):
    """C3/C5: bordered-block-diagonal 'circuit-like' matrix.

    Body: ``n-border`` rows cut into ``blocks`` contiguous diagonal blocks
    (linspace cuts), in-block band offsets 1..band each kept with prob ``keep``.
    Ports: the last ``ports`` columns of every body block couple to
    ``port_links`` distinct random border nodes.  Border: random symmetric
    pairs at ``border_density``.  Pattern symmetric; (i,j) and (j,i) carry
    independent U(-1,1) values.  Diagonal = max(row-sum, col-sum of |offdiag|)
    + U(0.5,1.5): row AND column dominant, so block-local pivoting never swaps.
    """
    rng = np.random.default_rng(seed)
    body = n - border
    cuts = np.linspace(0, body, blocks + 1).round().astype(np.int64)
    li, lj = [], []
    # band entries inside each diagonal block (strict lower triangle i > j)
    blk_of = np.repeat(np.arange(blocks), np.diff(cuts))
    for off in range(1, band + 1):
        i = np.arange(off, body, dtype=np.int64)
        same = blk_of[i] == blk_of[i - off]
        i = i[same]
        sel = rng.random(len(i)) < keep
        li.append(i[sel])
        lj.append(i[sel] - off)
    # ports: last `ports` columns of each block -> `port_links` distinct border nodes
    for b in range(blocks):
        c0 = max(cuts[b], cuts[b + 1] - ports)
        for col in range(c0, cuts[b + 1]):
            tgt = body + rng.choice(border, size=min(port_links, border), replace=False)
            li.append(tgt.astype(np.int64))
            lj.append(np.full(len(tgt), col, dtype=np.int64))
    # border block: random pairs, symmetric, no diagonal
    m = int(round(border_density * border * border / 2))
    if m and border > 1:
        a = rng.integers(0, border, size=m)
        b_ = rng.integers(0, border, size=m)
        lo = np.minimum(a, b_)
        hi = np.maximum(a, b_)
        ok = lo != hi
        key = np.unique(hi[ok] * border + lo[ok])
        li.append(body + key // border)
        lj.append(body + key % border)
    li = np.concatenate(li)
    lj = np.concatenate(lj)
    key = np.unique(li * n + lj)  # dedupe structural pairs
    li, lj = key // n, key % n
    v_lower = rng.uniform(-1.0, 1.0, len(li))
    v_upper = rng.uniform(-1.0, 1.0, len(li))
    absr = np.bincount(li, weights=np.abs(v_lower), minlength=n) + np.bincount(
        lj, weights=np.abs(v_upper), minlength=n)
    absc = np.bincount(lj, weights=np.abs(v_lower), minlength=n) + np.bincount(
        li, weights=np.abs(v_upper), minlength=n)
    diag = np.maximum(absr, absc) + rng.uniform(0.5, 1.5, n)
    rows = np.concatenate([li, lj, np.arange(n)])
    cols = np.concatenate([lj, li, np.arange(n)])
    vals = np.concatenate([v_lower, v_upper, diag])
    return rows, cols, vals


CONFIGS = {
    "C1": lambda: poisson2d(64),
    "C2": lambda: poisson3d(64, "nd"),
    "C3": lambda: bbd(1_000_000, 10_000, 1000, seed=0),
    "C4": lambda: poisson3d(96, "nd"),
    "C5": lambda: bbd(200_000, 4_000, 200, seed=0),
}
