"""Numerical factorization on the B200 — the drop-in for lublock.factorize.

Public names and signatures follow pkg/src/lublock/factorize.py:
``factorize`` (:245-384), ``LUFactors`` (:195-239), ``solve`` (:451-457),
``residual`` (:438-448) and the kernel-level entries ``factor_diagonal``
(:133-147), ``factor_u_panel`` (:150-156), ``factor_l_panel`` (:159-168),
``schur_update`` (:171-173).  Every one of them executes the hand-written
sm_100a kernels of csrc/lbk_device.cu through the C-ABI of include/lbk.h;
there is no CPU fallback — without liblbk.so or a CUDA device they raise.

Host work here is plumbing only: pooling the grid (a no-op for grids built
by this package), building the LUFactors views from the downloaded values
(exact zeros dropped like factorize.py:179-192) and the host solve/residual
the reference also runs on the host.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular

from . import _native
from .blocking import BlockingPlan
from .errors import DeviceError, DimensionMismatch, SupportViolation, ZeroPivot
from .grid import GESSM, GETRF, SSSSM, TSTRF, GridPool, SparseBlock, pool_grid
from .matrix_io import CscMatrix

DEFAULT_PIVOT_TOL = 1e-12
DEFAULT_CHUNK = 8
# compressed-tile tag: a block whose nonempty-rows x nonempty-columns rectangle
# holds >= this fraction of entries runs on the DMMA kernels (the reference's
# own dense tag is 0.5 of the FULL block, factorize.py:274).  0.05: at 0.1 the 74
# blocks of C4 that stayed CSC cost 620 ms of its 1,464 ms; as compressed tiles
# they add 2 % executed flops and the factorization takes 907 ms
# (profiles/r2_bench_c4_tau*.json); C2, C3 and C5 have no block below 0.1.
DEFAULT_DENSE_THRESHOLD = 0.05

P = _native.ptr
i64p, i32p, i8p, f64p = _native.c_i64p, _native.c_i32p, _native.c_i8p, _native.c_f64p


def _dev():
    lib = _native._dev
    if lib is not None:
        return lib
    import os

    if not os.path.exists(_native.DEV_LIB):
        raise DeviceError(f"{_native.DEV_LIB} missing: build with __graft_entry__.build(); "
                          "there is no CPU fallback for the numerical factorization")
    lib = C.CDLL(_native.DEV_LIB)
    st = C.POINTER(_native.LbkStatus)
    d = _native._declare
    vp = C.c_void_p
    d(lib, "lbk_create", C.c_int, [C.POINTER(vp), C.c_int, st])
    d(lib, "lbk_destroy", None, [vp])
    d(lib, "lbk_plan", C.c_int, [vp, C.c_int64, C.c_int64, i64p, C.c_int64, i64p, i64p, i64p, C.c_int64,
                                 i8p, i32p, i32p, i32p, i32p, i64p, C.c_int32, C.c_int32, C.c_double, st])
    d(lib, "lbk_upload_values", C.c_int, [vp, f64p, st])
    d(lib, "lbk_factorize", C.c_int, [vp, C.c_double, C.c_double, C.POINTER(C.c_float), st])
    d(lib, "lbk_factorize_host", C.c_int, [vp, f64p, f64p, i32p, C.c_double, C.c_double, st])
    d(lib, "lbk_download", C.c_int, [vp, f64p, i32p, st])
    d(lib, "lbk_set_perms", C.c_int, [vp, i32p, st])
    d(lib, "lbk_host_alloc", C.c_int, [C.POINTER(vp), C.c_int64])
    d(lib, "lbk_host_free", None, [vp])
    d(lib, "lbk_plan_info", C.c_int, [vp, i64p])
    d(lib, "lbk_level_times", C.c_int, [vp, C.c_double, C.c_double, C.POINTER(C.c_float), st])
    d(lib, "lbk_fp64_peak", C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)])
    d(lib, "lbk_task_routes", C.c_int, [vp, i8p])
    d(lib, "lbk_download_work", C.c_int, [vp, f64p, i64p, st])
    d(lib, "lbk_exec_trace", C.c_int, [vp, C.c_double, C.c_double, C.POINTER(C.c_uint64), i32p, i64p, st])
    d(lib, "lbk_plan_levels", C.c_int, [vp, i64p, i32p])
    d(lib, "lbk_exec_graph", C.c_int, [vp, i32p, i32p, i64p, i64p])
    d(lib, "lbk_set_task_mask", C.c_int, [vp, C.c_int64, i8p, st])
    d(lib, "lbk_set_cuts", C.c_int, [vp, C.c_int64, i8p, st])
    d(lib, "lbk_set_task_defer", C.c_int, [vp, C.c_int64, i8p, st])
    d(lib, "lbk_solve", C.c_int, [vp, f64p, f64p, st])
    d(lib, "lbk_bind_matrix", C.c_int, [vp, C.c_int64, i64p, st])
    d(lib, "lbk_refactor_host", C.c_int, [vp, f64p, f64p, i32p, C.c_double, C.c_double, st])
    d(lib, "lbk_num_segments", C.c_int, [vp])
    d(lib, "lbk_run_segment", C.c_int, [vp, C.c_int32, C.c_double, C.c_double, st])
    d(lib, "lbk_finish_raw", C.c_int, [vp, C.POINTER(C.c_float), C.POINTER(C.c_uint64), st])
    d(lib, "lbk_status_from_err", C.c_int, [C.POINTER(C.c_uint64), st])
    d(lib, "lbk_stream", vp, [vp])
    d(lib, "lbk_work_ptrs", C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)])
    d(lib, "lbk_block_layout", C.c_int, [vp, i64p])
    d(lib, "lbk_set_export", C.c_int, [vp, C.c_int64, i64p, i64p, st])
    d(lib, "lbk_num_out", C.c_int64, [vp])
    d(lib, "lbk_export_zero_counts", C.c_int, [vp, i64p, st])
    _native._dev = lib
    return lib


def defer_flags(tree) -> np.ndarray | None:
    """int8 per task: its slack, min(successor level) - own level, capped at
    100 (0 for tasks without successors is never produced: every update has
    one).  Slack >= 2: the task may run concurrently with the following
    slack - 1 levels (the engine defers such DMMA SSSSM updates onto low-
    priority side branches: lookahead across levels).  Needs the tree's
    predecessor lists (grid.py:172-181); None without them."""
    pp = getattr(tree, "pred_ptr", None)
    pi = getattr(tree, "pred_idx", None)
    if pp is None or pi is None:
        return None
    lv = np.asarray(tree.levels_of, np.int64)
    nt = len(lv)
    minsucc = np.full(nt, np.iinfo(np.int64).max, np.int64)
    np.minimum.at(minsucc, np.asarray(pi, np.int64), np.repeat(lv, np.diff(np.asarray(pp, np.int64))))
    return np.clip(minsucc - lv, 0, 100).astype(np.int8)


def fp64_peak(device: int = 0) -> tuple[float, float]:
    """Measured FP64 tensor (DMMA) and DFMA TFLOP/s of this device (csrc/lbk_peak.cu)."""
    a, b = C.c_double(), C.c_double()
    if _dev().lbk_fp64_peak(device, C.byref(a), C.byref(b)):
        raise DeviceError("lbk_fp64_peak failed")
    return a.value, b.value


def pinned_empty(nbytes_or_count, dtype=np.float64):
    """numpy array over page-locked host memory (freed with the array)."""
    lib = _dev()
    dt = np.dtype(dtype)
    count = int(nbytes_or_count)
    ptr = C.c_void_p()
    if lib.lbk_host_alloc(C.byref(ptr), count * dt.itemsize) != 0:
        raise MemoryError("cudaHostAlloc failed")
    buf = (C.c_char * max(count * dt.itemsize, 1)).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dt, count=count)

    class _Owner:
        def __init__(self, p):
            self.p = p

        def __del__(self):
            lib.lbk_host_free(self.p)

    arr_owner = _Owner(ptr)
    # keep the owner alive as long as the array: stash on a subclass view
    out = arr.view(_PinnedArray)
    out._owner = arr_owner
    return out


class _PinnedArray(np.ndarray):
    _owner = None


_PINNED_FREE: dict = {}  # (count, dtype) -> page-locked arrays no longer referenced by any result
_PINNED_KEEP = 2


class _Recycle:
    """Owner of a recycled page-locked array: when the last view of it dies (e.g. the
    LUFactors built on it), the array returns to the free list instead of being
    unpinned - cudaHostAlloc of gigabytes costs far more than a factorization."""

    def __init__(self, key, arr):
        self.key, self.arr = key, arr

    def __del__(self):
        try:
            free = _PINNED_FREE.setdefault(self.key, [])
            if len(free) < _PINNED_KEEP:
                free.append(self.arr)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


def pinned_recycled(count, dtype=np.float64) -> np.ndarray:
    """Page-locked array from the recycle list (allocated on a miss); returned to
    the list when no view of it is alive any more."""
    key = (int(count), np.dtype(dtype).str)
    free = _PINNED_FREE.get(key)
    arr = free.pop() if free else pinned_empty(count, dtype)
    out = arr.view(_PinnedArray)
    out._owner = _Recycle(key, arr)
    return out


class Engine:
    """One device plan (block structure + task schedule) on one GPU.

    Built once per (grid, tree); ``run`` refactors new values with the same
    pattern.  This is the unit bench.py times.
    """

    def __init__(self, grid, tree, *, device: int = 0, chunk: int = DEFAULT_CHUNK, pool: GridPool | None = None,
                 dense: bool = False, dense_threshold: float | None = DEFAULT_DENSE_THRESHOLD,
                 dense_kernels: bool = True, mask: np.ndarray | None = None, cuts: np.ndarray | None = None,
                 lookahead: bool = True, refine: bool = True):
        """dense=True: dense-scratch mode (every block a full tile, true row swaps).
        dense_threshold: tau of the compressed-tile tag (see include/lbk.h lbk_plan);
        None / dense_kernels=False keeps every block CSC (sparse kernels only).
        mask (int8 per task) / cuts (int8 per tree level): distributed plans
        (parallel.DistEngine) — run only the masked tasks, and split the graph
        into segments after the cut levels.
        refine: segment-level scheduling of banded diagonal blocks (lbk_plan flags bit 2;
        such a plan cannot run static pivoting — use refine=False for that)."""
        self.lib = _dev()
        self.grid = grid
        self.tree = tree
        self.pool = pool if pool is not None else pool_grid(grid)
        use_tiles = dense_kernels and dense_threshold is not None
        self.dense_threshold = 0.0 if dense else (dense_threshold if use_tiles else None)
        self.device = device
        ctx = C.c_void_p()
        st = _native.LbkStatus()
        rc = self.lib.lbk_create(C.byref(ctx), device, C.byref(st))
        if rc:
            _native.raise_status(st, "lbk_create")
        self.ctx = ctx
        if mask is not None:
            mk = np.ascontiguousarray(mask, dtype=np.int8)
            if self.lib.lbk_set_task_mask(ctx, len(mk), P(mk, i8p), C.byref(st)):
                _native.raise_status(st, "lbk_set_task_mask")
        df = defer_flags(tree) if lookahead else None
        if df is not None:
            self._defer = df
            if self.lib.lbk_set_task_defer(ctx, len(df), P(df, i8p), C.byref(st)):
                _native.raise_status(st, "lbk_set_task_defer")
        if cuts is not None:
            ct = np.ascontiguousarray(cuts, dtype=np.int8)
            if self.lib.lbk_set_cuts(ctx, len(ct), P(ct, i8p), C.byref(st)):
                _native.raise_status(st, "lbk_set_cuts")
        pos = np.ascontiguousarray(grid.plan.positions, dtype=np.int64)
        pl = self.pool
        self._keep = [np.ascontiguousarray(pl.table, dtype=np.int64),
                      np.ascontiguousarray(pl.col_ptr, dtype=np.int64),
                      np.ascontiguousarray(pl.row_idx, dtype=np.int64),
                      np.ascontiguousarray(tree.kinds, dtype=np.int8),
                      np.ascontiguousarray(tree.steps, dtype=np.int32),
                      np.ascontiguousarray(tree.rows, dtype=np.int32),
                      np.ascontiguousarray(tree.cols, dtype=np.int32),
                      np.ascontiguousarray(tree.levels_of, dtype=np.int32),
                      np.ascontiguousarray(tree.costs, dtype=np.int64)]
        if dense:
            # full-rectangle blocks: after a row swap a structurally empty
            # product can become numerically nonzero, so run every update
            # whose target exists (factorize.py:311-325 semantics)
            kk = self._keep[3]
            tgt = np.ones(len(kk), np.int64)
            upd = kk == SSSSM
            bn = np.zeros((grid.p, grid.p), np.int64)
            bn[pl.table[0], pl.table[1]] = 1
            tgt[upd] = bn[self._keep[5][upd], self._keep[6][upd]]
            self._keep[8] = tgt
        t, cp, ri, k, s, r, c, lv, co = self._keep
        rc = self.lib.lbk_plan(ctx, grid.n, grid.p, P(pos, i64p), pl.nblocks, P(t, i64p), P(cp, i64p),
                               P(ri, i64p), len(k), P(k, i8p), P(s, i32p), P(r, i32p), P(c, i32p),
                               P(lv, i32p), P(co, i64p), int(chunk),
                               (1 if (use_tiles or dense) else 0) | (2 if dense else 0) | (4 if refine else 0),
                               float(dense_threshold if use_tiles else 1.0), C.byref(st))
        if rc:
            _native.raise_status(st, "lbk_plan")
        self.nnz = int(pl.values.shape[0])
        self.nout = self.nnz  # output entries (enable_export: the LUFactors layout)
        self.export = None
        self.bound_a = None  # a_pos array bound with bind_matrix (refactorization input)
        info = np.zeros(14, np.int64)
        self.lib.lbk_plan_info(ctx, P(info, i64p))
        self.info = info
        self.n_launch_levels, self.n_items, self.n_diag_rows = int(info[0]), int(info[1]), int(info[2])
        self.n_gemm_tiles, self.n_dense_items, self.n_launches = int(info[4]), int(info[5]), int(info[6])
        self.nnz_work = int(info[7])
        self.n_sparse_blocks, self.n_rect_blocks, self.n_full_blocks = int(info[8]), int(info[9]), int(info[10])
        self.n_tile_items = int(info[11])
        self.dmma_flops_executed, self.exec_flops_executed = float(info[12]), float(info[13])
        self._resident = False
        self.generation = 0  # bumped by every factorization: device factors of LUFactors stay valid until then

    def enable_export(self) -> None:
        """Make every output of this engine the LUFactors layout of the reference's
        export (factorize.py:370-384): off-diagonal blocks as stored, diagonal blocks
        split into triu(d) then tril(d,-1)+I.  Structures are computed once here; a
        factorization then returns values the blocks view without a host-side copy."""
        if getattr(self, "export", None) is not None:
            return
        t = self.pool.table
        cpool, rpool = self.pool.col_ptr, self.pool.row_idx
        xref, xoff, shapes = [], [0], []
        for b in range(self.pool.nblocks):
            bi, bj, nr, nc, nz, cpo, eo = (int(x) for x in t[:, b])
            cp = cpool[cpo:cpo + nc + 1]
            ri = rpool[eo:eo + nz]
            if bi != bj:
                xref.append(np.arange(eo, eo + nz, dtype=np.int64))
                shapes.append((cp, ri, None, None))
                xoff.append(xoff[-1] + nz)
                continue
            m = nr
            cols = np.repeat(np.arange(m, dtype=np.int64), np.diff(cp))
            up = ri <= cols
            ucp = np.zeros(m + 1, np.int64)
            np.cumsum(np.bincount(cols[up], minlength=m), out=ucp[1:])
            lo = ~up
            lcp = np.zeros(m + 1, np.int64)
            np.cumsum(np.bincount(cols[lo], minlength=m) + 1, out=lcp[1:])
            unit = lcp[:-1]
            lref = np.empty(lcp[-1], np.int64)
            lrow = np.empty(lcp[-1], np.int64)
            other = np.ones(lcp[-1], bool)
            other[unit] = False
            lref[unit] = -1
            lrow[unit] = np.arange(m)
            lref[other] = eo + np.flatnonzero(lo)
            lrow[other] = ri[lo]
            xref.append(eo + np.flatnonzero(up))
            xref.append(lref)
            shapes.append((ucp, ri[up], lcp, lrow))
            xoff.append(xoff[-1] + int(up.sum()) + len(lref))
        # per block: (key, L/U/diag, rows, cols, x0, split, x1, read-only structures) for build_factors_export
        recs = []
        for b in range(self.pool.nblocks):
            bi, bj, nr, nc = (int(x) for x in t[:4, b])
            cp, ri, lcp, lrow = shapes[b]
            x0, x1 = xoff[b], xoff[b + 1]
            kind = 0 if bi > bj else (1 if bi < bj else 2)
            recs.append(((bi, bj), kind, nr, nc, x0, x0 + len(ri), x1, _ro(cp), _ro(ri),
                         None if lcp is None else _ro(lcp), None if lrow is None else _ro(lrow)))
        self.export_recs = recs
        xr = np.concatenate(xref) if xref else np.zeros(0, np.int64)
        xo = np.asarray(xoff, np.int64)
        st = _native.LbkStatus()
        if self.lib.lbk_set_export(self.ctx, len(xr), P(xr, i64p), P(xo, i64p), C.byref(st)):
            _native.raise_status(st, "lbk_set_export")
        self.export = (xo, shapes)
        self.nout = int(len(xr))

    def export_zero_counts(self) -> np.ndarray:
        zc = np.zeros(self.pool.nblocks, np.int64)
        st = _native.LbkStatus()
        if self.lib.lbk_export_zero_counts(self.ctx, P(zc, i64p), C.byref(st)):
            _native.raise_status(st, "lbk_export_zero_counts")
        return zc

    def solve(self, b) -> np.ndarray:
        """x = U^-1 L^-1 b[perm_global] on the device-resident factors of the
        last factorization (factorize.py:451-457)."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.shape != (self.grid.n,):
            raise DimensionMismatch(f"rhs must have length {self.grid.n}")
        x = np.empty(self.grid.n, np.float64)
        st = _native.LbkStatus()
        if self.lib.lbk_solve(self.ctx, P(b, f64p), P(x, f64p), C.byref(st)):
            _native.raise_status(st, "lbk_solve")
        return x

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.lbk_destroy(self.ctx)
            self.ctx = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _eps(static_pivot, value_max):
        if static_pivot is None:
            return math.nan
        return float(static_pivot) * (value_max or 1.0)

    def upload(self, values=None):
        v = np.ascontiguousarray(self.pool.values if values is None else values, dtype=np.float64)
        st = _native.LbkStatus()
        self.generation += 1  # replaces the resident values: factors of earlier runs are stale
        if self.lib.lbk_upload_values(self.ctx, P(v, f64p), C.byref(st)):
            _native.raise_status(st, "lbk_upload_values")
        self._resident = True

    def run_device(self, pivot_tol=DEFAULT_PIVOT_TOL, static_pivot=None) -> float:
        """Factor the resident values on the device; returns graph device ms."""
        if not self._resident:
            self.upload()
        ms = C.c_float()
        st = _native.LbkStatus()
        self.generation += 1
        self.lib.lbk_factorize(self.ctx, pivot_tol, self._eps(static_pivot, self.grid.value_max),
                               C.byref(ms), C.byref(st))
        _native.raise_status(st, "lbk_factorize")
        return float(ms.value)

    def run_host(self, a_values, out_values, out_perms, pivot_tol=DEFAULT_PIVOT_TOL, static_pivot=None):
        """End-to-end: host values in -> host factor values + perms out. Returns lbk_status."""
        st = _native.LbkStatus()
        self.generation += 1
        self.lib.lbk_factorize_host(self.ctx, P(a_values, f64p), P(out_values, f64p),
                                    P(out_perms, i32p) if out_perms is not None else None,
                                    pivot_tol, self._eps(static_pivot, self.grid.value_max), C.byref(st))
        return st

    def bind_matrix(self, pool_pos) -> None:
        """Reference-pool position of every entry of A (grid.pool_positions): enables refactor_host."""
        pp = np.ascontiguousarray(pool_pos, dtype=np.int64)
        st = _native.LbkStatus()
        if self.lib.lbk_bind_matrix(self.ctx, len(pp), P(pp, i64p), C.byref(st)):
            _native.raise_status(st, "lbk_bind_matrix")
        self.nnz_a = len(pp)

    def refactor_host(self, a_values, out_values, out_perms, pivot_tol=DEFAULT_PIVOT_TOL, static_pivot=None):
        """End to end from A's own values (CSC order, nnz(A)): new values on the
        same pattern in, factor values (reference pool order) + perms out."""
        st = _native.LbkStatus()
        self.generation += 1
        self.lib.lbk_refactor_host(self.ctx, P(a_values, f64p), P(out_values, f64p),
                                   P(out_perms, i32p) if out_perms is not None else None,
                                   pivot_tol, self._eps(static_pivot, self.grid.value_max), C.byref(st))
        return st

    def level_times(self, pivot_tol=DEFAULT_PIVOT_TOL, static_pivot=None, check=True) -> np.ndarray:
        """[levels x 5] device ms from one instrumented replay: level, DMMA SSSSM,
        panel solves, tiled GETRF, CSC kernel.  check=False: timing only (a
        distributed plan replayed without its exchanges computes garbage)."""
        if not self._resident:
            self.upload()
        out = np.zeros((self.n_launch_levels, 5), np.float32)
        st = _native.LbkStatus()
        self.generation += 1
        self.lib.lbk_level_times(self.ctx, pivot_tol, self._eps(static_pivot, self.grid.value_max),
                                 out.ctypes.data_as(C.POINTER(C.c_float)), C.byref(st))
        if check or st.code in (_native.LBK_ERR_CUDA, _native.LBK_ERR_OOM):
            _native.raise_status(st, "lbk_level_times")
        return out

    # ---- segment-wise execution (distributed plans) ----

    @property
    def n_segments(self) -> int:
        return int(self.lib.lbk_num_segments(self.ctx))

    def run_segment(self, seg: int, pivot_tol=DEFAULT_PIVOT_TOL, static_pivot=None) -> None:
        """Enqueue graph segment `seg` on the engine stream (asynchronous)."""
        st = _native.LbkStatus()
        if seg == 0:
            self.generation += 1
        if self.lib.lbk_run_segment(self.ctx, int(seg), pivot_tol, self._eps(static_pivot, self.grid.value_max),
                                    C.byref(st)):
            _native.raise_status(st, "lbk_run_segment")

    def finish_raw(self):
        """Synchronize; (device ms of segments 0..last, raw error words uint64[2])."""
        ms = C.c_float()
        err = (C.c_uint64 * 2)()
        st = _native.LbkStatus()
        if self.lib.lbk_finish_raw(self.ctx, C.byref(ms), err, C.byref(st)):
            _native.raise_status(st, "lbk_finish_raw")
        return float(ms.value), np.array([err[0], err[1]], np.uint64)

    def status_from_err(self, err) -> "_native.LbkStatus":
        e = (C.c_uint64 * 2)(int(err[0]), int(err[1]))
        st = _native.LbkStatus()
        self.lib.lbk_status_from_err(e, C.byref(st))
        return st

    @property
    def stream_ptr(self) -> int:
        return int(self.lib.lbk_stream(self.ctx) or 0)

    def work_ptrs(self):
        """Device addresses of (working pool f64, per-diagonal-row perms i32, output pool f64)."""
        v, p, o = C.c_void_p(), C.c_void_p(), C.c_void_p()
        self.lib.lbk_work_ptrs(self.ctx, C.byref(v), C.byref(p), C.byref(o))
        return int(v.value or 0), int(p.value or 0), int(o.value or 0)

    def block_layout(self) -> np.ndarray:
        """[3 x nblocks]: working offset, working entries, diagonal-row offset (-1 off-diagonal)."""
        out = np.zeros((3, self.pool.nblocks), np.int64)
        self.lib.lbk_block_layout(self.ctx, P(out, i64p))
        return out

    def download_work(self) -> np.ndarray:
        """Working-layout values (dense-scratch mode: full tiles in pool block order)."""
        n = C.c_int64()
        st = _native.LbkStatus()
        self.lib.lbk_download_work(self.ctx, None, C.byref(n), C.byref(st))
        out = np.empty(n.value, np.float64)
        if self.lib.lbk_download_work(self.ctx, P(out, f64p), C.byref(n), C.byref(st)):
            _native.raise_status(st, "lbk_download_work")
        return out

    def exec_trace(self, pivot_tol=DEFAULT_PIVOT_TOL):
        """(trace[n,8] ns, info[n,6]) of the persistent executor's tile tasks (one instrumented replay):
        dequeue, ready, done, in-task phase stamps 0..3 (GETRF / TRSM_L), writes fenced."""
        if not self._resident:
            self.upload()
        n = C.c_int64()
        st = _native.LbkStatus()
        self.generation += 1
        self.lib.lbk_exec_trace(self.ctx, pivot_tol, math.nan, None, None, C.byref(n), C.byref(st))
        tr = np.zeros((n.value, 8), np.uint64)
        info = np.zeros((n.value, 6), np.int32)
        self.lib.lbk_exec_trace(self.ctx, pivot_tol, math.nan, tr.ctypes.data_as(C.POINTER(C.c_uint64)),
                                P(info, i32p), C.byref(n), C.byref(st))
        _native.raise_status(st, "lbk_exec_trace")
        return tr, info

    def exec_graph(self):
        """(sptr, succ) of the executor's task DAG: per launch level nexec + 1 local successor
        offsets, entries (local successor << 1) | phase (analysis tooling, scripts/exec_dag.py)."""
        ns, ne = C.c_int64(), C.c_int64()
        self.lib.lbk_exec_graph(self.ctx, None, None, C.byref(ns), C.byref(ne))
        sptr = np.zeros(max(ns.value, 1), np.int32)
        succ = np.zeros(max(ne.value, 1), np.int32)
        rc = self.lib.lbk_exec_graph(self.ctx, P(sptr, i32p), P(succ, i32p), C.byref(ns), C.byref(ne))
        if rc:
            raise DeviceError(f"lbk_exec_graph: code {rc}")
        return sptr[: ns.value], succ[: ne.value]

    def task_routes(self) -> np.ndarray:
        """Kernel family per task: -1 skipped, 0 CSC, 1 DMMA SSSSM, 2 panel, 3 tiled GETRF."""
        r = np.zeros(self.tree.task_count, np.int8)
        self.lib.lbk_task_routes(self.ctx, P(r, i8p))
        return r

    def plan_levels(self):
        """(levels[4, L], items[6, T]) of the launched schedule."""
        lv = np.zeros((4, self.n_launch_levels), np.int64)
        it = np.zeros((6, self.n_items), np.int32)
        self.lib.lbk_plan_levels(self.ctx, P(lv, i64p), P(it, i32p))
        return lv, it

    def download(self):
        vals = np.empty(self.nout, np.float64)
        perms = np.empty(max(self.n_diag_rows, 1), np.int32)
        st = _native.LbkStatus()
        if self.lib.lbk_download(self.ctx, P(vals, f64p), P(perms, i32p), C.byref(st)):
            _native.raise_status(st, "lbk_download")
        return vals, perms[: self.n_diag_rows]

    def set_perms(self, perms):
        p = np.ascontiguousarray(perms, dtype=np.int32)
        st = _native.LbkStatus()
        if self.lib.lbk_set_perms(self.ctx, P(p, i32p), C.byref(st)):
            _native.raise_status(st, "lbk_set_perms")


# --- factor container ----------------------------------------------------------


@dataclass
class LUFactors:
    """Blocked factors P_block . A_filled = L U (factorize.py:195-239)."""

    n: int
    plan: BlockingPlan
    l_blocks: dict
    u_blocks: dict
    perms: list
    _assembled: dict = field(default_factory=dict, repr=False)
    _device: tuple | None = field(default=None, repr=False)  # (Engine, generation) holding these factors

    def perm_global(self) -> np.ndarray:
        if "perm" not in self._assembled:
            off = self.plan.positions
            self._assembled["perm"] = np.concatenate([off[i] + self.perms[i] for i in range(self.plan.p)])
        return self._assembled["perm"]

    def _assemble(self, blocks) -> sp.csr_matrix:
        off = self.plan.positions
        r, c, v = [], [], []
        for (bi, bj), b in blocks.items():
            r.append(b.row_idx + off[bi])
            c.append(np.repeat(np.arange(b.ncols), np.diff(b.col_ptr)) + off[bj])
            v.append(b.values)
        cat = lambda xs, dt: np.concatenate(xs) if xs else np.empty(0, dt)  # noqa: E731
        return sp.coo_matrix((cat(v, np.float64), (cat(r, np.int64), cat(c, np.int64))),
                             shape=(self.n, self.n)).tocsr()

    def l_matrix(self) -> sp.csr_matrix:
        if "L" not in self._assembled:
            self._assembled["L"] = self._assemble(self.l_blocks)
        return self._assembled["L"]

    def u_matrix(self) -> sp.csr_matrix:
        if "U" not in self._assembled:
            self._assembled["U"] = self._assemble(self.u_blocks)
        return self._assembled["U"]


def _drop_zeros(nrows, ncols, cp, ri, vv) -> SparseBlock:
    keep = vv != 0.0
    if keep.all():
        return SparseBlock(nrows, ncols, cp, ri, vv)
    cols = np.repeat(np.arange(ncols), np.diff(cp))[keep]
    ncp = np.zeros(ncols + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=ncols), out=ncp[1:])
    return SparseBlock(nrows, ncols, ncp, ri[keep], vv[keep])


def _split_diagonal(m, cp, ri, vv):
    """(L, U) of a factored diagonal block: tril(d,-1)+I and triu(d) (factorize.py:377-381)."""
    cols = np.repeat(np.arange(m), np.diff(cp))
    up = ri <= cols
    U = _drop_zeros(m, m, np.concatenate([[0], np.cumsum(np.bincount(cols[up], minlength=m))]).astype(np.int64),
                    ri[up], vv[up])
    lo = (ri > cols) & (vv != 0.0)
    lr = np.concatenate([ri[lo], np.arange(m)])
    lc = np.concatenate([cols[lo], np.arange(m)])
    lv = np.concatenate([vv[lo], np.ones(m)])
    order = np.lexsort((lr, lc))
    Lcp = np.concatenate([[0], np.cumsum(np.bincount(lc, minlength=m))]).astype(np.int64)
    return SparseBlock(m, m, Lcp, lr[order].astype(np.int64), lv[order]), U


def build_factors(grid, pool: GridPool, values: np.ndarray, perms_pool: np.ndarray | None) -> LUFactors:
    """LUFactors from factor values laid out like the pool (factorize.py:364-384)."""
    t = pool.table
    lb, ub = {}, {}
    for b in range(pool.nblocks):
        bi, bj, nr, nc, nz, cpo, eo = (int(x) for x in t[:, b])
        cp = pool.col_ptr[cpo:cpo + nc + 1]
        ri = pool.row_idx[eo:eo + nz]
        vv = values[eo:eo + nz]
        if bi > bj:
            lb[(bi, bj)] = _drop_zeros(nr, nc, cp, ri, vv)
        elif bi < bj:
            ub[(bi, bj)] = _drop_zeros(nr, nc, cp, ri, vv)
        else:
            lb[(bi, bi)], ub[(bi, bi)] = _split_diagonal(nr, cp, ri, vv)
    spans = np.diff(grid.plan.positions)
    perms = []
    off = 0
    for i in range(grid.p):
        s = int(spans[i])
        if perms_pool is not None and len(perms_pool):
            perms.append(perms_pool[off:off + s].astype(np.int64))
        else:
            perms.append(np.arange(s))
        off += s
    return LUFactors(n=grid.n, plan=grid.plan, l_blocks=lb, u_blocks=ub, perms=perms)


def _ro(a: np.ndarray) -> np.ndarray:
    v = a.view()
    v.flags.writeable = False
    return v


def _perm_list(grid, perms_pool):
    spans = np.diff(grid.plan.positions)
    perms = []
    off = 0
    for i in range(grid.p):
        s = int(spans[i])
        if perms_pool is not None and len(perms_pool):
            perms.append(perms_pool[off:off + s].astype(np.int64))
        else:
            perms.append(np.arange(s))
        off += s
    return perms


def build_factors_export(grid, eng, out: np.ndarray, zero_counts: np.ndarray, perms_pool) -> LUFactors:
    """LUFactors over the export-layout output of ``eng`` (Engine.enable_export):
    block values are views of ``out`` (which they keep alive), structures are the
    cached read-only export structures; blocks holding exact zeros are compacted
    like the reference's export (factorize.py:179-192)."""
    lb, ub = {}, {}
    zb = set(np.flatnonzero(zero_counts).tolist())
    for b, (key, kind, nr, nc, x0, xs, x1, cp, ri, lcp, lrow) in enumerate(eng.export_recs):
        if b in zb:
            if kind == 2:
                ub[key] = _drop_zeros(nr, nr, cp, ri, out[x0:xs])
                lb[key] = _drop_zeros(nr, nr, lcp, lrow, out[xs:x1])
            else:
                (lb if kind == 0 else ub)[key] = _drop_zeros(nr, nc, cp, ri, out[x0:x1])
        elif kind == 2:
            ub[key] = SparseBlock(nr, nr, cp, ri, out[x0:xs])
            lb[key] = SparseBlock(nr, nr, lcp, lrow, out[xs:x1])
        else:
            (lb if kind == 0 else ub)[key] = SparseBlock(nr, nc, cp, ri, out[x0:x1])
    return LUFactors(n=grid.n, plan=grid.plan, l_blocks=lb, u_blocks=ub, perms=_perm_list(grid, perms_pool))


def _block_from_tile(d: np.ndarray) -> SparseBlock:
    """Dense tile -> CSC dropping exact zeros (factorize.py:179-192)."""
    cols, rows = np.nonzero(d.T)
    cp = np.zeros(d.shape[1] + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=d.shape[1]), out=cp[1:])
    return SparseBlock(d.shape[0], d.shape[1], cp, rows.astype(np.int64), d.T[cols, rows])


def build_factors_full(grid, pool: GridPool, work: np.ndarray, perms_pool: np.ndarray) -> LUFactors:
    """LUFactors from dense-scratch mode (every block a full tile in pool block
    order): supports that moved under row swaps are rebuilt like the reference."""
    t = pool.table
    lb, ub = {}, {}
    off = 0
    for b in range(pool.nblocks):
        bi, bj, nr, nc = (int(x) for x in t[:4, b])
        d = work[off:off + nr * nc].reshape(nc, nr).T
        off += nr * nc
        if bi > bj:
            lb[(bi, bj)] = _block_from_tile(d)
        elif bi < bj:
            ub[(bi, bj)] = _block_from_tile(d)
        else:
            lb[(bi, bi)] = _block_from_tile(np.tril(d, -1) + np.eye(nr))
            ub[(bi, bi)] = _block_from_tile(np.triu(d))
    f = build_factors(grid, GridPool(table=t[:, :0], col_ptr=pool.col_ptr, row_idx=pool.row_idx,
                                     values=pool.values), pool.values[:0], perms_pool)
    return LUFactors(n=grid.n, plan=grid.plan, l_blocks=lb, u_blocks=ub, perms=f.perms)


def check_support(grid, tree) -> None:
    """The reference's support checks (factorize.py:277-324), structurally, once per grid.

    The reference raises SupportViolation when an SSSSM product is nonzero outside the
    target block's filled support (or hits an absent block).  A grid built by this
    package's ``partition`` is elimination-closed by construction (grid.py:3-5), so no
    product can leave the support.  For any other grid (e.g. hand-made), the union of
    the block patterns is checked for closure with the native symbolic factorization;
    only if it is not closed are the products walked in construction order, and the
    first one whose STRUCTURAL support leaves its target raises, with the reference's
    message.  (The reference tests the numeric product, so it would stay silent on an
    exact cancellation, and it stops checking after the first row swap.)"""
    if getattr(grid, "a_pos", None) is not None or getattr(grid, "_lbk_support_ok", False):
        return
    from .symbolic import symbolic_factorize, symmetrize_pattern

    pool = pool_grid(grid)
    t = pool.table
    pos = np.asarray(grid.plan.positions, np.int64)
    nc = t[3]
    cols_local = np.concatenate([np.repeat(np.arange(int(c)), np.diff(pool.col_ptr[int(o):int(o) + int(c) + 1]))
                                 for c, o in zip(nc, t[5])]) if t.shape[1] else np.zeros(0, np.int64)
    r = pool.row_idx + np.repeat(pos[t[0]], t[4])
    c = cols_local + np.repeat(pos[t[1]], t[4])
    m = sp.coo_matrix((np.ones(len(r)), (r, c)), shape=(grid.n, grid.n)).tocsc()
    m.sum_duplicates()
    a = CscMatrix(grid.n, m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data)
    closed = False
    try:
        closed = symbolic_factorize(symmetrize_pattern(a)).nnz_filled == a.nnz
    except Exception:
        closed = False
    if not closed:
        def pat(key):
            b = grid.blocks[key]
            return sp.csc_matrix((np.ones(b.nnz), np.asarray(b.row_idx), np.asarray(b.col_ptr)),
                                 shape=(b.nrows, b.ncols))
        for q in np.flatnonzero(np.asarray(tree.kinds) == SSSSM):
            i, rr, cc = int(tree.steps[q]), int(tree.rows[q]), int(tree.cols[q])
            prod = (pat((rr, i)) @ pat((i, cc))).tocoo()
            if (rr, cc) not in grid.blocks:
                if prod.nnz:
                    raise SupportViolation(f"update from step {i} hits empty block ({rr}, {cc})")
                continue
            tgt = pat((rr, cc)).tocsr()
            if np.any(np.asarray(tgt[prod.row, prod.col]).ravel() == 0):
                raise SupportViolation(f"update from step {i} writes outside filled support of block ({rr}, {cc})")
    try:
        grid._lbk_support_ok = True
    except AttributeError:
        pass


def engine_for(grid, tree, *, device: int = 0, dense: bool = False, chunk: int = DEFAULT_CHUNK,
               dense_threshold: float | None = DEFAULT_DENSE_THRESHOLD, refine: bool = True) -> Engine:
    """Cached device plan of (grid, tree); dense=True uses full-rectangle blocks everywhere.

    One plan per (device, dense, chunk, dense_threshold) and grid: a call with a different
    tree object closes the cached plan (frees its device memory) and replaces it, so
    calling ``factorize(grid, dependency_levels(grid))`` in a loop does not grow memory."""
    cache = getattr(grid, "_lbk_engines", None)
    if cache is None:
        cache = {}
        try:
            grid._lbk_engines = cache
        except AttributeError:
            pass
    key = (device, dense, chunk, dense_threshold, refine)
    eng = cache.get(key)
    if eng is not None and eng.tree is not tree:
        eng.close()
        eng = None
    if eng is None:
        cache.pop(key, None)
        # one plan per grid and mode: the variant with the other `refine` setting (static pivoting
        # toggled between calls) is released first, so C4-sized plans never coexist
        other = cache.pop((device, dense, chunk, dense_threshold, not refine), None)
        if other is not None:
            other.close()
        eng = Engine(grid, tree, device=device, chunk=chunk, dense=dense, dense_threshold=dense_threshold,
                     refine=refine)
        cache[key] = eng
    return eng


def factorize(grid, tree, workers: int = 1, pivot_tol: float = DEFAULT_PIVOT_TOL,
              static_pivot: float | None = None, dense_blas: bool = False, *, device: int = 0,
              chunk: int = DEFAULT_CHUNK, dense_threshold: float | None = DEFAULT_DENSE_THRESHOLD) -> LUFactors:
    """Blocked right-looking LU on the B200 (factorize.py:245-384).

    ``workers`` is accepted for signature compatibility and ignored: the
    device schedule is level-parallel and the result does not depend on it.
    ``dense_blas`` is accepted and ignored (results never depend on it beyond
    rounding).  Row swaps inside a diagonal block whose block row is stored
    sparse re-run the factorization on full-rectangle blocks (the
    reference's dense-scratch semantics) — still on the device.
    """
    if workers < 1:
        raise DimensionMismatch(f"workers must be >= 1, got {workers}")
    check_support(grid, tree)
    # static pivoting runs the exact whole-block GETRF: no segment-refined levels for it
    eng = engine_for(grid, tree, device=device, dense=False, chunk=chunk, dense_threshold=dense_threshold,
                     refine=static_pivot is None)
    eng.enable_export()
    out = pinned_recycled(eng.nout)
    perms = np.empty(max(eng.n_diag_rows, 1), np.int32)
    a_pos = getattr(grid, "a_pos", None)
    if a_pos is not None and eng.pool is getattr(grid, "pool", None) and not eng.pool.values.flags.writeable:
        # a grid built by partition(): its read-only pool holds A's values at a_pos and
        # exact zeros (the fill) elsewhere, so only A's nnz values travel to the device
        if eng.bound_a is not a_pos:
            eng.bind_matrix(a_pos)
            eng.bound_a = a_pos
            eng.a_stage = pinned_empty(len(a_pos))
            eng.a_staged_from = None
        if eng.a_staged_from is not eng.pool.values:  # read-only values: the staged copy stays valid
            np.take(eng.pool.values, a_pos, out=eng.a_stage)
            eng.a_staged_from = eng.pool.values
        st = eng.refactor_host(eng.a_stage, out, perms, pivot_tol, static_pivot)  # H2D of A's values inside
    else:  # foreign (e.g. reference-built) grid: the whole pooled value array
        st = eng.run_host(np.ascontiguousarray(eng.pool.values, dtype=np.float64), out, perms, pivot_tol,
                          static_pivot)
    if st.code != _native.LBK_ERR_PIVOT_SWAP:
        _native.raise_status(st, "factorize")
        lu = build_factors_export(grid, eng, out, eng.export_zero_counts(), perms[: eng.n_diag_rows])
        lu._device = (eng, eng.generation)
        return lu
    # a row swap inside a diagonal block whose block row is stored compressed:
    # the reference's dense-scratch semantics on full-rectangle blocks (still on the device)
    eng = engine_for(grid, tree, device=device, dense=True, chunk=chunk, dense_threshold=dense_threshold)
    vals_in = np.ascontiguousarray(eng.pool.values, dtype=np.float64)
    out = np.empty(eng.nnz, np.float64)
    st = eng.run_host(vals_in, out, perms, pivot_tol, static_pivot)
    _native.raise_status(st, "factorize")
    lu = build_factors_full(grid, eng.pool, eng.download_work(), perms[: eng.n_diag_rows])
    lu._device = (eng, eng.generation)
    return lu


# --- validation (host, like the reference) -------------------------------------


def residual(a: CscMatrix, f: LUFactors) -> float:
    """||P A - L U||_F / ||A||_F (factorize.py:438-448)."""
    if a.n != f.n:
        raise DimensionMismatch(f"order mismatch: {a.n} vs {f.n}")
    pa = a.to_scipy().tocsr()[f.perm_global(), :]
    d = (pa - f.l_matrix() @ f.u_matrix()).tocoo()
    num = math.sqrt(float(np.sum(d.data * d.data)))
    den = math.sqrt(float(np.sum(a.values * a.values)))
    if den == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return num / den


def solve(f: LUFactors, b) -> np.ndarray:
    """x = U^-1 L^-1 b[perm] (factorize.py:451-457).

    Factors returned by ``factorize`` are still resident on the device: the
    solve runs there (lbk_solve, blocked substitution on the factor blocks)
    while no later factorization has overwritten them.  Otherwise (factors
    built on the host, or stale) it is the reference's host solve."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (f.n,):
        raise DimensionMismatch(f"rhs must have length {f.n}")
    if f._device is not None:
        eng, gen = f._device
        if eng.ctx is not None and eng.generation == gen:
            return eng.solve(b)
    return solve_host(f, b)


def solve_host(f: LUFactors, b) -> np.ndarray:
    """The reference's host solve (scipy spsolve_triangular on the assembled CSR)."""
    b = np.asarray(b, dtype=np.float64)
    y = spsolve_triangular(f.l_matrix(), b[f.perm_global()], lower=True)
    return spsolve_triangular(f.u_matrix(), y, lower=False)


# --- kernel-level entry points (each one device launch over a tiny grid) ----------


class _MiniGrid:
    def __init__(self, n, positions, pool, value_max=1.0):
        self.n = n
        self.p = len(positions) - 1
        self.plan = BlockingPlan(n, np.asarray(positions, np.int64), "kernel")
        self.pool = pool
        self.value_max = value_max


class _MiniTree:
    def __init__(self, tasks):
        tasks = list(tasks)
        self.kinds = np.array([t[0] for t in tasks], np.int8)
        self.steps = np.array([t[1] for t in tasks], np.int32)
        self.rows = np.array([t[2] for t in tasks], np.int32)
        self.cols = np.array([t[3] for t in tasks], np.int32)
        self.levels_of = np.zeros(len(tasks), np.int32)
        self.costs = np.ones(len(tasks), np.int64)


def _full_pool(blocks):
    """Pool of full-rectangle blocks {(bi,bj): dense ndarray}, column-major block order."""
    keys = sorted(blocks, key=lambda k: (k[1], k[0]))
    t = np.zeros((7, len(keys)), np.int64)
    cps, ris, vals = [], [], []
    cpo = eo = 0
    for b, k in enumerate(keys):
        d = np.asarray(blocks[k], dtype=np.float64)
        nr, nc = d.shape
        t[:, b] = (k[0], k[1], nr, nc, nr * nc, cpo, eo)
        cps.append(np.arange(nc + 1, dtype=np.int64) * nr)
        ris.append(np.tile(np.arange(nr, dtype=np.int64), nc))
        vals.append(np.ascontiguousarray(d.T).ravel())
        cpo += nc + 1
        eo += nr * nc
    return keys, GridPool(table=t, col_ptr=np.concatenate(cps), row_idx=np.concatenate(ris),
                          values=np.concatenate(vals))


def _run_mini(blocks, positions, tasks, perms=None, pivot_tol=DEFAULT_PIVOT_TOL, static_eps=None):
    keys, pool = _full_pool(blocks)
    n = int(positions[-1])
    g = _MiniGrid(n, positions, pool)
    eng = Engine(g, _MiniTree(tasks), pool=pool, dense=True)
    try:
        eng.upload(pool.values)
        if perms is not None:
            eng.set_perms(perms)
        ms = C.c_float()
        st = _native.LbkStatus()
        eng.lib.lbk_factorize(eng.ctx, pivot_tol, math.nan if static_eps is None else static_eps,
                              C.byref(ms), C.byref(st))
        if st.code != 0:
            return None, None, st
        vals, pv = eng.download()
    finally:
        eng.close()
    out = {}
    for b, k in enumerate(keys):
        nr, nc, eo = int(pool.table[2, b]), int(pool.table[3, b]), int(pool.table[6, b])
        out[k] = vals[eo:eo + nr * nc].reshape(nc, nr).T.copy()
    return out, pv, None


def factor_diagonal(block, pivot_tol: float = DEFAULT_PIVOT_TOL, static_pivot_value: float | None = None,
                    block_index: int = 0):
    """perm . block = L U on the device (factorize.py:133-147)."""
    d = np.array(block, dtype=np.float64, copy=True)
    if d.ndim != 2 or d.shape[0] != d.shape[1]:
        raise DimensionMismatch("diagonal block must be square")
    m = d.shape[0]
    if m == 0:
        return np.zeros((0, 0)), np.zeros((0, 0)), np.arange(0)
    out, pv, st = _run_mini({(0, 0): d}, [0, m], [(GETRF, 0, 0, 0)], pivot_tol=pivot_tol,
                            static_eps=static_pivot_value)
    if st is not None:
        if st.code == _native.LBK_ERR_ZERO_PIVOT:
            raise ZeroPivot(block_index, int(st.col))
        _native.raise_status(st, "factor_diagonal")
    lu = out[(0, 0)]
    return np.tril(lu, -1) + np.eye(m), np.triu(lu), pv.astype(np.int64)


def factor_u_panel(l_ii, perm_i, b_ij):
    """L_ii^-1 applied to the row-permuted panel (factorize.py:150-156)."""
    x = np.array(b_ij, dtype=np.float64, copy=True)
    if not x.size:
        return x
    lsrc = np.asarray(l_ii, dtype=np.float64)
    m, nc = x.shape
    perms = np.concatenate([np.asarray(perm_i, dtype=np.int32), np.arange(nc, dtype=np.int32)])
    out, _, st = _run_mini({(0, 0): lsrc, (0, 1): x, (1, 1): np.eye(nc)}, [0, m, m + nc],
                           [(GESSM, 0, 0, 1)], perms=perms)
    if st is not None:
        _native.raise_status(st, "factor_u_panel")
    return out[(0, 1)]


def factor_l_panel(b_ji, u_ii):
    """Panel times U_ii^-1 (factorize.py:159-168)."""
    x = np.array(b_ji, dtype=np.float64, copy=True)
    u = np.asarray(u_ii, dtype=np.float64)
    if not x.size:
        return x
    diag = np.abs(np.diag(u))
    if np.any(diag == 0.0):
        raise ZeroPivot(0, int(np.argmin(diag)))
    m = u.shape[0]
    nr = x.shape[0]
    out, _, st = _run_mini({(0, 0): u, (1, 0): x, (1, 1): np.eye(nr)}, [0, m, m + nr], [(TSTRF, 0, 1, 0)])
    if st is not None:
        _native.raise_status(st, "factor_l_panel")
    return out[(1, 0)]


def schur_update(b_kj, l_ki, u_ij):
    """b_kj - l_ki @ u_ij (factorize.py:171-173)."""
    b = np.array(b_kj, dtype=np.float64, copy=True)
    lk = np.asarray(l_ki, dtype=np.float64)
    uj = np.asarray(u_ij, dtype=np.float64)
    mk, mi = lk.shape
    mj = uj.shape[1]
    if b.size == 0 or mi == 0:
        return b  # empty inner dimension: the product is exactly zero
    pos = [0, mi, mi + mk, mi + mk + mj]
    blocks = {(0, 0): np.eye(mi), (1, 1): np.eye(mk), (2, 2): np.eye(mj), (1, 0): lk, (0, 2): uj, (1, 2): b}
    out, _, st = _run_mini(blocks, pos, [(SSSSM, 0, 1, 2)])
    if st is not None:
        _native.raise_status(st, "schur_update")
    return out[(1, 2)]
