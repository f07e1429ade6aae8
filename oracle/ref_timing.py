"""CPU timing of the UNMODIFIED reference (TEST/BENCH INFRASTRUCTURE ONLY).

Runs the reference package ``lublock`` itself — installed, not copied, by
``python -m pip install --no-index --no-build-isolation --no-deps --target
baseline/_ref /root/reference/pkg`` (``paper_2512_04389_b200.build``; the
directory is git-ignored and travels to the GPU box with the snapshot) —
through its own public API and stock code path, exactly like ``cmd_factor``
(``/root/reference/pkg/src/lublock/cli.py:194-215``):

    a = csc_from_triplets(...)                       matrix_io.py:99-139
    filled = symbolic_factorize(symmetrize_pattern(a))   symbolic.py:37-108
    curve = percentage_curve(diag_block_pointer(filled)) features.py:44-68
    plan = irregular_plan(curve, a.n)                blocking.py:49-114
    grid = partition(filled, a, plan); tree = dependency_levels(grid)
    t = perf_counter(); factorize(grid, tree, workers=1); perf_counter() - t

Only the input triplets come from this repository's generators (numpy only,
no native library is loaded: the reference has no Poisson / BBD / ND
generator).  The work count is the scalar sparse-LU flop count
Σ_k c_k(1 + 2 c_k) over the filled pattern (c_k = strictly-lower entries of
column k), which equals Σ_t F_t of SURVEY.md §8d exactly.

Memory / time guard: the full C2 run needs > 1,930 s and
> 62 GB on a CPU host, so the timed instance is the largest member of the
same family whose predicted peak memory fits 0.8 × MemAvailable and whose
predicted factorize time fits the caller's per-run budget.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(REPO, "baseline", "_ref")


def import_reference():
    """The installed reference package (raises ImportError when it is not installed)."""
    if not os.path.isdir(os.path.join(REF_DIR, "lublock")):
        raise ImportError(f"{REF_DIR}/lublock missing: run __graft_entry__.build() where /root/reference exists")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import lublock

    assert os.path.abspath(lublock.__file__).startswith(REF_DIR), lublock.__file__
    return lublock


def family_triplets(family: str, size: int, seed: int = 0):
    """(n, rows, cols, values) for a member of a BASELINE config family.

    family "poisson3d": 7-point Laplacian on size^3, geometric ND (C2 = 64, C4 = 96);
    family "bbd": bordered block diagonal, n = size, 1 % border, size/1000 bodies (C3 = 10^6);
    family "bbd2": n = size, 2 % border, 200 bodies (C5 = 2·10^5);
    family "poisson2d": 5-point, natural order (C1 = 64).
    """
    from paper_2512_04389_b200 import generators as G

    if family == "poisson3d":
        return G.poisson3d_triplets(size, "nd")
    if family == "poisson2d":
        return G.poisson2d_triplets(size)
    if family == "bbd":
        return (size,) + G.bbd_triplets(size, size // 100, max(size // 1000, 1), seed=seed)
    if family == "bbd2":
        return (size,) + G.bbd_triplets(size, size // 50, 200, seed=seed)
    raise ValueError(family)


# config -> (family, full size, ladder of same-family sizes, smallest first)
FAMILIES = {
    "C1": ("poisson2d", 64, (64,)),
    "C2": ("poisson3d", 64, (16, 20, 24, 28, 32, 40, 48, 64)),
    "C3": ("bbd", 1_000_000, (100_000, 200_000, 400_000, 1_000_000)),
    "C4": ("poisson3d", 96, (16, 20, 24, 28, 32, 40, 48, 64, 96)),
    "C5": ("bbd2", 200_000, (25_000, 50_000, 100_000, 200_000)),
}


def mem_available() -> float:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return float(line.split()[1]) * 1024.0
    except OSError:
        pass
    return float("inf")


def blas_threads() -> int | None:
    try:
        from threadpoolctl import threadpool_info

        for d in threadpool_info():
            if d.get("internal_api") in ("openblas", "mkl", "blis"):
                return int(d.get("num_threads"))
    except Exception:
        pass
    return None


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class RefCase:
    """One instance prepared through the reference's own structure path (untimed, like cmd_factor)."""

    def __init__(self, family: str, size: int, seed: int = 0):
        L = import_reference()
        t0 = time.perf_counter()
        n, r, c, v = family_triplets(family, size, seed)
        self.a = L.csc_from_triplets(n, (r, c, v))
        filled = L.symbolic_factorize(L.symmetrize_pattern(self.a))
        curve = L.percentage_curve(L.diag_block_pointer(filled))
        self.plan = L.irregular_plan(curve, self.a.n)
        self.grid = L.partition(filled, self.a, self.plan)
        self.tree = L.dependency_levels(self.grid)
        cp = np.asarray(filled.col_ptr, dtype=np.int64)
        ri = np.asarray(filled.row_idx, dtype=np.int64)
        col = np.repeat(np.arange(filled.n, dtype=np.int64), np.diff(cp))
        ck = np.bincount(col[ri > col], minlength=filled.n).astype(np.float64)
        self.flops = float(np.sum(ck * (1.0 + 2.0 * ck)))
        self.nnz_filled = int(len(ri))
        self.family, self.size, self.n = family, size, int(n)
        self.scratch_bytes = sum(8.0 * b.nrows * b.ncols for b in self.grid.blocks.values())
        self.structure_s = time.perf_counter() - t0
        self._L = L

    def predicted_peak_bytes(self) -> float:
        """SURVEY.md §8d memory guard: dense scratch + 3 copies of the (value, index) pattern."""
        return self.scratch_bytes + 3.0 * 12.0 * self.nnz_filled

    def factorize_seconds(self) -> float:
        """One stock ``lublock.factorize(grid, tree, workers=1)``, perf_counter around it (cli.py:203-215)."""
        t0 = time.perf_counter()
        self._L.factorize(self.grid, self.tree, workers=1)
        return time.perf_counter() - t0

    def describe(self) -> str:
        return (f"lublock.factorize(grid, tree, workers=1) to completion on {self.family} size {self.size} "
                f"(n={self.n}, nnz(L+U)={self.nnz_filled}, p={self.grid.p}, {len(self.tree.kinds)} tasks, "
                f"{self.flops / 1e9:.3f} GFLOP)")


def pick_case(config: str, run_budget_s: float, seed: int = 0, log=print):
    """Largest same-family instance whose predicted memory and single-run time fit.

    Walks the ladder smallest first, timing one factorization per rung; the next
    rung's time is predicted from the last measured time scaled by flops^0.7
    (measured here on poisson3d 16/20/24: time grows like flops^0.5, because
    per-task Python overhead dominates the small instances and BLAS the large
    ones; 0.7 errs on the long side).  Returns (case, first measured seconds on that case).
    """
    fam, full, ladder = FAMILIES[config]
    best = None
    for size in ladder:
        case = RefCase(fam, size, seed)
        if case.predicted_peak_bytes() > 0.8 * mem_available():
            log(f"[ref] {fam} {size}: needs {case.predicted_peak_bytes() / 1e9:.1f} GB, infeasible here")
            break
        if best is not None:
            pred = best[1] * (case.flops / best[0].flops) ** 0.7
            if pred > run_budget_s:
                log(f"[ref] {fam} {size}: predicted {pred:.1f}s per run > budget {run_budget_s:.1f}s")
                break
        s = case.factorize_seconds()
        log(f"[ref] {fam} {size}: {s:.2f}s, {case.flops / s / 1e9:.4f} GFLOP/s (structure {case.structure_s:.1f}s)")
        if s > run_budget_s and best is not None:
            break  # over budget: keep the previous rung
        best = (case, s)
        if s > run_budget_s:
            break
    if best is None:
        raise RuntimeError(f"no {fam} instance fits the memory guard on this host")
    return best
