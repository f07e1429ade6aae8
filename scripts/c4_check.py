"""C4 (3D Poisson 96^3 + ND, 9.9 TFLOP) on the device vs the oracle, value by value.

The reference cannot run C4 in either container (its dense scratch alone is ~400 GB,
SURVEY.md 8d), so C4 is checked like the C2 full-size test (tests/test_full_configs.py):
every value of every block final after the oracle's prefix of steps 0..s (oracle.numeric.
factorize_prefix, pinned to the reference on the small / named / C5 cases) against the
device factors at 1e-10 of the block scale, plus the solve residual.  Too large for the
GPU test suite (140 GB of HBM, ~14 GB of exported factors); run once under gpurun:

    python scripts/c4_check.py [budget_s] > gpurun_out/r2_c4_check.txt
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2512_04389_b200 as M  # noqa: E402
from oracle import numeric as ON  # noqa: E402
from oracle import structure as OS  # noqa: E402
from paper_2512_04389_b200 import generators as G  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 90.0
t0 = time.perf_counter()
a = G.CONFIGS["C4"]()
f = M.symbolic_factorize(M.symmetrize_pattern(a))
pl = M.irregular_plan(M.percentage_curve(M.diag_block_pointer(f)), a.n)
g = M.partition(f, a, pl)
t = M.dependency_levels(g)
print(f"C4: n={a.n} nnz(L+U)={f.nnz_filled} p={g.p} tasks={t.task_count} structure {time.perf_counter() - t0:.1f}s",
      flush=True)
t1 = time.perf_counter()
lu = M.factorize(g, t)
print(f"factorize (drop-in, first call incl. plan) {time.perf_counter() - t1:.1f}s", flush=True)
og = OS.Grid(a.n, g.p, g.plan.positions, g.blocks, g.block_nnz, g.value_max)
t2 = time.perf_counter()
s, final = ON.factorize_prefix(og, t, budget_s=budget)
lb, ub = ON.export(final)
amax = float(np.abs(a.values).max())
compared, worst = 0, 0.0
for blocks, ob in ((lu.l_blocks, lb), (lu.u_blocks, ub)):
    for k, want in ob.items():
        got = blocks[k]
        assert np.array_equal(got.col_ptr, want.col_ptr) and np.array_equal(got.row_idx, want.row_idx), k
        scale = max(float(np.abs(want.values).max(initial=0.0)), 1e-3 * amax)
        err = float(np.abs(got.values - want.values).max(initial=0.0))
        assert err <= 1e-10 * scale, (k, err, scale)
        worst = max(worst, err / scale)
        compared += len(want.values)
total = sum(b.nnz for b in lu.l_blocks.values()) + sum(b.nnz for b in lu.u_blocks.values())
print(f"oracle prefix steps 0..{s} of {g.p} ({time.perf_counter() - t2:.1f}s): {compared}/{total} factor values "
      f"compared, worst rel {worst:.2e}", flush=True)
A = a.to_scipy()
b = A @ np.ones(a.n)
x = M.solve(lu, b)
print(f"solve relres {float(np.linalg.norm(A @ x - b) / np.linalg.norm(b)):.3e}")
