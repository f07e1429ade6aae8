"""A small factorization + solve for compute-sanitizer runs (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python scripts/sanitize_case.py p3d10
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2512_04389_b200 as M  # noqa: E402
from paper_2512_04389_b200 import generators as G  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "p3d10"
a = {"p3d10": lambda: G.poisson3d(10, "nd"), "c1": lambda: G.poisson2d(64),
     "bbd": lambda: G.bbd(6000, 120, 12, seed=3), "dense": lambda: M.generate("dense", 300),
     "p3d12r": lambda: G.poisson3d(12, "nd")}[name]()
f = M.symbolic_factorize(M.symmetrize_pattern(a))
plan = (M.regular_plan(a.n, 150) if name == "dense"
        else M.regular_plan(a.n, 864) if name == "p3d12r"  # blocks of several subtrees: subtree-aligned tiles
        else M.irregular_plan(M.percentage_curve(M.diag_block_pointer(f)), a.n))
g = M.partition(f, a, plan)
t = M.dependency_levels(g)
lu = M.factorize(g, t)
b = a.to_scipy() @ np.ones(a.n)
x = M.solve(lu, b)
print(name, "relres", float(np.linalg.norm(a.to_scipy() @ x - b) / np.linalg.norm(b)))
