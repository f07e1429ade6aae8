"""One device solve of a config for an ncu launch list (plan, factorize, warm-up solve, profiled solve)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2512_04389_b200 as M  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
a, f, g, t = bench.build_case(cfg)
lu = M.factorize(g, t)
b = a.to_scipy() @ np.ones(a.n)
M.solve(lu, b)
import ctypes  # noqa: E402

ctypes.CDLL("libcudart.so").cudaProfilerStart() if False else None
x = M.solve(lu, b)
print("relres", float(np.linalg.norm(a.to_scipy() @ x - b) / np.linalg.norm(b)))
