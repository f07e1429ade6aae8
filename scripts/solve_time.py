import sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2512_04389_b200.numeric import Engine
a, f, g, t = bench.build_case(sys.argv[1] if len(sys.argv) > 1 else "C2")
eng = Engine(g, t); eng.upload(); eng.run_device()
rhs = a.to_scipy() @ np.ones(a.n)
eng.solve(rhs)
ts = []
for _ in range(3):
    t0 = time.perf_counter(); eng.solve(rhs); ts.append(time.perf_counter() - t0)
print("solve ms", 1e3 * np.median(ts))
