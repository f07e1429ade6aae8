"""One factorization of a config for ncu: plan + upload + 1 warm-up + 1 profiled replay."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2512_04389_b200.numeric import Engine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
a, f, g, t = bench.build_case(cfg)
eng = Engine(g, t, dense_threshold=tau)
eng.upload()
eng.run_device()  # warm-up (graph build)
print("ms", eng.run_device(), "launches", eng.n_launches, flush=True)
