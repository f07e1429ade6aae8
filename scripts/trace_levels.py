"""Executor task statistics per task type over a whole factorization (one instrumented replay)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2512_04389_b200.numeric import Engine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
a, f, g, t = bench.build_case(cfg)
eng = Engine(g, t)
eng.upload()
eng.run_device()
tr, info = eng.exec_trace()
tr = tr.astype(np.int64)
names = ["COLMAX", "GETRF", "TRSM_L", "TRSM_U", "GEMM", "FINAL", "PG_DIAG", "PG_UPD", "PT_DIAG", "PT_UPD", "BAND", "GETRF_UPD", "PG_FUSED", "PT_FUSED"]
ok = tr[:, 2] > 0
for ty in np.unique(info[:, 0]):
    sel = (info[:, 0] == ty) & ok
    run = (tr[sel, 2] - tr[sel, 1]) / 1e3
    wait = (tr[sel, 1] - tr[sel, 0]) / 1e3
    print(f"{names[ty]:8s} n={sel.sum():7d} run us med {np.median(run):7.2f} p90 {np.percentile(run, 90):7.2f} "
          f"sum {run.sum() / 1e3:8.1f} ms  wait med {np.median(wait):7.2f}")
# per launch level: span (first ready -> last done) and the chain of the slowest panel column
lv = info[:, 5]
for L in np.unique(lv)[:0]:
    pass
np.savez(f"gpurun_out/trace_{cfg}.npz", trace=tr, info=info)
