"""Where a factorization's device time goes, level by level (one instrumented replay).

    python scripts/level_profile.py C5 [--plan regular:200] [--top 15]

Prints the levels with the largest device time, their per-family split
(DMMA SSSSM / panel / executor / CSC) and the executor task mix, plus totals.
"""
import argparse
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2512_04389_b200.numeric import Engine  # noqa: E402

NAMES = ["COLMAX", "GETRF", "TRSM_L", "TRSM_U", "GEMM", "FINAL", "PG_DIAG", "PG_UPD", "PT_DIAG", "PT_UPD",
         "BAND", "GETRF_UPD", "PG_FUSED", "PT_FUSED", "NOP", "SSSSM"]

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("--plan", default="irregular")
ap.add_argument("--top", type=int, default=15)
ap.add_argument("--range", default=None, help="also list levels lo:hi in order")
args = ap.parse_args()
strategy, bs = (args.plan, None) if ":" not in args.plan else ("regular", int(args.plan.split(":")[1]))
a, f, g, t = bench.build_case(args.cfg, strategy, bs)
eng = Engine(g, t)
eng.upload()
eng.run_device()
ms = sorted(eng.run_device() for _ in range(3))[1]
lt = eng.level_times()
tr, info = eng.exec_trace()
tr = tr.astype(np.int64)
print(f"# {args.cfg} {args.plan}: graph {ms:.2f} ms; instrumented level sum {lt[:, 0].sum():.2f} ms "
      f"(dmma {lt[:, 1].sum():.2f} panel {lt[:, 2].sum():.2f} exec {lt[:, 3].sum():.2f} csc {lt[:, 4].sum():.2f})")
order = list(np.argsort(-lt[:, 0])[: args.top])
if args.range:
    lo, hi = (int(v) for v in args.range.split(":"))
    order += list(range(lo, min(hi, len(lt))))
for L in order:
    sel = info[:, 5] == L
    mix = {}
    for ty, cnt in zip(*np.unique(info[sel, 0], return_counts=True)):
        mix[NAMES[ty]] = int(cnt)
    run = ((tr[sel, 2] - tr[sel, 1]) / 1e3) if sel.any() else np.zeros(1)
    print(f"L{L:4d} {lt[L, 0]:7.3f} ms  dmma {lt[L, 1]:6.3f} panel {lt[L, 2]:6.3f} exec {lt[L, 3]:6.3f} "
          f"csc {lt[L, 4]:6.3f}  exec-task-us sum {run.sum():9.1f} max {run.max():7.1f}  {mix}")
# totals by task type
ok = tr[:, 2] > 0
for ty in np.unique(info[:, 0]):
    s = (info[:, 0] == ty) & ok
    run = (tr[s, 2] - tr[s, 1]) / 1e3
    print(f"{NAMES[ty]:9s} n={s.sum():7d} run us med {np.median(run):7.2f} max {run.max():8.1f} sum {run.sum() / 1e3:8.2f} ms")
