"""Per-task statistics of the executor's band sweeps (X_BAND) over one factorization:
segment length m, bandwidths, device duration, ns per column.

    python scripts/band_stats.py C5 [--plan regular:200]
"""
import argparse
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2512_04389_b200.numeric import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("--plan", default="irregular")
args = ap.parse_args()
strategy, bs = (args.plan, None) if ":" not in args.plan else ("regular", int(args.plan.split(":")[1]))
a, f, g, t = bench.build_case(args.cfg, strategy, bs)
eng = Engine(g, t)
eng.upload()
eng.run_device()
tr, info = eng.exec_trace()
tr = tr.astype(np.int64)
sel = (info[:, 0] == 10) & (tr[:, 2] > 0)
m = info[sel, 4]
bl, bu = info[sel, 2], info[sel, 3]
dur = (tr[sel, 2] - tr[sel, 1]) / 1e3
print(f"# {args.cfg} {args.plan}: {sel.sum()} band tasks, bl {np.unique(bl)}, bu {np.unique(bu)}")
print(f"m: min {m.min()} med {np.median(m):.0f} max {m.max()}; us: med {np.median(dur):.1f} max {dur.max():.1f}")
ns = dur * 1e3 / m
print(f"ns/column: med {np.median(ns):.1f} p10 {np.percentile(ns, 10):.1f} p90 {np.percentile(ns, 90):.1f}")
for q in np.argsort(-dur)[:5]:
    print(f"  m={m[q]} bl={bl[q]} bu={bu[q]} {dur[q]:.1f} us")
