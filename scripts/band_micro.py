"""Band sweep in isolation: one full-band diagonal block (no independent
segments), the executor's X_BAND task timed by the in-kernel trace.

    python scripts/band_micro.py [--n 4000] [--bw 1,2,4,8,15]
"""
import argparse
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2512_04389_b200 as M  # noqa: E402
from paper_2512_04389_b200.numeric import Engine  # noqa: E402
from test_band_getrf import banded  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4000)
ap.add_argument("--bw", default="1,2,4,8,15")
args = ap.parse_args()
for bw in (int(v) for v in args.bw.split(",")):
    a = banded(args.n, bw, bw, np.random.default_rng(bw), keep=1.0)
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    g = M.partition(f, a, M.BlockingPlan(a.n, np.array([0, a.n], np.int64), "given"))
    t = M.dependency_levels(g)
    eng = Engine(g, t)
    eng.upload()
    eng.run_device()
    ms = sorted(eng.run_device() for _ in range(5))[2]
    tr, info = eng.exec_trace()
    tr = tr.astype(np.int64)
    sel = info[:, 0] == 10
    dur = (tr[sel, 2] - tr[sel, 1]).sum() / 1e3
    print(f"bw={bw:2d} n={args.n}: band tasks {sel.sum()}, sweep {dur:8.1f} us = {dur * 1e3 / args.n:6.1f} ns/column; "
          f"whole factorization {ms * 1e3:8.1f} us")
    eng.close()
