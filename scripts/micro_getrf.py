"""Micro benchmark: one dense diagonal block (single-block plan) -> tiled GETRF only."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2512_04389_b200 as M  # noqa: E402
from paper_2512_04389_b200.numeric import Engine  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
nb = int(sys.argv[2]) if len(sys.argv) > 2 else m
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
a = M.generate("dense", m)
f = M.symbolic_factorize(M.symmetrize_pattern(a))
g = M.partition(f, a, M.regular_plan(m, nb))
t = M.dependency_levels(g)
eng = Engine(g, t)
eng.upload()
for _ in range(2):
    eng.run_device()
ms = [eng.run_device() for _ in range(reps)]
lv = eng.level_times()
print(f"m={m} bs={nb} p={g.p} tasks={t.task_count} exec_items={eng.n_tile_items} launches={eng.n_launches} "
      f"ms/step={np.median(ms):.3f} levels_ms={lv[:, 0].sum():.3f} exec_ms={lv[:, 3].sum():.3f} "
      f"gemm_ms={lv[:, 1].sum():.3f} csc_ms={lv[:, 4].sum():.3f} GF/s={2 / 3 * m ** 3 / np.median(ms) / 1e6:.1f}")

if "--trace" in sys.argv:
    tr, info = eng.exec_trace()
    tr = tr.astype(np.int64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    names = ["COLMAX", "GETRF", "TRSM_L", "TRSM_U", "GEMM", "FINAL", "PG_DIAG", "PG_UPD", "PT_DIAG", "PT_UPD", "BAND", "GETRF_UPD", "PG_FUSED", "PT_FUSED"]
    for ty in np.unique(info[:, 0]):
        sel = info[:, 0] == ty
        run = (tr[sel, 2] - tr[sel, 1]) / 1e3
        wait = (tr[sel, 1] - tr[sel, 0]) / 1e3
        ph = tr[sel][:, [1, 3, 4, 5, 6, 7, 2]].astype(np.float64)
        d = np.diff(ph, axis=1) / 1e3
        d[(ph[:, 1:] == 0) | (ph[:, :-1] == 0)] = np.nan
        print(f"{names[ty]:8s} n={sel.sum():6d} run us med {np.median(run):7.2f} p90 {np.percentile(run, 90):7.2f}"
              f" wait med {np.median(wait):8.2f} phases(ready>p0>p1>p2>p3>fence>done) "
              + " ".join("-" if np.all(np.isnan(d[:, k])) else f"{np.nanmedian(d[:, k]):.2f}" for k in range(6)))
    g = np.flatnonzero((info[:, 0] == 1) | (info[:, 0] == 11))
    for t in g[:6]:
        print(f"GETRF k={info[t, 4]} dequeue {(tr[t, 0] - t0) / 1e3:9.1f} ready {(tr[t, 1] - t0) / 1e3:9.1f}"
              f" done {(tr[t, 2] - t0) / 1e3:9.1f} us")
    np.savez("gpurun_out/exec_trace.npz", trace=tr, info=info)
