"""Per launch level: DMMA SSSSM device ms and tile counts (is the SSSSM launch tail- or throughput-bound?).

    python scripts/dmma_levels.py C2 gpurun_out/c2_dmma_levels.npz
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2512_04389_b200.numeric import Engine  # noqa: E402

a, f, g, t = bench.build_case(sys.argv[1], "irregular", None)
eng = Engine(g, t)
eng.upload()
eng.run_device()
ms = sorted(eng.run_device() for _ in range(3))[1]
lt = eng.level_times()
lv, _ = eng.plan_levels()
np.savez(sys.argv[2], lt=lt, lv=lv, ms=ms)
ng = lv[2]
order = np.argsort(-lt[:, 1])
print(f"graph {ms:.2f} ms; dmma sum {lt[:, 1].sum():.2f} ms over {(lt[:, 1] > 0).sum()} levels")
for L in order[:40]:
    print(f"L{L:4d} dmma {lt[L, 1]:7.3f} ms tiles {ng[L]:6d}  us/tile-wave {lt[L, 1] * 1e3 / max(1, np.ceil(ng[L] / 296)):7.1f}")
