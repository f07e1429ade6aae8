"""Micro benchmark of the DMMA SSSSM kernel (gemm_map_kernel): one C -= L U task on FULL tiles."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2512_04389_b200.grid import SSSSM  # noqa: E402
from paper_2512_04389_b200.numeric import Engine, _full_pool, _MiniGrid, _MiniTree  # noqa: E402

for (m, n, k) in [(2048, 2048, 1024), (2048, 2048, 256), (1024, 1024, 512), (512, 512, 512)]:
    rng = np.random.default_rng(0)
    blocks = {(0, 0): np.eye(k), (1, 1): np.eye(m), (2, 2): np.eye(n), (1, 0): rng.standard_normal((m, k)),
              (0, 2): rng.standard_normal((k, n)), (1, 2): rng.standard_normal((m, n))}
    keys, pool = _full_pool(blocks)
    pos = [0, k, k + m, k + m + n]
    g = _MiniGrid(pos[-1], pos, pool)
    eng = Engine(g, _MiniTree([(SSSSM, 0, 1, 2)]), pool=pool, dense=True)
    eng.upload(pool.values)
    for _ in range(3):
        eng.run_device()
    lv = np.stack([eng.level_times()[:, 1] for _ in range(5)])
    ms = float(np.median(lv.sum(axis=1)))
    print(f"gemm_map {m}x{n}x{k}: {ms:.3f} ms  {2 * m * n * k / ms / 1e9:.2f} TF/s")
    eng.close()
