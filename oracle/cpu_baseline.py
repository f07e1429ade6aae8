"""Bounded CPU baseline (TEST/BENCH INFRASTRUCTURE ONLY).

Runs the oracle's restatement of the reference's serial factorization
(factorize.py:245-384, workers=1; kernels in oracle.numeric) in construction
order over a bounded prefix of the task list, densifying blocks on first
touch exactly like the reference's scatter (factorize.py:265, inside its
timed region), until a wall-clock budget is spent.  Reports the algorithmic
flops of the completed tasks per second.  The full C2 run is infeasible on
a CPU host (>1,930 s and >62 GB), hence the bounded sample.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import numeric as ON


def sample(grid, tree, flops_t, budget_s: float = 15.0, max_tasks: int | None = None):
    """-> dict(value GFLOP/s, tasks, flops, seconds)."""
    state = {}

    def blk(key):
        d = state.get(key)
        if d is None:
            d = ON.dense(grid.blocks[key])
            state[key] = d
        return d

    perms = [None] * grid.p
    nt = len(tree.kinds) if max_tasks is None else min(max_tasks, len(tree.kinds))
    done = 0
    fl = 0.0
    t0 = time.perf_counter()
    for t in range(nt):
        kind, i, r, c = int(tree.kinds[t]), int(tree.steps[t]), int(tree.rows[t]), int(tree.cols[t])
        if kind == 3:
            if (r, c) in grid.blocks:
                blk((r, c))[...] -= blk((r, i)) @ blk((i, c))
        elif kind == 1:
            x = blk((i, c))
            if perms[i] is not None:
                x[:] = x[perms[i]]
            ON.gessm(blk((i, i)), x)
        elif kind == 2:
            ON.tstrf(blk((r, i)), blk((i, i)))
        else:
            perm, sw = ON.getrf(blk((i, i)))
            perms[i] = perm if sw else None
        done += 1
        fl += float(flops_t[t])
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": fl / dt / 1e9 if dt > 0 else 0.0, "tasks": done, "flops": fl, "seconds": dt,
            "total_tasks": len(tree.kinds)}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def blas_threads() -> int | None:
    try:
        from threadpoolctl import threadpool_info

        for info in threadpool_info():
            if info.get("user_api") == "blas":
                return int(info.get("num_threads"))
    except Exception:
        pass
    return None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


_ = np  # numpy is the arithmetic of the port
