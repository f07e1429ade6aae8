"""Irregular-vs-regular blocking on the GPU (the reference's `lublock bench`,
pkg/src/lublock/cli.py:245-339, with the numeric phase on the B200).

    python scripts/balance_bench.py C5 [C3 ...] [--sizes 500,1000,2000,5000] [--repeats 3] [--out f.csv]

Per (matrix, plan) row: p, blocks, tasks, levels, the reference's balance
metrics (block_nnz_stats CV, level_work_stats last-level share, 4-worker
makespan model, pkg/src/lublock/metrics.py:45-138), and the measured device
numeric-factorization time (median), GFLOP/s, the summed per-level device
time and its split over the kernel families (DMMA SSSSM, tile-DAG
executor, CSC kernel).  Rows "pangulu_select" and "best_regular" repeat the
matching regular rows like cmd_bench.  --taus adds irregular-plan rows for
other density tags (sparse-kernel vs DMMA selection; "off" = CSC only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2512_04389_b200 as M  # noqa: E402
from paper_2512_04389_b200.blocking import PANGULU_SIZES  # noqa: E402
from paper_2512_04389_b200.generators import CONFIGS, bbd  # noqa: E402
from paper_2512_04389_b200.metrics import block_nnz_stats, level_work_stats, makespan_model  # noqa: E402
from paper_2512_04389_b200.numeric import Engine  # noqa: E402
from paper_2512_04389_b200.workmodel import task_work  # noqa: E402


def matrix(name):
    if name in CONFIGS:
        return CONFIGS[name]()
    if name.startswith("bbd"):  # bbd<n>[_b<border%>][_k<blocks>][_s<seed>]
        parts = name[3:].split("_")
        n = int(parts[0])
        opts = {p[0]: p[1:] for p in parts[1:]}
        border = int(n * float(opts.get("b", "2")) / 100)
        return bbd(n, border, int(opts.get("k", "200")), seed=int(opts.get("s", "0")))
    raise SystemExit(f"unknown matrix {name}")


def run_plan(a, f, plan, repeats, tau, check):
    g = M.partition(f, a, plan)
    t = M.dependency_levels(g)
    flops_t, _ = task_work(g, t)
    eng = Engine(g, t, dense_threshold=tau)
    eng.upload()
    eng.run_device()
    ms = [eng.run_device() for _ in range(repeats)]
    lvl = eng.level_times()
    lw = level_work_stats(t)
    bs = block_nnz_stats(g)
    med = statistics.median(ms)
    row = {"p": g.p, "blocks": len(g.blocks), "tasks": t.task_count, "levels": t.n_levels,
           "block_cv": bs.cv, "block_cv_all_cells": bs.cv_all_cells, "last_level_share": lw.last_level_share,
           "makespan4_model": makespan_model(t, 4), "gflop": float(flops_t.sum()) / 1e9, "gpu_ms": med,
           "gpu_gflops": float(flops_t.sum()) / (med / 1e3) / 1e9, "level_ms_sum": float(lvl[:, 0].sum()),
           "dmma_ms": float(lvl[:, 1].sum()), "exec_ms": float(lvl[:, 3].sum()), "csc_ms": float(lvl[:, 4].sum()),
           "launch_levels": int(eng.n_launch_levels), "working_entries": int(eng.nnz_work)}
    if check:
        lu = M.factorize(g, t, dense_threshold=tau)
        b = a.to_scipy() @ np.ones(a.n)
        x = M.solve(lu, b)
        row["relres"] = float(np.linalg.norm(a.to_scipy() @ x - b) / np.linalg.norm(b))
    eng.close()
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("matrices", nargs="+")
    ap.add_argument("--sizes", default=None, help="regular block sizes (default: PANGULU_SIZES <= n)")
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--tau", type=float, default=0.05)
    ap.add_argument("--check", action="store_true", help="also solve and report ||Ax-b||/||b||")
    ap.add_argument("--out", default=None, help="JSON lines output")
    ap.add_argument("--grid", default=None,
                    help="irregular-plan variants 'steps:max_nums', e.g. 1,2,4:1,3,7 (blocking.py:49-114 knobs)")
    ap.add_argument("--taus", default=None,
                    help="also sweep the density tag on the irregular plan, e.g. 0.05,0.1,0.25,0.5,off")
    args = ap.parse_args()
    out = open(args.out, "w") if args.out else None
    for name in args.matrices:
        t0 = time.perf_counter()
        a = matrix(name)
        f = M.symbolic_factorize(M.symmetrize_pattern(a))
        curve = M.percentage_curve(M.diag_block_pointer(f))
        print(f"# {name}: n={a.n} nnz(A)={a.nnz} nnz(L+U)={f.nnz_filled} ({time.perf_counter() - t0:.1f}s)",
              flush=True)
        sizes = [int(x) for x in args.sizes.split(",")] if args.sizes else [b for b in PANGULU_SIZES if b <= a.n]
        plans = [("irregular", M.irregular_plan(curve, a.n))] + [(f"regular_{b}", M.regular_plan(a.n, b))
                                                                 for b in sizes]
        if args.grid:
            st_s, mx_s = args.grid.split(":")
            for stp in (int(x) for x in st_s.split(",")):
                for mx in (int(x) for x in mx_s.split(",")):
                    if (stp, mx) != (2, 3):  # the defaults are the "irregular" row
                        plans.append((f"irregular_s{stp}_m{mx}", M.irregular_plan(curve, a.n, stp, mx)))
        sel = min(M.pangulu_size_select(a.n, f.nnz_filled), a.n)
        if f"regular_{sel}" not in [p[0] for p in plans]:
            plans.append((f"regular_{sel}", M.regular_plan(a.n, sel)))
        rows = {}
        for label, plan in plans:
            try:
                r = run_plan(a, f, plan, args.repeats, args.tau, args.check)
                r["status"] = "ok"
            except Exception as exc:  # a plan can exceed device limits (span > smem accumulator)
                r = {"status": f"error:{type(exc).__name__}: {exc}"[:200]}
            r.update({"matrix": name, "plan": label})
            rows[label] = r
            line = json.dumps(r)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
        if args.taus:
            irr = M.irregular_plan(curve, a.n)
            for tv in args.taus.split(","):
                tau = None if tv == "off" else float(tv)
                try:
                    r = run_plan(a, f, irr, args.repeats, tau, False)
                    r["status"] = "ok"
                except Exception as exc:
                    r = {"status": f"error:{type(exc).__name__}: {exc}"[:200]}
                r.update({"matrix": name, "plan": f"irregular_tau_{tv}"})
                line = json.dumps(r)
                print(line, flush=True)
                if out:
                    out.write(line + "\n")
        regs = {k: v for k, v in rows.items() if k.startswith("regular_") and v["status"] == "ok"}
        extra = []
        if f"regular_{sel}" in regs:
            extra.append(dict(regs[f"regular_{sel}"], plan="pangulu_select"))
        if regs:
            extra.append(dict(min(regs.values(), key=lambda r: r["gpu_ms"]), plan="best_regular"))
        for r in extra:
            line = json.dumps(r)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
        if "irregular" in rows and regs and rows["irregular"]["status"] == "ok":
            best = min(regs.values(), key=lambda r: r["gpu_ms"])
            print(f"# {name}: irregular {rows['irregular']['gpu_ms']:.2f} ms vs best regular "
                  f"{best['plan']} {best['gpu_ms']:.2f} ms -> speedup {best['gpu_ms'] / rows['irregular']['gpu_ms']:.2f}x",
                  flush=True)
    if out:
        out.close()


if __name__ == "__main__":
    main()
