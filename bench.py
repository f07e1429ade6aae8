"""Benchmark: numeric-factorization time & GFLOP/s on B200 vs the CPU reference.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One "step" = one numerical factorization (every level of the task DAG) of
the configuration's matrix with its values resident in HBM.  Default
workload: BASELINE.json configs[1] = C2, 3D 7-point Poisson 64^3 (n=262,144)
after geometric nested dissection, irregular blocking (p=174, 20,544 tasks,
268 levels), FP64.  Inputs (2.8 GB of factor values) exceed the 126 MB L2,
and every step starts by restoring A's values with a device copy, so no step
sees a warm L2 from the previous one.

Multi-GPU (--gpus N under torchrun, NCCL): ONE factorization of the same
matrix distributed 2D block-cyclically over the N GPUs (process grid 1x2 /
2x2 / 2x4, owner-computes, finished diagonal and panel blocks exchanged
between dependency levels with grouped NCCL point-to-point over NVLink;
paper_2512_04389_b200/parallel.py DistEngine) — strong scaling, timing =
max over ranks of the device time.  --replicas runs N independent copies
instead (weak scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

METRIC = "numeric-factorization time & GFLOP/s at 1/2/4/8 B200 vs CPU reference"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def build_case(name: str, strategy: str = "irregular", block_size: int | None = None):
    import paper_2512_04389_b200 as M
    from paper_2512_04389_b200.generators import CONFIGS, bbd

    t0 = time.perf_counter()
    if name in CONFIGS:
        a = CONFIGS[name]()
    elif name.startswith("poisson3d"):
        from paper_2512_04389_b200.generators import poisson3d

        a = poisson3d(int(name[9:]), "nd")
    elif name.startswith("bbd"):
        n = int(name[3:])
        a = bbd(n, n // 50, 200, seed=0)
    else:
        raise SystemExit(f"unknown config {name}")
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    curve = M.percentage_curve(M.diag_block_pointer(f))
    if strategy == "irregular":
        plan = M.irregular_plan(curve, a.n)
    elif strategy == "selector":  # PanguLU-like size selector (blocking.py:130-151)
        plan = M.regular_plan(a.n, M.pangulu_size_select(a.n, f.nnz_filled))
    else:
        plan = M.regular_plan(a.n, block_size)
    g = M.partition(f, a, plan)
    t = M.dependency_levels(g)
    log(f"[bench] {name}: n={a.n} nnz(A)={a.nnz} nnz(L+U)={f.nnz_filled} p={g.p} blocks={len(g.blocks)} "
        f"tasks={t.task_count} levels={t.n_levels} structure {time.perf_counter() - t0:.1f}s")
    return a, f, g, t


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def dist_init(backend=None):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        import datetime

        # a hung exchange aborts through the NCCL watchdog instead of hanging the job
        dist.init_process_group(backend, timeout=datetime.timedelta(minutes=10))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reference_cpu(config: str, run_budget_s: float, runs: int):
    """The unmodified reference (baseline/_ref) timed to completion on the host cores.

    oracle/ref_timing.py: ``lublock.factorize(grid, tree, workers=1)`` like cmd_factor
    (cli.py:194-215) on the largest same-family instance whose predicted memory and
    per-run time fit (SURVEY.md §8d guard).  ``runs`` further runs after the sizing run;
    returns (cpu_baseline dict, list of per-run seconds, case).
    """
    from oracle import ref_timing as R

    case, s0 = R.pick_case(config, run_budget_s, log=log)
    secs = [case.factorize_seconds() for _ in range(runs)] if runs > 0 else [s0]
    v = case.flops / statistics.median(secs) / 1e9
    fam, full, _ = R.FAMILIES[config]
    scope = ("the full configuration" if case.size == full else
             f"the largest {fam} instance whose predicted run time fits {run_budget_s:.0f}s and whose predicted "
             f"memory fits 0.8 x MemAvailable (full size {full} does not)")
    cpu = {"value": v, "unit": "GFLOP/s", "cores": os.cpu_count(), "blas_threads": R.blas_threads(),
           "cpu": R.cpu_model(), "kind": "reference",
           "sample": f"{case.describe()}; median of {len(secs)} runs ({statistics.median(secs):.2f}s); {scope}"}
    return cpu, secs, case


def spawn(n: int, backend: str | None) -> int:
    """``bench.py --gpus N`` without a launcher: re-exec under torch.distributed.run, N ranks."""
    import socket

    import torch

    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if have < n and backend != "gloo":
        raise SystemExit(f"bench.py --gpus {n}: only {have} CUDA device(s) visible; the 2D block-cyclic run "
                         f"needs one GPU per rank (use --dist-backend gloo to share one GPU in tests)")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    log(f"[bench] spawning {n} ranks: {' '.join(cmd[2:])}")
    return subprocess.call(cmd)


def plan_arg(s: str):
    """'irregular' | 'selector' | 'regular:<block size>'."""
    if s.startswith("regular:"):
        return "regular", int(s.split(":", 1)[1])
    if s not in ("irregular", "selector"):
        raise SystemExit(f"bad --plan {s}")
    return s, None


def run_reference(args):
    """--impl reference: the reference's own CPU factorization, rank 0 only (others exit 0)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    # each step is one full reference factorization; size the instance so that the whole
    # warmup + steps run ends within a few minutes
    budget = min(max(args.ref_budget_s / max(args.steps + args.warmup, 1), 2.0), 120.0)
    from oracle import ref_timing as R

    case, s0 = R.pick_case(args.config, budget, log=log)
    for _ in range(max(args.warmup - 1, 0)):  # the sizing run above was the first warm-up
        case.factorize_seconds()
    secs = [case.factorize_seconds() for _ in range(args.steps)]
    med = statistics.median(secs)
    v = case.flops / med / 1e9
    fam, full, _ = R.FAMILIES[args.config]
    scope = ("the full configuration" if case.size == full else
             f"largest same-family instance with predicted run <= {budget:.1f}s and memory <= 0.8 x MemAvailable; "
             f"full size {full} does not fit the bench budget (the full C2 reference run took 749 s on the GPU "
             f"box's 16 host cores, 1.12 GFLOP/s: profiles/r2_ref_full_c2.jsonl)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * med, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "plan": args.plan, "instance": f"{fam} {case.size}", "n": case.n,
                       "nnz_filled": case.nnz_filled, "gflop": case.flops / 1e9},
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": os.cpu_count(),
                             "blas_threads": R.blas_threads(), "cpu": R.cpu_model(), "kind": "reference",
                             "sample": f"{case.describe()}; each step one full run; {scope}"},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "runs_s": secs}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-s", type=float, default=30.0, help="per-run budget of the cpu_baseline leg")
    ap.add_argument("--ref-budget-s", type=float, default=400.0,
                    help="--impl reference: target seconds for all warmup + timed reference runs")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--levels-out", default=None, help="write per-level device times + work to this .npz")
    ap.add_argument("--dense-threshold", type=float, default=0.05,
                    help="compressed-tile density tag for the FP64 DMMA kernels; <0 = CSC kernels only")
    ap.add_argument("--plan", default="irregular", help="irregular | selector | regular:<block size>")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of 2D block-cyclic")
    ap.add_argument("--dist-backend", default=None, help="nccl (default with CUDA) | gloo (host-staged, 1-GPU tests)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args.gpus, args.dist_backend)

    world, rank, local = dist_init(args.dist_backend)
    import torch

    if torch.cuda.is_available():
        local = local % torch.cuda.device_count()  # several ranks may share a GPU in gloo tests
    import paper_2512_04389_b200 as M  # noqa: F401
    from paper_2512_04389_b200.numeric import Engine, pinned_empty
    from paper_2512_04389_b200.workmodel import task_work

    strategy, bs = plan_arg(args.plan)
    a, f, g, t = build_case(args.config, strategy, bs)
    flops_t, bytes_t = task_work(g, t)
    total_flops = float(flops_t.sum())
    t0 = time.perf_counter()
    dt = None if args.dense_threshold < 0 else args.dense_threshold
    distributed = world > 1 and not args.replicas
    if distributed:
        from paper_2512_04389_b200.parallel import DistEngine

        de = DistEngine(g, t, device=local, dense_threshold=dt)
        de.upload()
        _, st0 = de.run()  # one trial factorization: the exchange must work before we time it
        if st0.code:
            raise SystemExit(f"[bench] rank {rank}: distributed trial factorization failed: code {st0.code}")
    if distributed:
        eng = de.eng

        def run_dev():
            ms_, st_ = de.run()
            if st_.code:
                raise SystemExit(f"distributed factorization failed: {st_.code}")
            return ms_

        def run_host(vi, vo, pv):
            return de.run_host(vi, vo, pv)

        log(f"[bench] rank {rank}: grid {de.pg.pr}x{de.pg.pc}, {eng.n_segments} segments, {de.messages} messages, "
            f"{de.bytes_out / 1e9:.2f} GB sent per factorization")
    else:
        eng = Engine(g, t, device=local, dense_threshold=dt, dense_kernels=dt is not None)
        run_dev = eng.run_device
        run_host = eng.run_host
    eng.upload()
    log(f"[bench] plan: {eng.n_launch_levels} levels, {eng.n_launches} launches, {eng.n_items} CSC items, "
        f"{eng.n_gemm_tiles} DMMA tiles, {eng.n_dense_items} panel items, {eng.n_tile_items} tiled-GETRF items; "
        f"blocks sparse/rect/full {eng.n_sparse_blocks}/{eng.n_rect_blocks}/{eng.n_full_blocks}, "
        f"working entries {eng.nnz_work / 1e6:.1f}M vs {eng.nnz / 1e6:.1f}M; {time.perf_counter() - t0:.1f}s")

    for _ in range(max(args.warmup, 0)):
        run_dev()
    barrier(world)
    with ClockSampler(local) as clk:
        ms = [run_dev() for _ in range(args.steps)]
    barrier(world)
    t_step = max_over_ranks(sum(ms) / len(ms), world)
    jobs = 1 if distributed else world  # factorizations per step over the whole job
    value = jobs * total_flops / (t_step / 1e3) / 1e9

    # per-level / per-kernel-family device times (instrumented replay) -> roofline
    # (distributed: this rank's own tasks, replayed without the exchanges: timing only)
    lvl = eng.level_times(check=not distributed)  # [levels x 5]: level, DMMA SSSSM, panel, tiled GETRF, CSC
    routes = eng.task_routes()
    fam_names = {1: "gemm_map_kernel (DMMA SSSSM)", 2: "panel_kernel (DMMA GESSM/TSTRF)",
                 3: "tiled GETRF (tile_getrf/trsm/gemm)", 0: "level_kernel (CSC SSSSM/GESSM/TSTRF)"}
    fam_col = {1: 1, 2: 2, 3: 3, 0: 4}
    if float(lvl[:, 2].sum()) == 0.0 and (routes == 2).any():
        # persistent executor: panel solves run inside the same tile-DAG launch as GETRF
        fam_names[3] = "exec_kernel (tile-DAG: GETRF + GESSM/TSTRF panels)"
        del fam_col[2]
        routes = np.where(routes == 2, 3, routes)
    fams = {}
    for r, col in fam_col.items():
        sel = routes == r
        ms_f = float(lvl[:, col].sum())
        fams[r] = {"kernel": fam_names[r], "ms": ms_f, "tasks": int(sel.sum()),
                   "gflop": float(flops_t[sel].sum()) / 1e9, "gbytes": float(bytes_t[sel].sum()) / 1e9,
                   "launches": int((lvl[:, col] > 0).sum())}
    dom = max(fams, key=lambda r: fams[r]["ms"])
    hbm_peak, hbm_src = peaks()
    try:
        from paper_2512_04389_b200.numeric import fp64_peak

        dmma_peak, dfma_peak = fp64_peak(local)
    except Exception as exc:  # pragma: no cover
        log(f"[bench] fp64 peak probe failed: {exc}")
        dmma_peak, dfma_peak = float("nan"), float("nan")
    for r, fv in fams.items():
        s = max(fv["ms"], 1e-9) / 1e3
        fv["tflops"] = fv["gflop"] / s / 1e3
        fv["gbs"] = fv["gbytes"] / s
        fv["frac_fp64_tensor"] = fv["tflops"] / dmma_peak if dmma_peak == dmma_peak else None
        fv["frac_hbm"] = fv["gbs"] / hbm_peak
    # executed (tile-shaped, structural zeros included) flop rates: tensor-pipe utilisation
    for r, ex in ((1, eng.dmma_flops_executed), (3, eng.exec_flops_executed)):
        if r in fams and ex > 0:
            s = max(fams[r]["ms"], 1e-9) / 1e3
            fams[r]["executed_gflop"] = ex / 1e9
            fams[r]["executed_tflops"] = ex / s / 1e12
            fams[r]["executed_frac_fp64_tensor"] = ex / s / 1e12 / dmma_peak if dmma_peak == dmma_peak else None
    D = fams[dom]
    if dom in (1, 2, 3):
        roof = {"bound": "tensor", "achieved": D["tflops"], "peak": dmma_peak, "unit": "TFLOP/s",
                "frac": D["tflops"] / dmma_peak if dmma_peak == dmma_peak else None,
                "peak_source": "FP64 DMMA.8x8x4 register loop measured on this GPU by csrc/lbk_peak.cu "
                               "(MEASURED_PEAKS.json has no FP64 entry)"}
    else:
        roof = {"bound": "hbm", "achieved": D["gbs"], "peak": hbm_peak, "unit": "GB/s",
                "frac": D["gbs"] / hbm_peak, "peak_source": hbm_src}
    traffic = None
    tp = os.path.join(REPO, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tp):
        tr = json.load(open(tp)).get("dram_bytes_per_launch")
        # per kernel (ncu dram__bytes_read.sum + dram__bytes_write.sum, averaged over launches)
        traffic = tr.get(D["kernel"].split(" ")[0]) if isinstance(tr, dict) else tr
    roof.update({"traffic": traffic, "kernel": D["kernel"], "launches_per_step": D["launches"],
                 "algorithmic": "flops = 2*tree.costs (SSSSM), GETRF/panel formulas of SURVEY 8d; "
                                "bytes = 8 B/value + 4 B/index per touched block",
                 "by_kernel": {fams[r]["kernel"]: {k: v for k, v in fams[r].items() if k != "kernel"}
                               for r in fams},
                 "fp64_peaks_tflops": {"dmma": dmma_peak, "dfma": dfma_peak},
                 "hbm_peak_gbs": hbm_peak})
    if args.levels_out:
        np.savez(args.levels_out, level_ms=lvl, routes=routes, flops=flops_t, bytes=bytes_t,
                 kinds=t.kinds, levels_of=t.levels_of, costs=t.costs)


    # end to end through the public API a reference user calls, host buffers, every
    # host<->device copy inside the timed region.  Single GPU: the drop-in
    # factorize(grid, tree) -> LUFactors (A's nnz values in from the grid, all factor
    # values out, streamed per finished block into page-locked memory the returned
    # blocks view); distributed: DistEngine.run_host per rank (pooled values in).
    ke = args.e2e_steps or max(1, min(args.steps, 3))
    solve_info = None
    e2e_cabi = None
    if distributed:
        vin = pinned_empty(eng.nnz)
        vin[:] = eng.pool.values
        vout = pinned_empty(eng.nnz)
        perms = np.empty(max(eng.n_diag_rows, 1), np.int32)
        run_host(vin, vout, perms)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(ke):
            st = run_host(vin, vout, perms)
            if st.code:
                raise SystemExit(f"e2e factorization failed: {st.code}")
        e2e_s = max_over_ranks((time.perf_counter() - t0) / ke, world)
        h2d_bytes, d2h_bytes = 8 * eng.nnz, 8 * eng.nnz + 4 * eng.n_diag_rows
        e2e_path = "DistEngine.run_host -> lbk_factorize_host per rank (pooled grid values in), pinned host buffers"
    else:
        # the C-ABI refactorization entry (KLU-style: A's values in, pool-order factors out)
        from paper_2512_04389_b200.grid import pool_positions

        eng.bind_matrix(pool_positions(f, a, g.plan))
        a_in = pinned_empty(a.nnz)
        a_in[:] = a.values
        vout = pinned_empty(eng.nnz)
        perms = np.empty(max(eng.n_diag_rows, 1), np.int32)
        eng.refactor_host(a_in, vout, perms)
        t0 = time.perf_counter()
        for _ in range(ke):
            eng.refactor_host(a_in, vout, perms)
        cabi_s = (time.perf_counter() - t0) / ke
        e2e_cabi = {"value": total_flops / cabi_s / 1e9, "unit": "GFLOP/s", "seconds_per_step": cabi_s,
                    "path": "Engine.refactor_host -> lbk_refactor_host (C-ABI): A's values (pinned) in, factor "
                            "values in reference pool order (pinned, streamed) + perms out"}
        eng.close()  # one device plan at a time (C4 needs most of the HBM)
        import gc

        gc.collect()
        lu = M.factorize(g, t, dense_threshold=dt)  # plans, captures, first run (untimed)
        lu = M.factorize(g, t, dense_threshold=dt)
        t0 = time.perf_counter()
        for _ in range(ke):
            lu = M.factorize(g, t, dense_threshold=dt)
        e2e_s = (time.perf_counter() - t0) / ke
        deng = lu._device[0]
        h2d_bytes, d2h_bytes = 8 * a.nnz, 8 * deng.nout + 4 * deng.n_diag_rows
        e2e_path = ("paper_2512_04389_b200.factorize(grid, tree) -> LUFactors (drop-in for lublock.factorize): "
                    "A's values from the grid in (pinned staging), all L/U block values out (page-locked, streamed "
                    "per finished block, blocks are views), perms out")
        # device triangular solve on the resident factors (factorize.py:451-457 on the device)
        A = a.to_scipy()
        rhs = A @ np.ones(a.n)
        M.solve(lu, rhs)  # builds the solve graph
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            x = M.solve(lu, rhs)
            ts.append(time.perf_counter() - t0)
        solve_info = {"ms": 1e3 * statistics.median(ts),
                      "relres": float(np.linalg.norm(A @ x - rhs) / np.linalg.norm(rhs)),
                      "path": "solve(LUFactors, b) -> lbk_solve on the resident factors (host b in, host x out), "
                              "b = A @ ones"}
    e2e_value = jobs * total_flops / e2e_s / 1e9

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, _, _ = reference_cpu(args.config, args.cpu_sample_s, 0)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True,
            "scaling": "strong" if distributed else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "matrix": "3D 7-point Poisson 64^3, geometric ND" if args.config == "C2"
                       else args.config, "plan": args.plan, "n": a.n, "nnz_A": a.nnz, "nnz_filled": f.nnz_filled,
                       "p": g.p, "tasks": t.task_count, "levels": t.n_levels, "gflop": total_flops / 1e9,
                       "parallelism": (f"2d-block-cyclic {de.pg.pr}x{de.pg.pc} (NCCL p2p)" if distributed
                                       else f"replicas{world}" if world > 1 else "single"),
                       "l2": "inputs (factor values, %.2f GB) larger than L2; values restored by a device copy "
                             "before every step" % (8 * eng.nnz / 1e9)},
            "e2e": {"value": e2e_value, "unit": "GFLOP/s", "seconds_per_step": e2e_s,
                    "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
                    "path": e2e_path, "c_abi": e2e_cabi},
            "roofline": roof,
            "plan": {"dense_threshold": dt, "launches_per_step": int(eng.n_launches),
                     "blocks_sparse_rect_full": [eng.n_sparse_blocks, eng.n_rect_blocks, eng.n_full_blocks],
                     "working_entries": eng.nnz_work, "reference_entries": eng.nnz,
                     "level_ms_sum": float(lvl[:, 0].sum())},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": int(args.steps * eng.n_launches),
            "solve": solve_info,
            "exchange": ({"segments": eng.n_segments, "messages_rank0": de.messages,
                          "bytes_sent_rank0": de.bytes_out,
                          "roofline_scope": "rank 0's own tasks"} if distributed else None),
        }
        print(json.dumps(line), flush=True)
    if distributed:
        eng.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
