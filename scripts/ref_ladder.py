"""Time the unmodified reference (baseline/_ref) to completion on a ladder of same-family sizes.

    python scripts/ref_ladder.py C2 16 24 32 48 --out gpurun_out/ref_ladder.jsonl

One JSON line per size: reference factorize seconds (median of --repeats), GFLOP/s, host cores,
BLAS threads, predicted peak memory (SURVEY.md §8d guard) and MemAvailable.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref_timing as R  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("sizes", nargs="+", type=int)
ap.add_argument("--repeats", type=int, default=1)
ap.add_argument("--out", default=None)
args = ap.parse_args()
fam = R.FAMILIES[args.config][0]
for size in args.sizes:
    c = R.RefCase(fam, size)
    rec = {"config": args.config, "family": fam, "size": size, "n": c.n, "nnz_filled": c.nnz_filled,
           "p": c.grid.p, "tasks": len(c.tree.kinds), "gflop": c.flops / 1e9, "structure_s": c.structure_s,
           "predicted_peak_gb": c.predicted_peak_bytes() / 1e9, "mem_available_gb": R.mem_available() / 1e9,
           "cores": os.cpu_count(), "blas_threads": R.blas_threads(), "cpu": R.cpu_model()}
    if c.predicted_peak_bytes() > 0.8 * R.mem_available():
        rec["infeasible"] = True
    else:
        ts = [c.factorize_seconds() for _ in range(args.repeats)]
        rec.update({"seconds": statistics.median(ts), "runs": ts, "gflops": c.flops / statistics.median(ts) / 1e9})
    line = json.dumps(rec)
    print(line, flush=True)
    if args.out:
        with open(args.out, "a") as fh:
            fh.write(line + "\n")
