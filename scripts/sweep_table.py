"""Markdown summary of a balance_bench sweep (scripts/c5_sweep.sh output).

    python scripts/sweep_table.py profiles/r2_c5_sweep.jsonl > profiles/r2_c5_sweep.md
"""
import collections
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1])]
by = collections.defaultdict(dict)
for r in rows:
    by[r["matrix"]][r["plan"]] = r


def ms(r):
    return r["gpu_ms"] if r and r.get("status") == "ok" else float("nan")


print("| instance | irregular (step 2, max_num 3) ms | best irregular variant | PanguLU selector ms | "
      "best regular | irregular vs selector | irregular vs best regular | block-nnz CV irr / sel | tau sweep (ms) |")
print("|---|---|---|---|---|---|---|---|---|")
for m, d in by.items():
    irr = {k: v for k, v in d.items() if k.startswith("irregular") and "tau" not in k and v.get("status") == "ok"}
    reg = {k: v for k, v in d.items() if k.startswith("regular_") and v.get("status") == "ok"}
    taus = {k[len("irregular_tau_"):]: round(ms(v), 2) for k, v in d.items() if "tau" in k}
    bi = min(irr, key=lambda k: ms(irr[k]))
    br = min(reg, key=lambda k: ms(reg[k]))
    sel = d.get("pangulu_select")
    i0 = ms(d["irregular"])
    print(f"| {m} | {i0:.2f} | {bi} {ms(irr[bi]):.2f} | {ms(sel):.2f} | {br} {ms(reg[br]):.2f} | "
          f"{ms(sel) / i0:.2f}x | {ms(reg[br]) / i0:.2f}x | {d['irregular']['block_cv']:.2f} / "
          f"{sel['block_cv'] if sel else float('nan'):.2f} | {taus if taus else ''} |")
