"""Generate golden fixtures by running the REFERENCE itself (lublock 0.1.0).

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--c2]

Outputs (committed, small):
  tests/golden/spec.json            SPEC known answers recomputed by the reference
  tests/golden/small_<name>.npz      full inputs + every reference output for n <= 64
  tests/golden/cases.json            per-config structure hashes + factor checksums
  tests/golden/case_<name>.npz       plan positions, per-block factor samples

Inputs of the named cases come from paper_2512_04389_b200.generators /
matrix_io.generate (deterministic); the reference consumes them through its
own csc_from_triplets, exactly as SURVEY.md §8d prescribes.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import lublock as R  # noqa: E402  (the reference)
import oracles as RO  # noqa: E402  (the reference's own test oracles)

from paper_2512_04389_b200 import generators as G  # noqa: E402  (inputs only)


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.kind in "iu":
        a = a.astype(np.int64)
    return hashlib.sha256(a.tobytes()).hexdigest()


def ref_csc(a):
    return R.CscMatrix(a.n, np.asarray(a.col_ptr), np.asarray(a.row_idx), np.asarray(a.values))


def spec_examples():
    out = {}
    # Alg. 2 examples
    def bp(pattern, n):
        rr, cc = zip(*sorted(pattern))
        a = R.csc_from_triplets(n, (np.array(rr), np.array(cc), np.ones(len(rr))))
        return R.diag_block_pointer(R.symbolic_factorize(R.symmetrize_pattern(a))).blockptr.tolist()
    out["blockptr_identity4"] = bp({(i, i) for i in range(4)}, 4)
    out["blockptr_dense3"] = bp({(i, j) for i in range(3) for j in range(3)}, 3)
    out["blockptr_tridiag4"] = bp({(i, j) for i in range(4) for j in range(4) if abs(i - j) <= 1}, 4)
    # Alg. 3 examples, both window variants
    curves = {
        "ex1": [0, .01, .02, .03, .04, .05, .06, .07, .08, .09, 1.0],
        "ex2": [0, .15, .30, .45, .60, .75, .80, .85, .90, .95, 1.0],
        "ex3": [k * k / 100 for k in range(11)],
    }
    for name, pct in curves.items():
        c = R.PercentCurve(n=1000, sample_points=10, pct=np.array(pct, dtype=np.float64))
        out[f"plan_{name}"] = R.irregular_plan(c, 1000, 2, 3, 0.2).positions.tolist()
        out[f"plan_{name}_overlap"] = R.irregular_plan(c, 1000, 2, 3, 0.2, True).positions.tolist()
        out[f"curve_{name}"] = pct
    out["regular"] = {f"{n}_{bs}": R.regular_plan(n, bs).positions.tolist()
                      for n, bs in ((10, 3), (10, 10), (10, 1), (1000, 300))}
    out["select"] = {f"{n}_{nnz}": R.pangulu_size_select(n, nnz)
                     for n, nnz in ((1000, 5000), (10**6, 10**7), (150, 400), (4096, 520318),
                                    (262144, 346856394), (10**6, 102394612), (200000, 15119658))}
    # partition example (SPEC.md:334-336; :336 is wrong in the SPEC, code is truth)
    a = R.generate("tridiagonal", 4)
    f = R.symbolic_factorize(R.symmetrize_pattern(a))
    g = R.partition(f, a, R.BlockingPlan(4, np.array([0, 2, 4]), "regular"))
    out["partition_tridiag4_block_nnz"] = g.block_nnz.tolist()
    # dense p=3 levels and block-diagonal p=3
    a = R.generate("dense", 9)
    f = R.symbolic_factorize(R.symmetrize_pattern(a))
    t = R.dependency_levels(R.partition(f, a, R.regular_plan(9, 3)))
    out["levels_dense9_bs3"] = {"tasks": t.task_count, "levels": t.n_levels,
                                "kinds": t.kinds.tolist(), "levels_of": t.levels_of.tolist()}
    # GETRF 2x2 examples
    for name, b in (("getrf_diag", [[2.0, 0.0], [0.0, 3.0]]), ("getrf_swap", [[0.0, 1.0], [1.0, 0.0]])):
        lo, up, perm = R.factor_diagonal(np.array(b))
        out[name] = {"L": lo.tolist(), "U": up.tolist(), "perm": perm.tolist()}
    out["arrowhead_100_10_nnz"] = R.generate("arrowhead", 100, b=10).nnz
    # generator hashes (pin the port of matrix_io.generate)
    gens = {}
    for kind, n, kw in (("tridiagonal", 50, {}), ("dense", 12, {}), ("arrowhead", 200, {"b": 20}),
                        ("random_spd", 300, {"bandwidth": 6, "density": 0.4})):
        for seed in (0, 3):
            m = R.generate(kind, n, seed=seed, **kw)
            gens[f"{kind}_{n}_{seed}"] = [sha(m.col_ptr), sha(m.row_idx), sha(m.values)]
    out["generate_sha"] = gens
    return out


def run_ref(a, plan="irregular", bs=None, static_pivot=None):
    ar = ref_csc(a)
    t0 = time.perf_counter()
    f = R.symbolic_factorize(R.symmetrize_pattern(ar))
    bptr = R.diag_block_pointer(f)
    curve = R.percentage_curve(bptr)
    pl = R.irregular_plan(curve, a.n) if plan == "irregular" else R.regular_plan(a.n, bs)
    g = R.partition(f, ar, pl)
    tr = R.dependency_levels(g)
    t1 = time.perf_counter()
    return ar, f, bptr, curve, pl, g, tr, t1 - t0


def structure_record(f, bptr, curve, pl, g, tr):
    keys = list(g.blocks.keys())
    bcp = np.concatenate([g.blocks[k].col_ptr for k in keys])
    bri = np.concatenate([g.blocks[k].row_idx for k in keys])
    bval = np.concatenate([g.blocks[k].values for k in keys])
    rec = {
        "n": int(f.n), "nnz_filled": int(f.nnz_filled), "p": int(pl.p), "nblocks": len(keys),
        "tasks": int(tr.task_count), "levels": int(tr.n_levels),
        "filled_col_ptr": sha(f.col_ptr), "filled_row_idx": sha(f.row_idx),
        "blockptr": sha(bptr.blockptr), "pct": sha(curve.pct), "positions": sha(pl.positions),
        "block_keys": sha(np.array(keys, dtype=np.int64).ravel()),
        "block_col_ptr": sha(bcp), "block_row_idx": sha(bri), "block_values": sha(bval),
        "block_nnz": sha(g.block_nnz), "value_max": float(g.value_max),
    }
    for fld in ("kinds", "steps", "rows", "cols", "weights", "costs", "levels_of", "pred_ptr", "pred_idx"):
        rec["tree_" + fld] = sha(getattr(tr, fld))
    return rec


def factor_samples(fac, keys_l, keys_u, per_block=8):
    """Per-block value samples: (key..., local index, value) for L and U, plus abs sums."""
    out = {}
    for tag, blocks, keys in (("L", fac.l_blocks, keys_l), ("U", fac.u_blocks, keys_u)):
        rows = []
        sums = []
        for (bi, bj) in keys:
            b = blocks[(bi, bj)]
            nz = b.nnz
            idx = np.unique(np.linspace(0, max(nz - 1, 0), min(per_block, nz)).astype(np.int64)) if nz else []
            for e in idx:
                rows.append((bi, bj, int(e), float(b.values[e])))
            sums.append((bi, bj, nz, float(np.abs(b.values).sum()), sha(b.col_ptr), sha(b.row_idx),
                         float(np.dot(proj_weights(nz), b.values)), float(np.abs(b.values).max(initial=0.0))))
        out[tag + "_samples"] = rows
        out[tag + "_blocks"] = sums
    return out


def named_case(name, a, plan="irregular", bs=None, factor=True):
    print(f"[{name}] n={a.n} nnz={a.nnz}", flush=True)
    ar, f, bptr, curve, pl, g, tr, tpre = run_ref(a, plan, bs)
    rec = structure_record(f, bptr, curve, pl, g, tr)
    rec["preprocess_s"] = tpre
    arrays = {"positions": pl.positions, "pct": curve.pct}
    if factor:
        t0 = time.perf_counter()
        fac = R.factorize(g, tr, workers=1)
        rec["factorize_s"] = time.perf_counter() - t0
        rec["residual"] = R.residual(ar, fac)
        b = ar.to_scipy() @ np.ones(a.n)
        x = R.solve(fac, b)
        rec["relres"] = float(np.linalg.norm(ar.to_scipy() @ x - b) / np.linalg.norm(b))
        rec["perm_global"] = sha(fac.perm_global())
        kl = sorted(fac.l_blocks, key=lambda k: (k[1], k[0]))
        ku = sorted(fac.u_blocks, key=lambda k: (k[1], k[0]))
        per = 32 if name == "C5" else max(1, min(8, 20000 // max(1, len(kl))))
        s = factor_samples(fac, kl, ku, per_block=per)
        for tag in ("L", "U"):
            arrays[tag + "_samples_key"] = np.array([r[:3] for r in s[tag + "_samples"]], np.int64)
            arrays[tag + "_samples_val"] = np.array([r[3] for r in s[tag + "_samples"]], np.float64)
            arrays[tag + "_blocks_key"] = np.array([r[:3] for r in s[tag + "_blocks"]], np.int64)
            arrays[tag + "_blocks_abssum"] = np.array([r[3] for r in s[tag + "_blocks"]], np.float64)
            arrays[tag + "_blocks_proj"] = np.array([r[6] for r in s[tag + "_blocks"]], np.float64)
            arrays[tag + "_blocks_absmax"] = np.array([r[7] for r in s[tag + "_blocks"]], np.float64)
            rec[tag + "_pattern_sha"] = sha(np.array([hash_pair(r[4], r[5]) for r in s[tag + "_blocks"]],
                                                     dtype=np.int64))
    np.savez_compressed(os.path.join(HERE, f"case_{name}.npz"), **arrays)
    print(f"   -> p={rec['p']} tasks={rec['tasks']} levels={rec['levels']} "
          f"factor={rec.get('factorize_s', 0):.2f}s res={rec.get('residual')}", flush=True)
    return rec


def proj_weights(m: int) -> np.ndarray:
    """Deterministic +-1 weights of a block's value projection (tests/golden: checksum of every value)."""
    e = np.arange(m, dtype=np.uint64)
    h = (e * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(40)
    return np.where(h & np.uint64(1), 1.0, -1.0)


def hash_pair(a: str, b: str) -> int:
    return int(hashlib.sha256((a + b).encode()).hexdigest()[:15], 16)


def small_cases():
    """Full inputs and outputs for n <= 64 random patterns (pinning bitwise behaviour)."""
    rng = np.random.default_rng(2512)
    made = 0
    for idx in range(22):
        n = int(rng.integers(4, 48))
        pat = RO.random_symmetric_pattern(n, rng, fill=float(rng.uniform(0.05, 0.3)))
        a = RO.pattern_to_matrix(n, pat, rng)
        static_pivot = None
        if idx >= 14:
            # non-dominant values: block-local pivoting swaps rows (the §3.2 quirk)
            vals = rng.uniform(-1.0, 1.0, a.nnz)
            if idx >= 19:
                # a singular leading column: ZeroPivot, or static pivoting for idx 21
                cols = np.repeat(np.arange(n), np.diff(a.col_ptr))
                vals[cols == 0] = 0.0
                static_pivot = 1e-8 if idx == 21 else None
            a = R.CscMatrix(n, a.col_ptr, a.row_idx, vals)
        if idx % 3 == 0:
            pos = R.regular_plan(n, max(1, n // int(rng.integers(1, 5)))).positions
        else:
            f0 = R.symbolic_factorize(R.symmetrize_pattern(a))
            pos = R.irregular_plan(R.percentage_curve(R.diag_block_pointer(f0), int(rng.integers(4, 40))),
                                   n).positions
        f = R.symbolic_factorize(R.symmetrize_pattern(a))
        plan = R.BlockingPlan(n, np.asarray(pos), "given")
        g = R.partition(f, a, plan)
        tr = R.dependency_levels(g)
        rec = {"n": n, "a_col_ptr": a.col_ptr, "a_row_idx": a.row_idx, "a_values": a.values,
               "filled_col_ptr": f.col_ptr, "filled_row_idx": f.row_idx,
               "blockptr": R.diag_block_pointer(f).blockptr, "positions": plan.positions}
        for fld in ("kinds", "steps", "rows", "cols", "weights", "costs", "levels_of", "pred_ptr", "pred_idx"):
            rec["tree_" + fld] = getattr(tr, fld)
        rec["static_pivot"] = np.array([np.nan if static_pivot is None else static_pivot])
        try:
            fac = R.factorize(g, tr, static_pivot=static_pivot)
            rec["zero_pivot"] = np.array([-1, -1])
            lk = sorted(fac.l_blocks)
            uk = sorted(fac.u_blocks)
            for tag, blocks, keys in (("L", fac.l_blocks, lk), ("U", fac.u_blocks, uk)):
                rec[tag + "_keys"] = np.array(keys, np.int64).reshape(-1, 2)
                rec[tag + "_col_ptr"] = np.concatenate([blocks[k].col_ptr for k in keys])
                rec[tag + "_row_idx"] = np.concatenate([blocks[k].row_idx for k in keys])
                rec[tag + "_values"] = np.concatenate([blocks[k].values for k in keys])
            rec["perm_global"] = fac.perm_global()
            rec["residual"] = np.array([R.residual(a, fac)])
            rec["swapped"] = np.array([int(not np.array_equal(fac.perm_global(), np.arange(n)))])
        except R.ZeroPivot as zp:
            rec["zero_pivot"] = np.array([zp.block, zp.col])
        np.savez_compressed(os.path.join(HERE, f"small_{idx:02d}.npz"), **rec)
        made += 1
    return made


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2", action="store_true", help="also pin C2 structure (~5 min, ~35 GB RAM)")
    ap.add_argument("--c3", action="store_true", help="pin C3 structure (reference symbolic on n=1e6)")
    ap.add_argument("--c5", action="store_true", help="pin C5 structure + factor checksums (~22 GB scratch)")
    ap.add_argument("--only", default=None, help="comma list of named cases to (re)make")
    ap.add_argument("--skip-small", action="store_true")
    args = ap.parse_args()
    with open(os.path.join(HERE, "spec.json"), "w") as fh:
        json.dump(spec_examples(), fh, indent=1)
    if not args.skip_small:
        print("small cases:", small_cases())
    cases_path = os.path.join(HERE, "cases.json")
    cases = json.load(open(cases_path)) if os.path.exists(cases_path) else {}
    from paper_2512_04389_b200.matrix_io import generate as gen
    todo = {
        "C1": (lambda: G.poisson2d(64), "irregular", None, True),
        "C1_reg200": (lambda: G.poisson2d(64), "regular", 200, True),
        "C1_reg500": (lambda: G.poisson2d(64), "regular", 500, True),
        "arrow1000": (lambda: gen("arrowhead", 1000, b=100), "irregular", None, True),
        "tridiag2000": (lambda: gen("tridiagonal", 2000), "irregular", None, True),
        "randspd3000": (lambda: gen("random_spd", 3000, bandwidth=20, density=0.3), "irregular", None, True),
        "poisson3d16nd": (lambda: G.poisson3d(16, "nd"), "irregular", None, True),
        "bbd20k": (lambda: G.bbd(20000, 400, 20, seed=1), "irregular", None, True),
        "bbd20k_reg500": (lambda: G.bbd(20000, 400, 20, seed=1), "regular", 500, True),
    }
    if args.c2:
        todo["C2"] = (lambda: G.poisson3d(64, "nd"), "irregular", None, False)
    if args.c3:
        todo["C3"] = (lambda: G.bbd(1_000_000, 10_000, 1000, seed=0), "irregular", None, False)
    if args.c5:
        todo["C5"] = (lambda: G.bbd(200_000, 4_000, 200, seed=0), "irregular", None, True)
    if args.only:
        keep = set(args.only.split(","))
        todo = {k: v for k, v in todo.items() if k in keep}
    for name, (mk, plan, bs, fac) in todo.items():
        a = mk()
        rec = named_case(name, a, plan, bs, fac)
        rec["a_sha"] = [sha(a.col_ptr), sha(a.row_idx), sha(a.values)]
        cases[name] = rec
        with open(cases_path, "w") as fh:
            json.dump(cases, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
