"""Executor DAG analysis: where do the tile-DAG levels lose time?

    python scripts/exec_dag.py capture C2 gpurun_out/c2_dag.npz     (GPU box: one traced replay)
    python scripts/exec_dag.py analyze gpurun_out/c2_dag.npz [--slots 296] [--top 20]

For every executor launch: the measured span, the critical path of its task DAG
with the measured task run times (ready -> done), the work bound (sum of run
times / CTA slots) and a list-schedule simulation with a ready queue (tasks
popped by upward rank only once their dependencies are met) — the gap between
the span and max(critical path, work bound) is scheduling loss.
"""
import argparse
import sys

import numpy as np

sys.path.insert(0, ".")

NAMES = ["COLMAX", "GETRF", "TRSM_L", "TRSM_U", "GEMM", "FINAL", "PG_DIAG", "PG_UPD", "PT_DIAG", "PT_UPD",
         "BAND", "GETRF_UPD", "PG_FUSED", "PT_FUSED", "NOP", "SSSSM"]


def capture(cfg, out):
    import bench
    from paper_2512_04389_b200.numeric import Engine

    a, f, g, t = bench.build_case(cfg, "irregular", None)
    eng = Engine(g, t)
    eng.upload()
    eng.run_device()
    ms = sorted(eng.run_device() for _ in range(3))[1]
    lt = eng.level_times()
    tr, info = eng.exec_trace()
    sptr, succ = eng.exec_graph()
    np.savez_compressed(out, trace=tr.astype(np.int64), info=info, sptr=sptr, succ=succ, lt=lt, ms=ms)
    print(f"captured {cfg}: graph {ms:.2f} ms, {len(info)} executor tasks -> {out}")


def _preds(m, lp, succ):
    pred = [[] for _ in range(m)]
    for i in range(m):
        for e in range(lp[i], lp[i + 1]):
            pred[succ[e] >> 1].append(i)
    return pred


def sim_inorder(m, run, lp, succ, slots):
    """The current executor: CTAs take tasks in index order and hold them until ready."""
    import heapq

    pred = _preds(m, lp, succ)
    free = [0.0] * slots
    heapq.heapify(free)
    fin = np.zeros(m)
    for i in range(m):
        t0 = heapq.heappop(free)
        ready = max((fin[p] for p in pred[i]), default=0.0)
        fin[i] = max(t0, ready) + run[i]
        heapq.heappush(free, fin[i])
    return fin.max() if m else 0.0


def sim_ready(m, run, lp, succ, slots):
    """A ready queue: an idle CTA takes the highest-priority (lowest index) READY task."""
    import heapq

    indeg = np.zeros(m, np.int64)
    for e in range(lp[0], lp[m]):
        indeg[succ[e] >> 1] += 1
    ready = [i for i in range(m) if indeg[i] == 0]
    heapq.heapify(ready)
    running = []  # (finish, task)
    idle = slots
    now = 0.0
    done = 0
    while done < m:
        while idle and ready:
            i = heapq.heappop(ready)
            heapq.heappush(running, (now + run[i], i))
            idle -= 1
        now, i = heapq.heappop(running)
        idle += 1
        done += 1
        for e in range(lp[i], lp[i + 1]):
            j = succ[e] >> 1
            indeg[j] -= 1
            if indeg[j] == 0:
                heapq.heappush(ready, j)
    return now


def analyze(path, slots, top):
    z = np.load(path)
    tr, info, sptr, succ, lt = z["trace"], z["info"], z["sptr"], z["succ"], z["lt"]
    n = len(info)
    lvl = info[:, 5]
    cnt = np.bincount(lvl, minlength=len(lt))
    first = np.r_[0, np.cumsum(cnt)]
    print(f"# graph {float(z['ms']):.2f} ms; executor level sum {lt[:, 3].sum():.2f} ms over "
          f"{int((cnt > 0).sum())} launches")
    rows = []
    sp_off = su_off = 0
    for l in range(len(lt)):  # every launch level owns nexec + 1 successor offsets
        lo, m = first[l], cnt[l]
        hi = lo + m
        lp = sptr[sp_off: sp_off + m + 1] + su_off  # local offsets into this level's successor entries
        sp_off += m + 1
        su_off = lp[-1]
        if m == 0:
            continue
        T = tr[lo:hi]
        ty = info[lo:hi, 0]
        # run time from the moment both dependency phases were met (slot 7: phase-2 operands complete)
        run = np.maximum(T[:, 2] - np.maximum(T[:, 1], T[:, 7]), 0) / 1e3
        span = (T[:, 2].max() - T[:, 0].min()) / 1e3
        # critical path (tasks are stored in a topological order: upward rank descending;
        # successor entries are level-local)
        fin = np.zeros(m)
        est = np.zeros(m)
        for i in range(m):
            fin[i] = est[i] + run[i]
            for e in range(lp[i], lp[i + 1]):
                j = succ[e] >> 1
                if fin[i] > est[j]:
                    est[j] = fin[i]
        cp = fin.max()
        work = run.sum() / slots
        sim_in = sim_inorder(m, run, lp, succ, slots)
        sim_rq = sim_ready(m, run, lp, succ, slots)
        rows.append((int(lvl[lo]), span, cp, work, m, run, ty, sim_in, sim_rq))
    rows.sort(key=lambda r: -r[1])
    tot_span = sum(r[1] for r in rows)
    tot_cp = sum(r[2] for r in rows)
    tot_lb = sum(max(r[2], r[3]) for r in rows)
    tot_in = sum(r[7] for r in rows)
    tot_rq = sum(r[8] for r in rows)
    print(f"# sum span {tot_span / 1e3:.2f} ms | sum critical path {tot_cp / 1e3:.2f} ms | "
          f"sum max(cp, work/slots) {tot_lb / 1e3:.2f} ms | simulated in-order {tot_in / 1e3:.2f} ms | "
          f"simulated ready-queue {tot_rq / 1e3:.2f} ms")
    print("# per launch (ms): measured span, critical path, work/slots, simulated in-order, simulated ready-queue")
    for L, span, cp, work, m, run, ty, si, sr in rows[:top]:
        mix = {NAMES[t]: int(c) for t, c in zip(*np.unique(ty, return_counts=True))}
        print(f"L{L:4d} span {span / 1e3:6.3f} cp {cp / 1e3:6.3f} work {work / 1e3:6.3f} "
              f"in-order {si / 1e3:6.3f} ready-q {sr / 1e3:6.3f} tasks {m:6d} {mix}")
    # per-type run time
    ok = tr[:, 2] > 0
    for t in np.unique(info[:, 0]):
        s = (info[:, 0] == t) & ok
        r = (tr[s, 2] - np.maximum(tr[s, 1], tr[s, 7])) / 1e3
        w = (np.maximum(tr[s, 1], tr[s, 7]) - tr[s, 0]) / 1e3
        print(f"{NAMES[t]:9s} n={s.sum():7d} run med {np.median(r):6.2f} us sum {r.sum() / 1e3:8.2f} ms | "
              f"held-while-waiting med {np.median(w):6.2f} us sum {w.sum() / 1e3:8.2f} ms")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["capture", "analyze"])
    ap.add_argument("arg1")
    ap.add_argument("arg2", nargs="?")
    ap.add_argument("--slots", type=int, default=296)
    ap.add_argument("--top", type=int, default=20)
    a = ap.parse_args()
    if a.mode == "capture":
        capture(a.arg1, a.arg2)
    else:
        analyze(a.arg1, a.slots, a.top)
