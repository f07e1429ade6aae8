"""Debug: 4-rank gloo DistEngine on one GPU vs the single engine, per block."""
import os, sys, socket
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import torch.multiprocessing as mp


def worker(rank, world, port, out):
    import torch.distributed as dist
    from test_dist_device import _case
    from paper_2512_04389_b200.parallel import DistEngine
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, t, sp = _case(sys.argv[1] if len(sys.argv) > 1 else "p3d")
    de = DistEngine(g, t)
    if rank == 2:
        lay = de.eng.block_layout()
        print("rank2 first segs", [[(k, peer, v.numel()) for k, peer, v in o][:6] for o in de.seg_ops[:3]], flush=True)
        print("layout first blocks", lay[:, :6].tolist(), "table", de.eng.pool.table[:, :6].tolist(), flush=True)
        print("vals ptr", de.vals.data_ptr(), de.eng.work_ptrs(), flush=True)
    de.upload()
    ms, st = de.run()
    v, p = de.eng.download()
    np.savez(f"{out}/r{rank}.npz", v=v, own=de.owned_entries(), nseg=de.eng.n_segments, msgs=de.messages,
             routes=de.eng.task_routes())
    dist.barrier(); dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    out = "gpurun_out/dbg"; os.makedirs(out, exist_ok=True)
    mp.spawn(worker, args=(world, port, out), nprocs=world, join=True)
    from test_dist_device import _case
    from paper_2512_04389_b200.numeric import Engine
    from paper_2512_04389_b200.parallel import ProcGrid, task_owners
    g, t, sp = _case(sys.argv[1] if len(sys.argv) > 1 else "p3d")
    e = Engine(g, t); e.upload(); e.run_device(); ref, _ = e.download()
    pg = ProcGrid.for_world(world)
    own = task_owners(t, pg)
    tab = e.pool.table
    starts = tab[6]
    for r in range(world):
        z = np.load(f"{out}/r{r}.npz")
        print("rank", r, "segments", int(z["nseg"]), "msgs", int(z["msgs"]), "routes", np.bincount(z["routes"] + 1))
    got = sum(np.where(np.load(f"{out}/r{r}.npz")["own"], np.load(f"{out}/r{r}.npz")["v"], 0.0) for r in range(world))
    bad = 0
    for b in range(tab.shape[1]):
        bi, bj, nr, nc, nz, cp, eo = tab[:, b]
        d = got[eo:eo + nz] - ref[eo:eo + nz]
        if np.any(d != 0):
            bad += 1
            if bad <= 12:
                ks = [(int(t.kinds[q]), int(t.steps[q]), int(t.levels_of[q]), int(own[q]))
                      for q in range(t.task_count)
                      if (t.kinds[q] in (1, 2, 3) and (t.rows[q], t.cols[q]) == (bi, bj)) or
                      (t.kinds[q] == 0 and bi == bj == t.steps[q]) or
                      (t.kinds[q] == 1 and (t.steps[q], t.cols[q]) == (bi, bj)) or
                      (t.kinds[q] == 2 and (t.rows[q], t.steps[q]) == (bi, bj))]
                print("block", (bi, bj), "owner", pg.owner(bi, bj), "maxdiff", np.abs(d).max(), "nz", nz,
                      "zeros got", int((got[eo:eo+nz] == 0).sum()), "tasks(kind,step,level,owner)", ks[:8])
    print("bad blocks", bad, "of", tab.shape[1])
