"""2D block-cyclic distribution: host logic + a world_size-2/4 gloo execution on CPU.

The gloo run executes the owner-computes schedule of parallel.exchange_plan
with the oracle's kernels in separate processes, moving block values with
torch.distributed send/recv exactly where the plan says, and checks that the
distributed factors are BITWISE equal to the serial ones (SURVEY.md §4,
multi-GPU tests (a) and (c), on CPU).
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2512_04389_b200 as M
from paper_2512_04389_b200 import generators as G
from paper_2512_04389_b200.parallel import ProcGrid, check_residency, comm_volume, exchange_plan, task_owners


def structure(a, bs=None):
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    pl = M.irregular_plan(M.percentage_curve(M.diag_block_pointer(f)), a.n) if bs is None else M.regular_plan(a.n, bs)
    g = M.partition(f, a, pl)
    return g, M.dependency_levels(g)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_residency_and_owner_chain(world):
    g, t = structure(G.poisson3d(12, "nd"))
    pg = ProcGrid.for_world(world)
    check_residency(g, t, pg)
    own = task_owners(t, pg)
    # the update chain of every target stays on one rank
    upd = t.kinds == M.SSSSM
    for r, c, o in zip(t.rows[upd], t.cols[upd], own[upd]):
        assert o == pg.owner(int(r), int(c))
    vol = comm_volume(g, t, pg)
    assert vol["total"] > 0 and len(vol["per_level"]) == t.n_levels


def test_single_rank_needs_no_messages():
    g, t = structure(G.poisson2d(24))
    assert all(len(lv) == 0 for lv in exchange_plan(t, ProcGrid(1, 1)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mat, bs, out_dir):
    import torch

    from oracle import numeric as ON

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = {"p2": lambda: G.poisson2d(20), "bbd": lambda: G.bbd(3000, 120, 10, seed=2)}[mat]()
    g, t = structure(a, bs)
    pg = ProcGrid.for_world(world)
    own = task_owners(t, pg)
    plan = exchange_plan(t, pg)
    state = {k: ON.dense(b) for k, b in g.blocks.items() if pg.owner(*k) == rank}
    recv = {}
    perms = {}

    def get(k):
        return state[k] if k in state else recv[k]

    for lv, tasks in enumerate(t.levels):
        for tid in tasks:
            if own[tid] != rank:
                continue
            kind, i, r, c = int(t.kinds[tid]), int(t.steps[tid]), int(t.rows[tid]), int(t.cols[tid])
            if kind == M.SSSSM:
                if (r, c) in state:
                    state[(r, c)] -= get((r, i)) @ get((i, c))
            elif kind == M.GESSM:
                x = state[(i, c)]
                if perms.get(i) is not None:
                    x[:] = x[perms[i]]
                ON.gessm(get((i, i)), x)
            elif kind == M.TSTRF:
                ON.tstrf(state[(r, i)], get((i, i)))
            else:
                p_, sw = ON.getrf(state[(i, i)])
                perms[i] = p_ if sw else None
        for ex in plan[lv]:
            for d in ex.dst:
                if rank == ex.src:
                    blk = state[ex.block]
                    dist.send(torch.from_numpy(np.ascontiguousarray(blk)), d)
                    if ex.with_perm:
                        pv = perms.get(ex.block[0])
                        pv = np.arange(blk.shape[0]) if pv is None else pv
                        dist.send(torch.from_numpy(pv.astype(np.int64)), d)
                elif rank == d:
                    bi, bj = ex.block
                    b = g.blocks[ex.block]
                    buf = torch.empty((b.nrows, b.ncols), dtype=torch.float64)
                    dist.recv(buf, ex.src)
                    recv[ex.block] = buf.numpy()
                    if ex.with_perm:
                        pb = torch.empty(b.nrows, dtype=torch.int64)
                        dist.recv(pb, ex.src)
                        pv = pb.numpy()
                        perms[bi] = None if np.array_equal(pv, np.arange(b.nrows)) else pv
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
             **{f"{k[0]}_{k[1]}": v for k, v in state.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mat,bs", [(2, "p2", None), (2, "bbd", None), (4, "p2", 50)])
def test_gloo_distributed_factors_bitwise_equal(tmp_path, world, mat, bs):
    from oracle import numeric as ON

    port = _free_port()
    mp.spawn(_worker, args=(world, port, mat, bs, str(tmp_path)), nprocs=world, join=True)
    a = {"p2": lambda: G.poisson2d(20), "bbd": lambda: G.bbd(3000, 120, 10, seed=2)}[mat]()
    g, t = structure(a, bs)
    from oracle import structure as OS

    og = OS.Grid(g.n, g.p, g.plan.positions, g.blocks, g.block_nnz, g.value_max)
    ref, _ = ON.factorize(og, t)
    got = {}
    for r in range(world):
        z = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        for k in z.files:
            bi, bj = map(int, k.split("_"))
            got[(bi, bj)] = z[k]
    assert set(got) == set(ref)
    for k in ref:
        assert got[k].tobytes() == ref[k].tobytes(), k


def test_bench_gpus_n_fails_loudly_without_enough_gpus():
    """bench.py --gpus N spawns N ranks itself; with fewer visible GPUs it exits non-zero and says why."""
    import subprocess
    import sys

    import torch

    if torch.cuda.is_available() and torch.cuda.device_count() >= 2:
        pytest.skip("enough GPUs to spawn")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "needs one GPU per rank" in r.stderr
