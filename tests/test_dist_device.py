"""Distributed device factorization (parallel.DistEngine) vs the single-GPU engine.

World sizes 2 (1x2) and 4 (2x2) run as separate processes sharing cuda:0
over the gloo backend (host-staged block exchange); the owner-computes
schedule, the task masks, the graph segments and the per-level exchange
lists are the ones the NCCL backend runs on 2-8 GPUs.  Factors must be
BITWISE equal to the single-GPU factors (SURVEY.md §8e parity), errors must
be raised identically on every rank.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2512_04389_b200 as M
from conftest import load_small
from paper_2512_04389_b200 import generators as G

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(name):
    if name.startswith("small"):
        d = load_small(int(name[5:]))
        a = M.CscMatrix(int(d["n"]), d["a_col_ptr"], d["a_row_idx"], d["a_values"])
        f = M.symbolic_factorize(M.symmetrize_pattern(a))
        g = M.partition(f, a, M.BlockingPlan(a.n, np.asarray(d["positions"], np.int64), "given"))
        sp = float(d["static_pivot"][0])
        return g, M.dependency_levels(g), (None if np.isnan(sp) else sp)
    a = {"p3d": lambda: G.poisson3d(10, "nd"), "bbd": lambda: G.bbd(6000, 200, 20, seed=1),
         "p2reg": lambda: G.poisson2d(24)}[name]()
    f = M.symbolic_factorize(M.symmetrize_pattern(a))
    plan = (M.regular_plan(a.n, 60) if name == "p2reg"
            else M.irregular_plan(M.percentage_curve(M.diag_block_pointer(f)), a.n))
    g = M.partition(f, a, plan)
    return g, M.dependency_levels(g), None


def _flatten(lu):
    out = {"perm": lu.perm_global()}
    for tag, blocks in (("L", lu.l_blocks), ("U", lu.u_blocks)):
        for (bi, bj), b in blocks.items():
            out[f"{tag}_{bi}_{bj}_cp"] = b.col_ptr
            out[f"{tag}_{bi}_{bj}_ri"] = b.row_idx
            out[f"{tag}_{bi}_{bj}_v"] = b.values
    return out


def _worker(rank, world, port, name, out_dir):
    import torch.distributed as dist

    from paper_2512_04389_b200.parallel import factorize_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, t, sp = _case(name)
    try:
        lu = factorize_distributed(g, t, static_pivot=sp)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **_flatten(lu))
    except M.ZeroPivot as e:
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), zero_pivot=np.array([e.block, e.col]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "p3d"), (4, "p3d"), (8, "p3d"), (2, "bbd"), (8, "bbd"), (4, "p2reg"),
                                        (2, "small15"), (2, "small21"), (2, "small19")])
def test_distributed_factors_bitwise_equal_to_single_gpu(tmp_path, world, name):
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    g, t, sp = _case(name)
    try:
        want = _flatten(M.factorize(g, t, static_pivot=sp))
    except M.ZeroPivot as e:
        want = {"zero_pivot": np.array([e.block, e.col])}
    for r in range(world):
        got = dict(np.load(os.path.join(tmp_path, f"rank{r}.npz")))
        assert set(got) == set(want), r
        for k in want:
            assert got[k].dtype == want[k].dtype or k == "zero_pivot", k
            assert got[k].tobytes() == want[k].tobytes(), (r, k)


def test_distributed_plan_splits_work_and_segments():
    """Single-process check of the distributed plan hooks: with a task mask the
    engine runs only the owned tasks, and the cuts become graph segments."""
    from paper_2512_04389_b200.numeric import Engine
    from paper_2512_04389_b200.parallel import ProcGrid, exchange_plan, task_owners

    g, t, _ = _case("p3d")
    pg = ProcGrid(1, 2)
    own = task_owners(t, pg)
    plan = exchange_plan(t, pg)
    cuts = np.array([any(ex.src == 0 or 0 in ex.dst for ex in lv) for lv in plan], np.int8)
    e0 = Engine(g, t, mask=(own == 0).astype(np.int8), cuts=cuts)
    full = Engine(g, t)
    r0, rf = e0.task_routes(), full.task_routes()
    assert np.all(r0[own != 0] == -1)
    assert np.array_equal(r0[own == 0], rf[own == 0])
    assert e0.n_segments == int(cuts.sum()) + 1
    lay = e0.block_layout()
    assert np.all(np.diff(lay[0]) >= 0)
    # working storage only for the blocks rank 0's tasks touch: its owned blocks + received operands
    touched = set()
    for q in np.flatnonzero(own == 0):
        i, r, c, k = int(t.steps[q]), int(t.rows[q]), int(t.cols[q]), int(t.kinds[q])
        touched.add((i, i))
        if k == M.GESSM:
            touched.add((i, c))
        elif k == M.TSTRF:
            touched.add((r, i))
        elif k == M.SSSSM:
            touched.update({(r, i), (i, c), (r, c)})
    keys = list(zip(e0.pool.table[0], e0.pool.table[1]))
    res = np.array([(int(bi), int(bj)) in touched for bi, bj in keys])
    assert np.all(lay[1][res] > 0) and np.all(lay[1][~res] == 0)
    assert e0.nnz_work < full.nnz_work
    e0.close()
    full.close()
