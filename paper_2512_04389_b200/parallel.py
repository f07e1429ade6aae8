"""2D block-cyclic distribution of the block LU over Pr x Pc GPUs (north-star subsystem 5).

The reference has no distribution.  Ownership follows
SURVEY.md §8e: block (bi, bj) lives on rank ``(bi % Pr) * Pc + (bj % Pc)``
and every task runs on the owner of the block it writes (owner-computes):
GETRF(i) @ (i,i), GESSM(i,j) @ (i,j), TSTRF(k,i) @ (k,i), SSSSM(k,j,i) @ (k,j).
The whole ascending-step update chain of a target therefore stays on one
rank, so distributed factors are bitwise equal to single-GPU factors.

After each dependency level, every block a task finished there is sent to
the ranks that read it later:
  GETRF(i)    -> owners of GESSM(i,·) and TSTRF(·,i)   (L_ii, U_ii, perm_i)
  GESSM(i,j)  -> owners of SSSSM(·,j,i)                (U_ij along process column j % Pc)
  TSTRF(k,i)  -> owners of SSSSM(k,·,i)                (L_ki along process row k % Pr)
Messages carry values only: the patterns are static and replicated at plan
time.  ``exchange_plan`` produces these per-level lists; the device engine
turns each level's list into one NCCL group of send/recv (or broadcasts on
row / column communicators).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import GESSM, GETRF, SSSSM, TSTRF


@dataclass(frozen=True)
class ProcGrid:
    pr: int
    pc: int

    @property
    def size(self) -> int:
        return self.pr * self.pc

    def owner(self, bi: int, bj: int) -> int:
        return (bi % self.pr) * self.pc + (bj % self.pc)

    @staticmethod
    def for_world(world: int) -> "ProcGrid":
        """1x1, 1x2, 2x2, 2x4 for 1/2/4/8 GPUs; otherwise 1 x world."""
        table = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}
        pr, pc = table.get(world, (1, world))
        return ProcGrid(pr, pc)


def task_targets(tree):
    """(row, col) of the block each task writes."""
    kinds = tree.kinds
    r = np.where(kinds == GETRF, tree.steps, tree.rows).astype(np.int64)
    c = np.where(kinds == TSTRF, tree.steps, tree.cols).astype(np.int64)
    r = np.where(kinds == GESSM, tree.steps, r)
    return r, c


def task_owners(tree, pg: ProcGrid) -> np.ndarray:
    r, c = task_targets(tree)
    return (r % pg.pr) * pg.pc + (c % pg.pc)


@dataclass
class Exchange:
    level: int
    block: tuple      # (bi, bj) produced at this level
    src: int
    dst: tuple        # ranks that need it, src excluded
    with_perm: bool   # GETRF output also carries the local permutation


def exchange_plan(tree, pg: ProcGrid) -> list[list[Exchange]]:
    """Per level (index = ASAP level) the messages sent after it completes."""
    own = task_owners(tree, pg)
    nl = tree.n_levels
    out: list[list[Exchange]] = [[] for _ in range(nl)]
    readers: dict = {}  # block -> set of ranks reading it as an operand
    kinds, steps, rows, cols = tree.kinds, tree.steps, tree.rows, tree.cols
    for t in range(tree.task_count):
        k = int(kinds[t])
        i, r, c = int(steps[t]), int(rows[t]), int(cols[t])
        o = int(own[t])
        if k in (GESSM, TSTRF):
            readers.setdefault((i, i), set()).add(o)
        elif k == SSSSM:
            readers.setdefault((r, i), set()).add(o)
            readers.setdefault((i, c), set()).add(o)
    for t in range(tree.task_count):
        k = int(kinds[t])
        if k == SSSSM:
            continue
        i, r, c = int(steps[t]), int(rows[t]), int(cols[t])
        blk = (i, i) if k == GETRF else ((i, c) if k == GESSM else (r, i))
        src = int(own[t])
        dst = tuple(sorted(readers.get(blk, set()) - {src}))
        if dst:
            out[int(tree.levels_of[t])].append(Exchange(int(tree.levels_of[t]), blk, src, dst, k == GETRF))
    return out


def check_residency(grid, tree, pg: ProcGrid) -> None:
    """Simulate the schedule: every operand a task reads must be on its rank.

    Raises AssertionError naming the first violation (multi-GPU test (a)).
    """
    own = task_owners(tree, pg)
    plan = exchange_plan(tree, pg)
    resident = {rank: set() for rank in range(pg.size)}
    for (bi, bj) in grid.blocks:
        resident[pg.owner(bi, bj)].add((bi, bj))
    by_level = tree.levels
    for lv, tasks in enumerate(by_level):
        for t in tasks:
            k = int(tree.kinds[t])
            i, r, c = int(tree.steps[t]), int(tree.rows[t]), int(tree.cols[t])
            o = int(own[t])
            need = {GETRF: [(i, i)], GESSM: [(i, i), (i, c)], TSTRF: [(i, i), (r, i)],
                    SSSSM: [(r, i), (i, c)]}[k]
            for blk in need:
                assert blk in resident[o], f"task {t} (kind {k}) on rank {o} lacks block {blk} at level {lv}"
        for ex in plan[lv]:
            for d in ex.dst:
                resident[d].add(ex.block)


def comm_volume(grid, tree, pg: ProcGrid) -> dict:
    """Bytes moved per level (values only, 8 B per stored entry) and in total."""
    plan = exchange_plan(tree, pg)
    per = []
    for lv in plan:
        b = 0
        for ex in lv:
            blk = grid.blocks[ex.block]
            b += 8 * blk.nnz * len(ex.dst) + (8 * blk.nrows * len(ex.dst) if ex.with_perm else 0)
        per.append(b)
    return {"per_level": per, "total": int(sum(per)), "messages": int(sum(len(lv) for lv in plan))}


# --- device execution over torch.distributed ------------------------------------------


class _DevView:
    """__cuda_array_interface__ over engine-owned device memory (zero copy into torch)."""

    def __init__(self, addr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr, "data": (int(addr), False),
                                         "version": 3, "strides": None}


def _pool_index(pool, p):
    bid = -np.ones((p, p), np.int64)
    bid[pool.table[0], pool.table[1]] = np.arange(pool.nblocks)
    return bid


class DistEngine:
    """Owner-computes 2D block-cyclic factorization of one (grid, tree) over the
    ranks of a torch.distributed process group, one GPU per rank.

    Every rank plans only the tasks it owns (``task_owners``) on a replica of
    the block layout; the device graph is cut after every tree level at which
    this rank sends or receives finished blocks (``exchange_plan``), and the
    exchange between segments is one grouped point-to-point call
    (``batch_isend_irecv``: one NCCL group over NVLink on the "nccl" backend)
    ordered on the engine's stream.  Messages are the finished blocks' values
    in the working layout (identical on every rank) plus the local
    permutation for diagonal blocks; patterns never move.  The per-target
    update order is the serial one, so the factors are bitwise equal to a
    single-GPU run.  The "gloo" backend stages messages through host memory
    (multi-process tests on one GPU).
    """

    def __init__(self, grid, tree, *, pg: ProcGrid | None = None, group=None, device: int = 0,
                 dense: bool = False, dense_threshold=None, engine_kw: dict | None = None):
        import torch
        import torch.distributed as dist

        from .numeric import DEFAULT_DENSE_THRESHOLD, Engine

        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        self.pg = pg or ProcGrid.for_world(world)
        if self.pg.size != world:
            raise ValueError(f"process grid {self.pg.pr}x{self.pg.pc} != world size {world}")
        self.backend = dist.get_backend(group)
        self.device = device
        torch.cuda.set_device(device)
        own = task_owners(tree, self.pg)
        xplan = exchange_plan(tree, self.pg)
        cuts = np.zeros(max(tree.n_levels, 1), np.int8)
        for lv, exs in enumerate(xplan):
            if any(ex.src == self.rank or self.rank in ex.dst for ex in exs):
                cuts[lv] = 1
        dt = DEFAULT_DENSE_THRESHOLD if dense_threshold is None else dense_threshold
        self.eng = Engine(grid, tree, device=device, dense=dense, dense_threshold=dt,
                          mask=(own == self.rank).astype(np.int8), cuts=cuts, **(engine_kw or {}))
        self.grid, self.tree, self.dense = grid, tree, dense
        lay = self.eng.block_layout()
        vaddr, paddr, oaddr = self.eng.work_ptrs()
        self.vals = torch.as_tensor(_DevView(vaddr, self.eng.nnz_work, "<f8"), device=f"cuda:{device}")
        self.perm = (torch.as_tensor(_DevView(paddr, self.eng.n_diag_rows, "<i4"), device=f"cuda:{device}")
                     if self.eng.n_diag_rows else None)
        self.vout = torch.as_tensor(_DevView(oaddr, self.eng.nnz, "<f8"), device=f"cuda:{device}")
        self.stream = torch.cuda.ExternalStream(self.eng.stream_ptr, device=f"cuda:{device}")
        bid = _pool_index(self.eng.pool, grid.p)
        # per segment boundary (in cut order): the point-to-point ops, both sides
        # walking exchange_plan in the same order so every pair's sends and
        # receives match
        self.seg_ops = []
        for lv in np.flatnonzero(cuts):
            ops = []
            for ex in xplan[lv]:
                b = int(bid[ex.block])
                views = [self.vals[lay[0, b]:lay[0, b] + lay[1, b]]]
                if ex.with_perm and lay[2, b] >= 0:
                    nr = int(self.eng.pool.table[2, b])
                    views.append(self.perm[lay[2, b]:lay[2, b] + nr])
                if ex.src == self.rank:
                    ops.extend(("send", d, v) for d in ex.dst for v in views)
                elif self.rank in ex.dst:
                    ops.extend(("recv", ex.src, v) for v in views)
            self.seg_ops.append(ops)
        if len(self.seg_ops) != self.eng.n_segments - 1:
            raise RuntimeError("segment count does not match the cut levels")
        self.owned_block = np.array([self.pg.owner(int(bi), int(bj)) == self.rank
                                     for bi, bj in zip(self.eng.pool.table[0], self.eng.pool.table[1])], bool)
        self.messages = sum(len(o) for o in self.seg_ops)
        self.bytes_out = sum(v.numel() * v.element_size() for o in self.seg_ops for k, _, v in o if k == "send")
        # bring the communicator up on every rank before the first grouped P2P call
        self._allreduce(torch.zeros(1, dtype=torch.float64), "sum")

    # ---- collectives ---------------------------------------------------------------

    def _on_dev(self):
        return self.backend == "nccl"

    def _allreduce(self, t, op):
        dist, torch = self.dist, self.torch
        rop = {"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}[op]
        if self._on_dev():
            d = t.to(f"cuda:{self.device}")
            dist.all_reduce(d, op=rop, group=self.group)
            torch.cuda.synchronize(self.device)
            return d.cpu()
        dist.all_reduce(t, op=rop, group=self.group)
        return t

    def _exchange(self, ops):
        if not ops:
            return
        dist, torch = self.dist, self.torch
        if self._on_dev():
            with torch.cuda.stream(self.stream):
                p2p = [dist.P2POp(dist.isend if k == "send" else dist.irecv, v, peer, self.group)
                       for k, peer, v in ops]
                for r in dist.batch_isend_irecv(p2p):
                    r.wait()
            return
        # host-staged (gloo): the stream must have produced the sent blocks
        self.stream.synchronize()
        host = [v.cpu() if k == "send" else torch.empty(v.shape, dtype=v.dtype) for k, _, v in ops]
        p2p = [dist.P2POp(dist.isend if k == "send" else dist.irecv, h, peer, self.group)
               for (k, peer, _), h in zip(ops, host)]
        for r in dist.batch_isend_irecv(p2p):
            r.wait()
        with torch.cuda.stream(self.stream):
            for (k, _, v), h in zip(ops, host):
                if k == "recv":
                    v.copy_(h)

    # ---- execution -------------------------------------------------------------------

    def run(self, pivot_tol=1e-12, static_pivot=None):
        """One distributed factorization of the resident values.  Returns
        (device ms on this rank, lbk_status combined over ranks)."""
        ns = self.eng.n_segments
        for s in range(ns):
            self.eng.run_segment(s, pivot_tol, static_pivot)
            if s < ns - 1:
                self._exchange(self.seg_ops[s])
        ms, err = self.eng.finish_raw()
        enc = np.where(err == np.uint64(0xFFFFFFFFFFFFFFFF), np.iinfo(np.int64).max,
                       err.astype(np.int64)).astype(np.int64)
        red = self._allreduce(self.torch.from_numpy(enc.copy()), "min").numpy()
        comb = np.where(red == np.iinfo(np.int64).max, np.uint64(0xFFFFFFFFFFFFFFFF), red.astype(np.uint64))
        return ms, self.eng.status_from_err(comb)

    def upload(self, values=None):
        self.eng.upload(values)

    def run_host(self, a_values, out_values, out_perms, pivot_tol=1e-12, static_pivot=None):
        """End to end on this rank: host A values in (H2D), distributed
        factorization, this rank's factor values out (D2H, reference pool
        order; entries of blocks other ranks own are not final here)."""
        import ctypes as C

        from . import _native
        from .numeric import P, f64p, i32p

        self.eng.upload(a_values)
        _, st = self.run(pivot_tol, static_pivot)
        if st.code:
            return st
        st2 = _native.LbkStatus()
        self.eng.lib.lbk_download(self.eng.ctx, P(out_values, f64p),
                                  P(out_perms, i32p) if out_perms is not None else None, C.byref(st2))
        return st2

    def owned_entries(self) -> np.ndarray:
        """Mask over the reference pool order: entries of blocks this rank owns."""
        t = self.eng.pool.table
        return np.repeat(self.owned_block, t[4])

    def gather_values(self):
        """(factor values in reference pool order, perms per diagonal row) assembled
        from every rank's owned blocks (sum of disjointly masked arrays)."""
        vals, perms = self.eng.download()
        v = np.where(self.owned_entries(), vals, 0.0)
        t = self.eng.pool.table
        diag = t[0] == t[1]
        own_rows = np.repeat(self.owned_block[diag], t[2][diag])
        pv = np.where(own_rows, perms.astype(np.int64), 0)
        v = self._allreduce(self.torch.from_numpy(v), "sum").numpy()
        pv = self._allreduce(self.torch.from_numpy(pv), "sum").numpy().astype(np.int32)
        return v, pv

    def gather_work(self):
        """Dense-scratch values (every block a full tile, pool block order, the layout
        ``build_factors_full`` reads) assembled from every rank's owned blocks.  Each rank's
        working pool only holds its resident blocks (compacted offsets), so the owned tiles
        are first placed at their offsets in the common full-tile layout."""
        w = self.eng.download_work()
        lay = self.eng.block_layout()
        t = self.eng.pool.table
        size = t[2] * t[3]
        off = np.concatenate([[0], np.cumsum(size)])
        out = np.zeros(int(off[-1]), np.float64)
        for b in np.flatnonzero(self.owned_block):
            out[off[b]:off[b + 1]] = w[lay[0, b]:lay[0, b] + lay[1, b]]
        return self._allreduce(self.torch.from_numpy(out), "sum").numpy()

    def pool_entries(self) -> int:
        """Working-pool entries this rank allocates (owned blocks + received operands)."""
        return int(self.eng.nnz_work)

    def close(self):
        self.eng.close()


def factorize_distributed(grid, tree, pivot_tol: float = 1e-12, static_pivot: float | None = None, *,
                          pg: ProcGrid | None = None, group=None, device: int = 0, dense_threshold=None):
    """``factorize`` (factorize.py:245-384) over all ranks of the process group:
    2D block-cyclic owner-computes on one GPU per rank; every rank returns the
    same complete LUFactors.  A needed row swap re-runs in dense-scratch mode
    on every rank (the same fallback as the single-GPU path)."""
    from . import _native
    from .numeric import build_factors, build_factors_full

    for dense in (False, True):
        de = DistEngine(grid, tree, pg=pg, group=group, device=device, dense=dense, dense_threshold=dense_threshold)
        try:
            de.upload()
            _, st = de.run(pivot_tol, static_pivot)
            if st.code == _native.LBK_ERR_PIVOT_SWAP and not dense:
                continue
            _native.raise_status(st, "factorize_distributed")
            vals, perms = de.gather_values()
            if dense:
                return build_factors_full(grid, de.eng.pool, de.gather_work(), perms)
            return build_factors(grid, de.eng.pool, vals, perms)
        finally:
            de.close()
    raise RuntimeError("unreachable")  # pragma: no cover
