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
