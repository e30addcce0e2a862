"""Shared helpers for the parity tests (test infrastructure)."""
import threading

import numpy as np

import paper_1401_3733_b200 as lb

# (group_rank, rep) of the BASELINE configs: SU(3)F (1,3), SU(2)F (2), SU(2)A (4), SU(4)AS (5)
REPS = [(3, lb.FUNDAMENTAL), (2, lb.FUNDAMENTAL), (2, lb.ADJOINT), (4, lb.ANTISYMMETRIC)]
REP_IDS = ["su3f", "su2f", "su2a", "su4as"]


def rel_l2(a, b):
    d = np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel())
    n = np.linalg.norm(np.asarray(b).ravel())
    return d / n if n else d


def global_index(L, grid, rank):
    """Global lexicographic index of each local interior site of `rank`."""
    loc = [L[d] // grid[d] for d in range(4)]
    c = []
    r = rank
    for d in (3, 2, 1, 0):
        c.append(r % grid[d])
        r //= grid[d]
    coords = c[::-1]
    t, x, y, z = np.meshgrid(*[np.arange(loc[d]) + coords[d] * loc[d] for d in range(4)], indexing="ij")
    return (((t * L[1] + x) * L[2] + y) * L[3] + z).reshape(-1)


def run_ranks(nranks, body):
    """Run body(rank) on one host thread per rank (reference run_workers model)."""
    errs = [None] * nranks
    outs = [None] * nranks

    def run(r):
        try:
            outs[r] = body(r)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    ths = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return outs
