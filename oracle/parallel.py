"""Multi-core execution of the oracle's float64 SpMM — TEST INFRASTRUCTURE
ONLY (see oracle/__init__.py).  Lets the full-size (Reddit / products shape)
parity tests and bench.py's CPU baseline run the oracle on every host core.

numpy's gather + add.reduceat hold the GIL for most of their time (a thread
pool measured no faster than one thread), so the workers are fork()ed
processes.  They inherit the registered operands (offsets / cols arrays) at
fork time; the dense [V, w] input and the output travel through anonymous
shared memory (multiprocessing.RawArray, no /dev/shm file).  Each call splits
the rows into one piece of equal edge count per worker; every row is summed
by exactly the serial code (oracle.ops._spmm_serial), so results are
bit-identical to the one-process oracle.

Use:

    pool = ForkSpmmPool({"csr": (off, cols), "csc": (t_off, t_cols)}, V, width)
    with oracle.ops.parallel(pool):
        ref = oracle.ops.gcn2_step(off, cols, t_off, t_cols, ...)   # SpMMs on the pool
    pool.close()

Inside ``parallel(pool)`` every ``oracle.ops.spmm`` call whose (offsets, cols)
are a registered operand (by identity), without edge values, and whose X has
at most ``width`` columns runs on the pool; anything else runs serially.
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

_STATE: dict = {}


def _worker(job):
    from . import ops as oo

    name, a, b, w, norm = job
    st = _STATE
    off, cols = st["ops"][name]
    V = st["V"]
    X = np.frombuffer(st["X"], dtype=np.float64, count=V * w).reshape(V, w)
    R = off.size - 1
    Y = np.frombuffer(st["Y"], dtype=np.float64, count=R * w).reshape(R, w)
    e0 = int(off[a])
    Y[a:b] = oo._spmm_serial(off[a:b + 1] - e0, cols[e0:int(off[b])], X, norm=norm)
    return b - a


class ForkSpmmPool:
    """fork()ed worker pool for ``oracle.ops.spmm`` over registered operands."""

    def __init__(self, operands: dict, V: int, width: int, workers: int | None = None):
        self.V, self.width = int(V), int(width)
        self.workers = workers or len(os.sched_getaffinity(0))
        rows = max([np.asarray(o).size - 1 for o, _ in operands.values()] + [self.V])
        self.X = mp.RawArray("d", self.V * self.width)
        self.Y = mp.RawArray("d", rows * self.width)
        self.ops = {k: (np.asarray(o, dtype=np.int64), c) for k, (o, c) in operands.items()}
        self._ident = {(id(o), id(c)): k for k, (o, c) in operands.items()}
        self._keep = operands  # the identities above stay valid while the pool lives
        _STATE.update(ops=self.ops, V=self.V, X=self.X, Y=self.Y)
        self.pool = mp.get_context("fork").Pool(self.workers)

    def spmm(self, name, X, norm=False, r0=0, r1=None):
        """Rows [r0, r1) of A_name X (float64; X is [V, w], w <= width)."""
        off, _ = self.ops[name]
        X = np.asarray(X, dtype=np.float64)
        w = X.shape[1]
        assert X.shape[0] == self.V and w <= self.width, (X.shape, self.V, self.width)
        r1 = off.size - 1 if r1 is None else r1
        np.frombuffer(self.X, dtype=np.float64, count=self.V * w).reshape(self.V, w)[:] = X
        cuts = np.searchsorted(off, np.linspace(off[r0], off[r1], self.workers + 1)).clip(r0, r1)
        cuts[0], cuts[-1] = r0, r1
        jobs = [(name, int(a), int(b), w, norm) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
        self.pool.map(_worker, jobs)
        R = off.size - 1
        Y = np.frombuffer(self.Y, dtype=np.float64, count=R * w).reshape(R, w)
        return Y[r0:r1].copy()

    def lookup(self, offsets, cols, X):
        """Operand name for an oracle.ops.spmm call the pool can take, else None."""
        name = self._ident.get((id(offsets), id(cols)))
        if name is None or np.ndim(X) != 2:
            return None
        if np.shape(X)[0] != self.V or np.shape(X)[1] > self.width:
            return None
        return name

    def close(self):
        self.pool.close()
        self.pool.join()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
