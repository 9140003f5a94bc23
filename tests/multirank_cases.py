"""Workloads of the multi-rank tests (tests/test_gpu_multirank.py): scaled
BASELINE configs covering every shard route of the library -- dense row
shards (Gaussian sketch in Gram-matrix mode with intervals split over ranks,
the same in pass mode, SRHT with zero-padded local rows, SJLT), CSR row
shards (CountSketch, Woodbury preconditioner, sparse Gram passes) and dense
column shards of the dual route (matrix right-hand side).

Each case is (name, workload, route, options); shard(n, world, rank) gives a
rank's [start, stop) the way bench.py and the reference's own interval split
do (contiguous blocks, sizes differing by at most one).
"""
import numpy as np

import workloads


def shard(n, world, rank):
    return (rank * n) // world, ((rank + 1) * n) // world


def cases():
    out = []
    w = workloads.c1(scale=0.25)
    w.T = 30
    out.append(("c1_gauss_matrix", w, "rows", {}))
    out.append(("c1_gauss_pass", w, "rows", {"gram_mode": 0}))
    w = workloads.c2(scale=1 / 64)
    w.T = 40
    out.append(("c2_srht", w, "rows", {}))
    w = workloads.c1(scale=0.25)
    w.T = 20
    w.sketch = dict(kind="sjlt", m=128, n=w.meta["n"], s=4, seed=3)
    out.append(("c1_sjlt", w, "rows", {}))
    w = workloads.c4(scale=1 / 1024)
    w.T = 40
    out.append(("c4_csr_countsketch_woodbury", w, "rows", {}))
    w = workloads.c5(scale=1 / 64, K=2)
    w.T = 20
    out.append(("c5_dual_cols", w, "cols", {}))
    return out


def csr_rows(a, r0, r1):
    """Rows [r0, r1) of a workloads CSR dict, offsets rebased to 0."""
    off = a["offsets"]
    lo, hi = off[r0], off[r1]
    return (r1 - r0, a["cols"], off[r0:r1 + 1] - lo, a["indices"][lo:hi], a["values"][lo:hi])


def grid(w, log_grid):
    return w.lambdas(log_grid)


def b_matrix(w):
    return np.asfortranarray(np.asarray(w.b).reshape(w.b.shape[0], -1))
