"""One rank of the multi-rank tests (tests/test_gpu_multirank.py).

Every rank holds its shard of each case's operator (rows, or columns for the
dual route) in its own library context and runs the product's path with a
host-side communicator over torch.distributed (gloo): the library's own shard
arithmetic (MT stream offsets r*n + row0, local CountSketch / SRHT rows, the
dual's column block), its all-reduces, interval split and divergence
agreement all run for real.  The ranks share one GPU, so they pass a
cross-process token (an flock) around: a rank holds it while it has device
work in flight and gives it up inside each collective (the library has
synchronized its stream before calling the callback).  Kernels of different
ranks therefore never run at the same time -- the GPU never time-slices a
TMA pipeline between contexts (profiles/r02_concurrency_root_cause.txt) and
no kernel waits on another rank.

    python tests/multirank_worker.py OUT_DIR LOCK_FILE   (env: RANK, WORLD_SIZE, MASTER_ADDR, MASTER_PORT)
"""
import fcntl
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import multirank_cases as mc  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


class Token:
    def __init__(self, path):
        self.fd = os.open(path, os.O_CREAT | os.O_RDWR, 0o644)

    def acquire(self):
        fcntl.flock(self.fd, fcntl.LOCK_EX)

    def release(self):
        fcntl.flock(self.fd, fcntl.LOCK_UN)


def main():
    out_dir, lock = sys.argv[1], sys.argv[2]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tok = Token(lock)
    stats = {"allreduce": 0, "allgather": 0}

    def allreduce(buf):
        stats["allreduce"] += 1
        tok.release()
        try:
            dist.all_reduce(torch.from_numpy(buf))
        finally:
            tok.acquire()

    def allgather(send, recv):
        stats["allgather"] += 1
        tok.release()
        try:
            outs = [torch.from_numpy(recv[r]) for r in range(world)]
            dist.all_gather(outs, torch.from_numpy(send.copy()))
        finally:
            tok.acquire()

    results = {}
    for name, w, route, opts in mc.cases():
        ctx = rp.Context(0)
        rp.comm_init_host(ctx, rank, world, allreduce, allgather)
        for k, v in opts.items():
            ctx.set_option(k, v)
        b = mc.b_matrix(w)
        K = b.shape[1]
        lam = mc.grid(w, rp.log_grid)
        T = len(lam)
        cfg = rp.PathConfig(w.lambda_min, w.lambda_max, lam, w.epsilon)
        sk = w.sketch
        spec = rp.SketchSpec(sk["kind"], sk["m"], sk["n"], sk["s"], sk["seed"])
        rho = rp.RhoBounds.manual(*w.rho)
        before = dict(stats)
        tok.acquire()
        try:
            if route == "rows":
                n = b.shape[0]
                r0, r1 = mc.shard(n, world, rank)
                if isinstance(w.a, dict):
                    rows, cols, off, idx, val = mc.csr_rows(w.a, r0, r1)
                    rp.set_csr_rows(ctx, n, r0, rp.Csr(rows, cols, off, idx, val))
                    d = cols
                else:
                    a_loc = np.asfortranarray(w.a[r0:r1])
                    d = a_loc.shape[1]
                    rp.set_dense_rows_host(ctx, n, r0, r1 - r0, d, a_loc.ctypes.data, max(r1 - r0, 1))
                b_loc = np.asfortranarray(b[r0:r1])
                x = np.empty(d * K * T)
                tm = rp.path_raw(ctx, b_loc.ctypes.data, K, cfg, spec, rho, x.ctypes.data, rp.RP_HOST)
                # train losses of every point, partial squared norms all-reduced over the row shards
                loss = np.empty(T)
                ctx.check(rp.lib().rp_losses(ctx.handle, rp._ptr(np.asfortranarray(b_loc).reshape(-1, order="F").copy()),
                                             K, T, rp._ptr(x), rp._ptr(np.asarray(lam, dtype=np.float64)),
                                             rp._ptr(loss), rp.RP_HOST))
                results[name + ":x"] = x
                results[name + ":loss"] = loss
                results[name + ":split"] = np.array([r0, r1])
            else:
                n, dg = w.a.shape
                c0, c1 = mc.shard(dg, world, rank)
                a_loc = np.asfortranarray(w.a[:, c0:c1])
                rp.set_dense_cols_host(ctx, n, dg, c0, c1 - c0, a_loc.ctypes.data, n)
                x = np.empty((c1 - c0) * K * T)
                tm = rp.path_raw(ctx, b.ctypes.data, K, cfg, spec, rho, x.ctypes.data, rp.RP_HOST, dual=True)
                results[name + ":x"] = x
                results[name + ":split"] = np.array([c0, c1])
            results[name + ":gram_mode"] = np.array([tm.gram_mode])
        finally:
            tok.release()
        results[name + ":collectives"] = np.array([stats["allreduce"] - before["allreduce"],
                                                   stats["allgather"] - before["allgather"]])
        del ctx
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **results)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
