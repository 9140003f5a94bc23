"""One sparse Gram product (C4 CSR, 128 right-hand columns) for ncu captures of
the panel passes (sparse_gram.cu).

    python tools/sparse_ncu.py [row_scale] [cols]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    cols = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    w = workloads.c4()
    n = int(w.meta["n"] * scale)
    off = w.a["offsets"][: n + 1]
    nnz = int(off[-1])
    d = w.meta["d"]
    ctx = rp.Context(0)
    ctx.set_operator(rp.Csr(n, d, off, w.a["indices"][:nnz], w.a["values"][:nnz]))
    x = torch.randn(d * cols, dtype=torch.float64, device="cuda")
    y = torch.empty(d * cols, dtype=torch.float64, device="cuda")
    for _ in range(2):
        rp.gram_apply_raw(ctx, x.data_ptr(), cols, y.data_ptr())
    torch.cuda.synchronize()
    print("ok", float(y.norm()))


if __name__ == "__main__":
    main()
