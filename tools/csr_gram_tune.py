"""Sweep the sparse Gram blocking (csr_panel_rows x csr_chunk) on the C4 CSR.

    python tools/csr_gram_tune.py [row_scale] [cols]

Times rp_gram_apply (device events, profile option) for a cols-wide W and
reports the effective gather rate 2 * nnz * 8 * cols / t.
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    cols = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    w = workloads.c4()
    n = int(w.meta["n"] * scale)
    off = w.a["offsets"][: n + 1]
    nnz = int(off[-1])
    d = w.meta["d"]
    a = rp.Csr(n, d, off, w.a["indices"][:nnz], w.a["values"][:nnz])
    ctx = rp.Context(0)
    ctx.set_operator(a)
    x = torch.randn(d * cols, dtype=torch.float64, device="cuda")
    y = torch.empty(d * cols, dtype=torch.float64, device="cuda")
    ref = None
    combos = [(p, c, l2) for p in (32768, 65536, 131072) for c in (64, 128) for l2 in (0, 1)]
    if os.environ.get("CSR_COMBOS"):
        combos = [tuple(int(v) for v in c.split(":")) for c in os.environ["CSR_COMBOS"].split(",")]
    for panel, chunk, l2 in combos:
        ctx.set_option("csr_panel_rows", panel)
        ctx.set_option("csr_chunk", chunk)
        ctx.set_option("csr_l2_persist", l2)
        rp.gram_apply_raw(ctx, x.data_ptr(), cols, y.data_ptr())
        if ref is None:
            ref = y.clone()
        assert torch.equal(ref, y), "blocking changed the bits"
        ctx.set_option("profile", 1)
        ts = []
        for _ in range(3):
            rp.gram_apply_raw(ctx, x.data_ptr(), cols, y.data_ptr())
            ts.append(rp.last_device_seconds(ctx))
        ctx.set_option("profile", 0)
        t = statistics.median(ts)
        print(f"panel {panel:7d} chunk {chunk:3d} l2persist {l2}: {t*1e3:8.2f} ms  {t/cols*1e6:7.2f} us/col  "
              f"gather {2*nnz*8*cols/t/1e12:6.2f} TB/s", flush=True)


if __name__ == "__main__":
    main()
