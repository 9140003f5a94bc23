"""The composition GEMM of one profiled path step (bench.py --dump-gemm + RP_GEMM_LOG): shape, device
time, TFLOP/s.  It is the last product with k = kmax that is batched over the intervals."""
import json
import sys

prof = json.load(open(sys.argv[1]))
log = [ln.split() for ln in open(sys.argv[2]) if ln.strip()][-len(prof["seconds"]):]
for sec, fl, by, g in list(zip(prof["seconds"], prof["flops"], prof["bytes"], log))[-4:]:
    print(f"m {g[0]} n {g[1]} k {g[2]} batch {g[4]} tile {g[8]}: {sec*1e6:.1f} us, {fl/sec/1e12:.2f} TFLOP/s, "
          f"{by/sec/1e9:.0f} GB/s of operand bytes")
