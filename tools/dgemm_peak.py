"""Measure cuBLAS DGEMM (torch.matmul float64) throughput: the FP64 roofline denominator."""
import torch, json, sys
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(5):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[n] = 2 * n**3 / best / 1e9
    print(f"cuBLAS DGEMM n={n}: {res[n]:.2f} TFLOP/s ({best:.2f} ms)")
