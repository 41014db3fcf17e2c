"""Context only: cuBLAS DGEMM (torch.matmul float64) throughput on this GPU."""
import json
import torch

for n in (1024, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10 if n < 8192 else 5
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"kind": "cublas_dgemm", "n": n, "ms": ms, "tflops": 2 * n ** 3 / ms / 1e9}))
