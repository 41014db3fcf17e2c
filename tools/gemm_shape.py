"""TF/s of one frob_dgemm shape (C = alpha A B + beta C): python tools/gemm_shape.py M N K [beta] [--lib PATH]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2208_01239_b200 as fb  # noqa: E402
from paper_2208_01239_b200 import frobinv as fbi  # noqa: E402
args = sys.argv[1:]
if "--lib" in args:
    i = args.index("--lib")
    fbi.load(args[i + 1])
    args = args[:i] + args[i + 2:]
m, n, k = (int(v) for v in args[:3])
beta = float(args[3]) if len(args) > 3 else 0.0
a = torch.randn(m, k, dtype=torch.float64, device="cuda")
b = torch.randn(k, n, dtype=torch.float64, device="cuda")
c = torch.randn(m, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    fb.dgemm(a, b, c, alpha=-1.0, beta=beta)
torch.cuda.synchronize()
reps = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    fb.dgemm(a, b, c, alpha=-1.0, beta=beta)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"M={m} N={n} K={k} beta={beta}: {ms:.3f} ms {2 * m * n * k / ms / 1e9:.2f} TF/s", flush=True)
