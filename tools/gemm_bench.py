"""GEMM engine throughput (frob_dgemm) vs cuBLAS DGEMM (torch.matmul, context only)."""
import json
import sys
import torch
sys.path.insert(0, ".")
import paper_2208_01239_b200 as fb
from paper_2208_01239_b200 import frobinv as fbi

# --lib PATH: an A/B variant of the library (tools/build_variant.sh)
args = sys.argv[1:]
if args and args[0] == "--lib":
    fbi.load(args[1])
    args = args[2:]
sys.argv = [sys.argv[0]] + args

for n in ([int(v) for v in sys.argv[1:]] or [1024, 2048, 4096, 8192]):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    res = {"n": n}
    for name, fn in (("frob_dgemm", lambda: fb.dgemm(a, b, c)), ("cublas", lambda: torch.matmul(a, b, out=c))):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10 if n <= 4096 else 3
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[name + "_tflops"] = 2 * n ** 3 / ms / 1e9
    ref = torch.matmul(a, b)
    fb.dgemm(a, b, c)
    res["max_abs_diff"] = float((c - ref).abs().max())
    print(json.dumps(res))
