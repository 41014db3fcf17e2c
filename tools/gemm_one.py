"""One frob_dgemm at n (for ncu): python tools/gemm_one.py N"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2208_01239_b200 as fb
n = int(sys.argv[1])
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)
for _ in range(3):
    fb.dgemm(a, b, c)
torch.cuda.synchronize()
