"""Median time of one real LU (frob_dgetrf) and one real inversion (frob_dinv) at size n.
Usage: python tools/time_lu.py N [reps]   (FROB_LU2_MAX=2048 routes n = 4096 to getrf)"""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2208_01239_b200 as fb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
g = torch.Generator().manual_seed(1)
a = (torch.randn(n, n, generator=g, dtype=torch.float64) + n ** 0.5 * torch.eye(n, dtype=torch.float64)).cuda()
x = torch.empty_like(a)
for name, fn in (("dgetrf", lambda: fb.dgetrf(a)), ("dinv", lambda: fb.dinv(a, out=x))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"n={n} {name} lu2_max={os.environ.get('FROB_LU2_MAX', 'default')}: {statistics.median(ts):.3f} ms")
