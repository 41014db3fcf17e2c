"""NEXT-1 vs literal Frobenius vs complex LU at n for an A/B library: python tools/time_fused.py [--lib PATH] N..."""
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2208_01239_b200 as fb  # noqa: E402
from paper_2208_01239_b200 import frobinv as fbi  # noqa: E402
import synth  # noqa: E402
args = sys.argv[1:]
lib = "default"
if args and args[0] == "--lib":
    lib = args[1]
    fbi.load(lib)
    args = args[2:]
for n in [int(v) for v in args]:
    z = torch.from_numpy(synth.config2(n, seed=0)).cuda()
    x = torch.empty_like(z)
    res = {}
    for name, f in (("literal", lambda: fb.inv(z, out=x)), ("fused", lambda: fb.inv(z, out=x, fused=True))):
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5 if n <= 8192 else 3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name] = statistics.median(ts)
    print(f"{os.path.basename(lib)} n={n}: literal {res['literal']:.2f} ms  fused {res['fused']:.2f} ms "
          f"({26 / 3 * n ** 3 / res['fused'] / 1e9:.1f} TF/s alg)", flush=True)
