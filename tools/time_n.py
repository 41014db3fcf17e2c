"""Median time of frob_inv / NEXT-1 / zinv at size n (no profiler, CUDA events). Usage: python tools/time_n.py N [frob|fused|zinv] [reps] [--lib PATH]"""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2208_01239_b200 as fb
if "--lib" in sys.argv:
    i = sys.argv.index("--lib")
    from paper_2208_01239_b200 import frobinv as fbi
    fbi.load(sys.argv[i + 1])
    del sys.argv[i:i + 2]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
which = sys.argv[2] if len(sys.argv) > 2 else "frob"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else (10 if n <= 8192 else 3)
z = torch.from_numpy(synth.config2(n)).cuda()
x = torch.empty_like(z)
fn = {"frob": lambda: fb.inv(z, out=x), "fused": lambda: fb.inv(z, out=x, fused=True),
      "zinv": lambda: fb.zinv(z, out=x)}[which]
for _ in range(3):
    fn()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"n={n} {which} {os.environ.get('FROB_LU2_LOOKAHEAD', 'default')}: {statistics.median(ts):.3f} ms")
