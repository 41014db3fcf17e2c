"""Per-kernel (and per GEMM role) time of one frob_inv / zinv at size n, from the library's
CUDA-event profiler.  Usage: python tools/profile_n.py N [frob|zinv] [reps] [--lib PATH]"""
import sys, os, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2208_01239_b200 as fb
from paper_2208_01239_b200 import frobinv as fbi
if "--lib" in sys.argv:
    i = sys.argv.index("--lib")
    fbi.load(sys.argv[i + 1])
    del sys.argv[i:i + 2]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
which = sys.argv[2] if len(sys.argv) > 2 else "frob"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
z = torch.from_numpy(synth.config2(n)).cuda()
x = torch.empty_like(z)
fn = (lambda: fb.inv(z, out=x)) if which == "frob" else (lambda: fb.zinv(z, out=x))
for _ in range(2):
    fn()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = statistics.median(ts)
fbi.profile_enable(True)
for _ in range(reps):
    fn()
torch.cuda.synchronize()
prof = fbi.profile_read()
fbi.profile_enable(False)
alg = (10.0 if which == "frob" else 8.0) * n ** 3
print(f"n={n} {which}: {t:.3f} ms, {alg / t / 1e9:.2f} TF/s algorithmic")
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"]):
    ms = v["total_ms"] / reps
    tf = v["flops"] / (v["total_ms"] * 1e-3) / 1e12 if v["total_ms"] else 0
    print(f"  {k:28s} {v['launches'] / reps:7.1f} launches  {ms:9.3f} ms  {100 * ms / t:5.1f}%  {tf:6.2f} TF/s  "
          f"{v['flops'] / reps / 1e9:9.2f} GFLOP")
