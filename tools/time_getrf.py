"""Median times of frob_dgetrf / frob_dinv / frob_inv at the given n for A/B variants of the library.
  python tools/time_getrf.py [--lib PATH] N..."""
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


def med(f, reps):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for n in [int(v) for v in args]:
    z = torch.from_numpy(synth.config2(n, seed=0)).cuda()
    a = z.real.contiguous()
    reps = 5 if n <= 8192 else 3
    t_lu = med(lambda: fb.dgetrf(a), reps)
    t_inv = med(lambda: fb.dinv(a), reps)
    t_frob = med(lambda: fb.inv(z), reps)
    print(f"{os.path.basename(lib)} n={n}: getrf {t_lu:.2f} ms ({2/3*n**3/t_lu/1e9:.1f} TF/s)  dinv {t_inv:.2f} ms  "
          f"frob {t_frob:.2f} ms ({10*n**3/t_frob/1e9:.1f} TF/s)", flush=True)
