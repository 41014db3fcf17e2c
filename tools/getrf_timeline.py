"""Chain vs far-column timeline of the blocked LU (getrf) from a -DFROB_TL build (tools/build_tl.sh):
  python tools/getrf_timeline.py LIB N
Events (ms from the first): 0 block start (chain stream), 1 inner steps done, 2 L11^-1 done,
10 / 11 far TRMM / GEMM done,
3 far update starts (aux stream), 4 far update done, 5 look-ahead starts (after far(t-1)),
6 look-ahead done, 7 blocked part done, 8 lu2 tail done, 9 end."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2208_01239_b200 as fb  # noqa: E402
from paper_2208_01239_b200 import frobinv as fbi  # noqa: E402
L = fbi.load(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
a = torch.from_numpy(synth.config2(n, seed=0)).cuda().real.contiguous()
for _ in range(2):
    fb.dgetrf(a)
torch.cuda.synchronize()
L.frob_evtrace_reset()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
fb.dgetrf(a)
e1.record()
torch.cuda.synchronize()
cap = 100000
codes = (ctypes.c_int * cap)()
ms = (ctypes.c_float * cap)()
cnt = L.frob_evtrace_read(codes, ms, cap)
ev = {}
for i in range(cnt):
    ev[(codes[i] // 100000, codes[i] % 100000)] = ms[i]
blocks = sorted({t for (k, t) in ev if k == 0})
print(f"n={n}: dgetrf {e0.elapsed_time(e1):.2f} ms (events span {max(ev.values()):.2f} ms)")
print("  t   start   inner   Linv  far_start far_dur  la_wait  la_dur  period | far: swap+trmm  gemm   copy  gemm_TF/s")
rows = []
for i, t in enumerate(blocks):
    g = lambda k: ev.get((k, t), float("nan"))  # noqa: E731
    nxt = ev.get((0, blocks[i + 1])) if i + 1 < len(blocks) else ev.get((7, 0))
    r = (t, g(0), g(1) - g(0), g(2) - g(1), g(3), g(4) - g(3), g(5) - g(2), g(6) - g(5), (nxt or float("nan")) - g(0))
    rows.append(r)
    K0 = t * 256
    m = n - K0 - 256
    fl = 2.0 * m * max(0, n - K0 - 512) * 256
    g10, g11 = ev.get((10, t), float("nan")), ev.get((11, t), float("nan"))
    gm = g11 - g10
    print("%3d %7.3f %7.3f %6.3f %8.3f %7.3f %8.3f %7.3f %7.3f" % r +
          " | %8.3f %7.3f %6.3f %6.1f" % (g10 - g(3), gm, g(4) - g11, fl / gm / 1e9 if gm == gm and gm > 0 else 0))
if (7, 0) in ev:
    print(f"blocked part ends {ev[(7, 0)]:.3f}; lu2 tail {ev.get((8, 0), float('nan')) - ev[(7, 0)]:.3f} ms; "
          f"end {ev.get((9, 0), float('nan')):.3f}")
tot = lambda j: sum(r[j] for r in rows if r[j] == r[j])  # noqa: E731
print(f"sums: inner {tot(2):.2f}  Linv {tot(3):.2f}  far {tot(5):.2f}  la_wait {tot(6):.2f}  la {tot(7):.2f}  "
      f"periods {tot(8):.2f} ms")
