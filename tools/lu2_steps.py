"""Per-step period of one lu2 factorisation from a -DFROB_TL build (tools/build_tl.sh):
  python tools/lu2_steps.py LIB N [frob|zinv] [call]
For each step k: panel start-to-start period, panel / NEXT / BULK durations, and which of
them ends last before the next panel starts (the step's bound)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2208_01239_b200 import frobinv as fbi
L = fbi.load(sys.argv[1])
import paper_2208_01239_b200 as fb
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
which = sys.argv[3] if len(sys.argv) > 3 else "frob"
call = int(sys.argv[4]) if len(sys.argv) > 4 else 0
z = torch.from_numpy(synth.config2(n)).cuda()
fn = (lambda: fb.inv(z)) if which == "frob" else (lambda: fb.zinv(z))
for _ in range(3):
    fn()
torch.cuda.synchronize()
L.frob_tl_reset()
fn()
torch.cuda.synchronize()
S = (ctypes.c_ulonglong * (5 * 1024))()
E = (ctypes.c_ulonglong * (5 * 1024))()
L.frob_tl_read(S, E)
steps = {}
for kind, nm in enumerate(["P", "P", "NX", "BK"]):
    for k in range(call * 128, call * 128 + 128):
        s, e = S[kind * 1024 + k], E[kind * 1024 + k]
        if e and s != (1 << 64) - 1:
            steps.setdefault(k - call * 128, {})[nm] = (s, e)
ks = sorted(steps)
t0 = min(v[0] for d in steps.values() for v in d.values())
tend = max(v[1] for d in steps.values() for v in d.values())
print(f"n={n} {which} call {call}: {len(ks)} steps, span {(tend - t0) / 1e3:.1f} us")
print(" k   period   panel    next    bulk   bulk_end-next_panel_start  bound")
agg = {}
for i, k in enumerate(ks):
    d = steps[k]
    ps = d["P"][0]
    nxt = steps[ks[i + 1]]["P"][0] if i + 1 < len(ks) else tend
    per = (nxt - ps) / 1e3
    pd = (d["P"][1] - d["P"][0]) / 1e3
    nx = (d["NX"][1] - d["NX"][0]) / 1e3 if "NX" in d else 0
    bk = (d["BK"][1] - d["BK"][0]) / 1e3 if "BK" in d else 0
    slack = (nxt - d["BK"][1]) / 1e3 if "BK" in d else float("nan")
    print(f"{k:3d} {per:7.1f} {pd:7.1f} {nx:7.1f} {bk:7.1f} {slack:9.1f}")
    band = k // 16
    a = agg.setdefault(band, [0, 0, 0, 0, 0])
    a[0] += per; a[1] += pd; a[2] += nx; a[3] += bk; a[4] += 1
print("band(16 steps)  avg period  panel  next  bulk")
for b, a in sorted(agg.items()):
    c = a[4]
    print(f"{b:2d}  {a[0] / c:7.1f} {a[1] / c:7.1f} {a[2] / c:7.1f} {a[3] / c:7.1f}")
