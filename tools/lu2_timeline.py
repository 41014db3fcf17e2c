"""Per-step kernel timeline of one lu2 factorisation (the last LU of one frob_inv / zinv call),
from a -DFROB_TL build of the library (tools/build_tl.sh):  python tools/lu2_timeline.py LIB N [frob|zinv]
Kinds: P = panel (one CTA), PC = panel (cluster), NX = NEXT update, BK = BULK update."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2208_01239_b200 import frobinv as fbi
L = fbi.load(sys.argv[1])
import paper_2208_01239_b200 as fb
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
which = sys.argv[3] if len(sys.argv) > 3 else "frob"
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
names = ["P", "PC", "NX", "BK", "-"]
ev = []
call = int(sys.argv[5]) if len(sys.argv) > 5 else 0  # which LU of the call (frob: 0 = LU(A), 1 = LU(M))
for kind in range(4):
    for k in range(call * 128, call * 128 + 128):
        s, e = S[kind * 1024 + k], E[kind * 1024 + k]
        if e and s != (1 << 64) - 1:
            ev.append((s, e, names[kind], k - call * 128))
ev.sort()
t0 = ev[0][0]
last_end = {}
tot = {}
for s, e, nm, k in ev:
    tot[nm] = tot.get(nm, 0) + (e - s)
print(f"n={n} {which}: {len(ev)} kernel-steps, span {(max(e for _, e, _, _ in ev) - t0) / 1e3:.1f} us")
for nm, v in tot.items():
    print(f"  {nm:3s} busy {v / 1e3:9.1f} us")
print("step  kind   start(us)  dur(us)  gap-from-prev-end(us)")
prev_end = t0
for s, e, nm, k in ev[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{k:4d}  {nm:3s} {(s - t0) / 1e3:10.1f} {(e - s) / 1e3:8.1f} {(s - prev_end) / 1e3:8.1f}")
    prev_end = max(prev_end, e)
if hasattr(L, "frob_nx_read"):
    T = (ctypes.c_longlong * 16)()
    L.frob_nx_read(T)
    for b in range(2):
        t = T[b * 8:(b + 1) * 8]
        print(f"NEXT step k0=320 CTA y={b}: loads+mv {t[1] - t[0]}  X/remap {t[2] - t[1]}  solve {t[3] - t[2]}  mma+store {t[5] - t[3]}  total {t[5] - t[0]} cycles")
