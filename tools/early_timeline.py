"""Event timeline of one frob_inv call's LU / inverse stages from a -DFROB_TL build
(tools/build_tl.sh): python tools/early_timeline.py LIB N
Labels: lu2 start/end (34/35), EarlyInv fork (36), aux start / assembled / U11,L11 inverted / V done
(30-33), inverse: wait (20), tri U22 start / done (21/22), top level done (23), product done (24);
20.1 / 23.1: the plain tri_inverses path."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2208_01239_b200 as fb  # noqa: E402
from paper_2208_01239_b200 import frobinv as fbi  # noqa: E402
L = fbi.load(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
z = torch.from_numpy(synth.config2(n)).cuda()
for _ in range(2):
    fb.inv(z)
torch.cuda.synchronize()
L.frob_evtrace_reset()
fb.inv(z)
torch.cuda.synchronize()
cap = 4096
codes = (ctypes.c_int * cap)()
ms = (ctypes.c_float * cap)()
cnt = L.frob_evtrace_read(codes, ms, cap)
names = {34: "lu2 start", 35: "lu2 end", 36: "early fork (chain at step h)", 30: "aux start", 31: "aux assembled",
         32: "aux U11/L11 inverted", 33: "aux V done", 20: "inv: wait early", 21: "inv: early joined",
         22: "inv: U22/L22 inverted", 23: "inv: top level done", 24: "inv: product done"}
ev = sorted((ms[i], codes[i]) for i in range(cnt))
for t, c in ev:
    k, sub = c // 100000, c % 100000
    print(f"{t:9.3f} ms  {names.get(k, str(k))}{'' if sub == 0 else ' (' + str(sub) + ')'}")
