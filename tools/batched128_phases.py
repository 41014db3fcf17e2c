"""Phase breakdown of frob_batched128_kernel from clock64 stamps (probe build: -DFROB_B128_TL).
   bash tools/build_variant.sh b128tl -DFROB_B128_TL && python tools/batched128_phases.py tools/ab/libfrobinv_b128tl.so"""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2208_01239_b200 as fb
import synth

lib = sys.argv[1]
fb.frobinv.load(lib)
L = ctypes.CDLL(lib)
z = torch.from_numpy(synth.batch(128, 2048, seed=0)).cuda().repeat(8, 1, 1).contiguous()
for _ in range(3):
    fb.inv_batched(z)
torch.cuda.synchronize()
h = np.zeros((16, 8), dtype=np.int64)
assert L.frob_b128_tl_read(h.ctypes.data_as(ctypes.c_void_p)) == 0
names = ["load + sweep A", "auto/branch", "a3 C=X^-1 Y", "a4 M=X+YC", "a5 sweep M", "a6 Im=-C Re"]
order = [0, 1, 2, 3, 4, 5, 6]
d = np.diff(h[:, order], axis=1)
tot = h[:, 6] - h[:, 0]
for i, nm in enumerate(names):
    print(f"{nm:14s} {np.median(d[:, i]):10.0f} cycles  ({np.median(d[:, i]) / np.median(tot) * 100:5.1f}%)")
t = np.zeros((16, 6), dtype=np.int64)
if L.frob_g8_tl_read(t.ctypes.data_as(ctypes.c_void_p)) == 0:
    print("block 0, last sweep, per panel (cycles): PW factor | factor end -> w0 past FACT | FACT -> U | U -> U2 (W/V) | U2 -> next PW factor start | w0 FACT -> w4 tri-inverses done")
    for b in range(15):
        print(b, t[b, 1] - t[b, 0], t[b, 2] - t[b, 1], t[b, 3] - t[b, 2], t[b, 4] - t[b, 3], t[b + 1, 0] - t[b, 4], t[b, 5] - t[b, 2])
print(f"{'total':14s} {np.median(tot):10.0f} cycles per matrix")
