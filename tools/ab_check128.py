"""Bitwise fingerprint of the batched n = 128 (and n = 32) outputs for an A/B build:
   python tools/ab_check128.py LIB|default   (same digest across builds = same arithmetic)"""
import hashlib
import sys
import torch
sys.path.insert(0, ".")
import paper_2208_01239_b200 as fb
import synth

lib = sys.argv[1]
if lib != "default":
    fb.frobinv.load(lib)
h = hashlib.sha256()
for n, cnt in ((128, 4096), (100, 512), (32, 4096)):
    z = torch.from_numpy(synth.batch(n, cnt, seed=3)).cuda()
    for br in ("auto", "a", "b"):
        x, info, bu = fb.inv_batched(z, branch=br)
        torch.cuda.synchronize()
        h.update(x.cpu().numpy().tobytes()); h.update(info.cpu().numpy().tobytes())
print(lib, h.hexdigest()[:16])
