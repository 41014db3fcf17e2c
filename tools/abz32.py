"""A/B timing of the batched complex comparator at n = 32: python tools/abz32.py default|<lib.so>"""
import sys, torch
sys.path.insert(0, ".")
import paper_2208_01239_b200 as fb, synth
lib = sys.argv[1]
if lib != "default":
    fb.frobinv.load(lib)
z = torch.from_numpy(synth.batch(32, 16384, seed=0)).cuda().repeat(4, 1, 1).contiguous()
for _ in range(2): fb.zinv_batched(z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): fb.zinv_batched(z)
e1.record(); torch.cuda.synchronize()
print(lib, "%.3f ms" % (e0.elapsed_time(e1) / 10))
