"""Does a CUDA graph (stream capture of the PDL-chained launches) shorten frob_inv at n = 1024?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2208_01239_b200 as fb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
z = torch.from_numpy(synth.config2(n)).cuda()
x = torch.empty_like(z)
def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for br in ("a", "auto"):
    print(br, "direct", round(timeit(lambda: fb.inv(z, branch=br, out=x)), 4), "ms")
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
fb.inv(z, branch="a", out=x)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    fb.inv(z, branch="a", out=x)
print("graph replay (branch a)", round(timeit(lambda: g.replay()), 4), "ms")
ref = fb.inv(z, branch="a")
g.replay(); torch.cuda.synchronize()
print("graph result == direct:", bool(torch.equal(ref, x)))
