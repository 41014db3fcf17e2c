"""Run one batched launch (for ncu): python tools/batched_run.py N COUNT [zinv]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2208_01239_b200 as fb
n, cnt = int(sys.argv[1]), int(sys.argv[2])
z = torch.from_numpy(synth.batch(n, cnt, seed=0)).cuda()
f = fb.zinv_batched if len(sys.argv) > 3 else fb.inv_batched
for _ in range(2):
    f(z)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); f(z); e.record(); torch.cuda.synchronize()
print(f"n={n} count={cnt}: {s.elapsed_time(e):.3f} ms -> {cnt / s.elapsed_time(e) * 1e3:.0f} inverses/s")
