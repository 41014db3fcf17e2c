"""One frob_dgetrf at n after warm-up (for ncu): python tools/getrf_one.py N"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2208_01239_b200 as fb  # noqa: E402
import synth  # noqa: E402
n = int(sys.argv[1])
a = torch.from_numpy(synth.config2(n, seed=0).real.copy()).cuda()
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    fb.dgetrf(a)
torch.cuda.synchronize()
