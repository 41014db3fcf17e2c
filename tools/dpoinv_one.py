"""One frob_dpoinv / frob_hpd_inv / zhpd_inv_chol at n after warm-up (ncu launch lists): python tools/dpoinv_one.py N [which]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2208_01239_b200 as fb  # noqa: E402
import synth  # noqa: E402
n = int(sys.argv[1])
which = sys.argv[2] if len(sys.argv) > 2 else "dpoinv"
z = torch.from_numpy(synth.hpd(n, seed=1)).cuda()
a = z.real.contiguous()
f = {"dpoinv": lambda: fb.dpoinv(a, check=False), "alg6": lambda: fb.hpd_inv(z, check=False),
     "alg8": lambda: fb.zhpd_inv(z, check=False)}[which]
for _ in range(2):
    f()
torch.cuda.synchronize()
f()
torch.cuda.synchronize()
