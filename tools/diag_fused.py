import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, synth, paper_2208_01239_b200 as fb
for n in (2048, 4096, 16384):
    z = torch.from_numpy(synth.config2(n, seed=0)).cuda()
    for fused in (False, True):
        x, info = fb.inv(z, fused=fused, info=True)
        print(n, "fused" if fused else "literal", {k: info[k] for k in ("branch_used", "kappa_a", "kappa_b", "rho_a")}, flush=True)
