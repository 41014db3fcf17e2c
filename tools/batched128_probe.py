import sys, torch
sys.path.insert(0, ".")
import paper_2208_01239_b200 as fb, synth
z = torch.from_numpy(synth.batch(128, 592, seed=0)).cuda()
for _ in range(2):
    fb.inv_batched(z)
torch.cuda.synchronize()
print("ok")
