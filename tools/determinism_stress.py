"""Repeat-run determinism of frob_inv / zinv across sizes that exercise every LU path (one CTA,
cluster panels, look-ahead pipeline, split-K, the blocked LU with its priority streams,
9..16-CTA panels and lu2 tail): a race would show up as a bitwise difference."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2208_01239_b200 as fb
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
bad = 0
for n in (100, 513, 1024, 1500, 2048, 3000, 4096, 4700, 8192):
    z = torch.from_numpy(synth.config2(n, seed=n)).cuda()
    for name, f in (("frob", fb.inv), ("zinv", fb.zinv)):
        ref = f(z)
        for r in range(reps):
            x = f(z)
            if not torch.equal(x, ref):
                bad += 1
                print(f"MISMATCH {name} n={n} rep={r} max|diff|={float((x - ref).abs().max()):.3e}")
    print(f"n={n} ok" if bad == 0 else f"n={n} bad={bad}", flush=True)
print("deterministic" if bad == 0 else f"NONDETERMINISTIC ({bad})")
