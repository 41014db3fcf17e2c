"""Time the batched kernels (config 3 shapes) through the C ABI."""
import json
import sys
import torch
sys.path.insert(0, ".")
import paper_2208_01239_b200 as fb
import synth

for n, cnt in ((32, 65536), (64, 16384), (128, 16384)):
    z = torch.from_numpy(synth.batch(n, min(cnt, 4096), seed=0)).cuda()
    z = z.repeat((cnt + z.shape[0] - 1) // z.shape[0], 1, 1)[:cnt].contiguous()
    out = {"n": n, "batch": cnt}
    for name, fn in (("frob", lambda: fb.inv_batched(z)), ("zinv", lambda: fb.zinv_batched(z))):
        if name == "zinv" and n > 64:
            continue
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        fl = (10 if name == "frob" else 8) * n ** 3 * cnt
        out[name] = {"ms": ms, "inv_per_s": cnt / ms * 1e3, "tflops_alg": fl / ms / 1e9}
    print(json.dumps(out))
