"""Small invocations of every hot-path entry point for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck, one tool per run): frob_inv (AUTO literal, forced S2, NEXT-1, device AUTO) and
zinv_lu at n = 300 (lu2, one-CTA panels) and n = 1100 (lu2 cluster panels + look-ahead pipeline),
frob_inv at n = 4200 (blocked getrf), the batched kernels at n = 32 / 128 and the complex batched
comparator.  Prints one line per case; exits non-zero on a wrong result.
  compute-sanitizer --tool memcheck python tools/sanitize_run.py [quick]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2208_01239_b200 as fb  # noqa: E402
import synth  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
eye_cache = {}


def resid(z, x):
    n = z.shape[0]
    e = z @ x - torch.eye(n, dtype=torch.complex128, device="cuda")
    return float(torch.linalg.norm(e))


ok = True
sizes = [300] if quick else [300, 1100, 4200]
for n in sizes:
    z = torch.from_numpy(synth.config2(n, seed=n)).cuda()
    for name, f in (("frob_auto", lambda: fb.inv(z)), ("frob_b", lambda: fb.inv(z, branch="b")),
                    ("frob_fused", lambda: fb.inv(z, fused=True)), ("frob_dev_auto", lambda: fb.inv(z, device_auto=True)),
                    ("zinv_lu", lambda: fb.zinv(z))):
        if n > 1100 and name in ("frob_b", "frob_fused"):
            continue
        x = f()
        r = resid(z, x)
        good = r <= 1e-8 * n
        ok &= good
        print(f"n={n} {name}: residual {r:.2e} {'ok' if good else 'BAD'}", flush=True)
for n, cnt in ((32, 64), (128, 8)):
    zb = torch.from_numpy(synth.batch(n, cnt, seed=1)).cuda()
    for name, f in (("frob_batched", lambda: fb.inv_batched(zb)[0]), ("zinv_batched", lambda: fb.zinv_batched(zb)[0])):
        x = f()
        e = torch.matmul(zb, x) - torch.eye(n, dtype=torch.complex128, device="cuda")
        r = float(torch.linalg.norm(e, dim=(1, 2)).max())
        good = r <= 1e-8 * n
        ok &= good
        print(f"batched n={n} x{cnt} {name}: max residual {r:.2e} {'ok' if good else 'BAD'}", flush=True)
torch.cuda.synchronize()
print("ALL OK" if ok else "FAILURES")
sys.exit(0 if ok else 1)
