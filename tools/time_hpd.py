"""HPD timings at n: Alg 6 (frob_hpd_inv), Alg 8 (zhpd_inv_chol), T_pinv (frob_dpoinv), T_mult: python tools/time_hpd.py N..."""
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2208_01239_b200 as fb  # noqa: E402
import synth  # noqa: E402


def med(f, reps=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for n in [int(v) for v in sys.argv[1:]]:
    z = torch.from_numpy(synth.hpd(n, seed=1)).cuda()
    a = z.real.contiguous()
    b = torch.empty_like(a)
    c = torch.empty_like(a)
    t6 = med(lambda: fb.hpd_inv(z, check=False))
    t8 = med(lambda: fb.zhpd_inv(z, check=False))
    tp = med(lambda: fb.dpoinv(a, check=False))
    tm = med(lambda: fb.dgemm(a, a, c))
    print(f"n={n}: alg6 {t6:.2f} ms  alg8 {t8:.2f} ms  T_pinv {tp:.2f} ms  T_mult {tm:.2f} ms  "
          f"T_pinv/T_mult {tp / tm:.2f}", flush=True)
