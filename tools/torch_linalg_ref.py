"""Context only (not the product): vendor-library timings on this GPU (cuSOLVER/MAGMA via torch)."""
import json
import torch

for n in (1024, 2048, 4096):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda") + n ** 0.5 * torch.eye(n, dtype=torch.float64, device="cuda")
    z = torch.complex(a, torch.randn_like(a))
    res = {"n": n}
    for name, fn in (("lu_factor_f64", lambda: torch.linalg.lu_factor(a)),
                     ("inv_f64", lambda: torch.linalg.inv(a)),
                     ("inv_c128", lambda: torch.linalg.inv(z))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name + "_ms"] = e0.elapsed_time(e1) / reps
    print(json.dumps(res))
