"""frob_inv_host_many (include/frobinv.h): count matrices in pinned host memory, the copies of
neighbouring matrices overlapping each inversion on two library-owned copy streams.  Every
result must equal the device-resident frob_inv of the same matrix bit for bit (same kernels,
double-buffered device copies), for count 1, 2 (no buffer reuse) and 5 (both buffers reused)."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,count,branch", [(300, 5, "auto"), (1024, 2, "a"), (1024, 5, "auto"), (77, 1, "b")])
def test_host_many_equals_device_calls(n, count, branch):
    import paper_2208_01239_b200 as fb
    zs = torch.stack([torch.from_numpy(synth.config2(n, seed=40 + i)) for i in range(count)]).pin_memory()
    xs = torch.empty_like(zs).pin_memory()
    fb.inv_host_many(zs, xs, branch=branch)
    for i in range(count):
        ref = fb.inv(zs[i].cuda(), branch=branch).cpu()
        assert torch.equal(xs[i], ref), i


def test_host_many_matches_inv_host():
    import paper_2208_01239_b200 as fb
    n = 512
    zs = torch.stack([torch.from_numpy(synth.config2(n, seed=7 + i)) for i in range(3)]).pin_memory()
    xs = fb.inv_host_many(zs)
    for i in range(3):
        assert torch.equal(xs[i], fb.inv_host(zs[i].contiguous().pin_memory()))


def test_inv_host_chunked_output_bitwise():
    """n >= 8192: frob_inv_host copies X out in 8 row blocks while the final GEMM continues; the result
    equals the device-resident frob_inv bit for bit."""
    import paper_2208_01239_b200 as fb
    n = 8192
    zh = torch.from_numpy(synth.config2(n, seed=3)).pin_memory()
    xh = fb.inv_host(zh)
    ref = fb.inv(zh.cuda()).cpu()
    assert torch.equal(xh, ref)
