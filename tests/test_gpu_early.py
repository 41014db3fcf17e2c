"""EarlyInv: for 2048 <= n <= 4096 (lu2) and 4096 < n <= 8192 (the blocked LU's lu2
tail) part of the triangular inverses, the top-level products and the product block U11^-1 L11^-1 are
formed on a low-priority stream while the LU's chain-bound tail still runs, then joined.  These tests
cover what the config-5 sizes do not: ragged n (the split h = n/2 rounded to the 32-column steps, a
Ktail that is not n/2), both forced branches and the device-decided AUTO (whose part-2 inversion uses
another scratch matrix), the real inversion frob_dinv (with a column permutation in the product
epilogue), and CUDA-graph capture of the fork / join (replay bitwise equal to the direct call)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
fb = pytest.importorskip("paper_2208_01239_b200")

DEV = "cuda"


def _t(z):
    return torch.from_numpy(np.ascontiguousarray(z)).to(DEV)


def _resid(z, x):
    e = z @ x - torch.eye(z.shape[0], dtype=z.dtype, device=DEV)
    return float(torch.linalg.norm(e))


@pytest.mark.parametrize("n", [2048, 2050, 2111, 3001])
@pytest.mark.parametrize("branch", ["auto", "b"])
def test_lu2_early_vs_oracle(n, branch):
    z = synth.config2(n, seed=n)
    x = fb.inv(_t(z), branch=branch).cpu().numpy()
    ref, _ = oracle.zinv_gj(z)
    assert oracle.rel_fro(x, ref) <= 1e-10 * max(1.0, np.linalg.cond(z) / 1e4)


@pytest.mark.parametrize("n", [2100, 4100])
def test_early_device_auto_switch_bitwise_host_auto(n):
    # A nearly singular: AUTO inverts both parts (part 2 takes EarlyInv's second scratch matrix)
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    a[:, 1] = a[:, 0] + 1e-13 * rng.standard_normal(n)
    b = rng.standard_normal((n, n)) + np.sqrt(n) * np.eye(n)
    zt = _t(a + 1j * b)
    xh, ih = fb.inv(zt, info=True)
    xd, idv = fb.inv(zt, device_auto=True, info=True)
    assert ih["branch_used"] == 2 and idv["branch_used"] == 2
    assert torch.equal(xh, xd)
    assert _resid(zt, xh) <= 1e-11 * n * max(1.0, np.linalg.cond(b) / 1e4) * 10


@pytest.mark.parametrize("n", [4200, 5000, 6001])
def test_getrf_early_residual_and_vs_complex_lu(n):
    z = synth.config2(n, seed=n)
    zt = _t(z)
    x = fb.inv(zt)
    r = _resid(zt, x)
    assert r <= 1e-11 * n * 10
    xz = fb.zinv(zt)
    assert float(torch.linalg.norm(x - xz) / torch.linalg.norm(xz)) <= 1e-10 * 10


@pytest.mark.parametrize("n", [2048, 2100, 3001])
def test_dinv_early_vs_oracle(n):
    a = synth.config2(n, seed=n + 5).real.copy()
    x = fb.dinv(_t(a)).cpu().numpy()
    ref, info, _ = oracle.dinv(a)
    assert info == 0
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) <= 1e-12 * max(1.0, np.linalg.cond(a) / 100)


@pytest.mark.parametrize("n", [2100, 4200])
def test_early_graph_capture_bitwise(n):
    z = _t(synth.config2(n, seed=7))
    direct = torch.empty_like(z)
    fb.inv(z, branch="a", out=direct)
    out = torch.empty_like(z)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fb.inv(z, branch="a", out=out)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fb.inv(z, branch="a", out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, direct)


def test_early_repeat_bitwise():
    # the auxiliary stream's work joins deterministically: repeated calls are bit-identical
    z = _t(synth.config2(2100, seed=11))
    x0 = fb.inv(z)
    for _ in range(3):
        assert torch.equal(fb.inv(z), x0)
