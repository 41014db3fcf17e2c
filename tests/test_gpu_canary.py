"""Out-of-bounds write detection without compute-sanitizer (closed on this GPU pool): every buffer a
call writes -- the output X, the workspace and the batched info arrays -- is carved from a larger
allocation whose margins hold a NaN canary pattern, and the margins must be intact after the call.
The sizes are ragged (not multiples of the 64 x 64 GEMM tile, the 32-column panel, the 512-row
cluster slice or the 2048-row NEXT-1 substitution block), so every edge path runs; outputs with a
leading dimension larger than n must also leave the gap columns untouched."""
import math

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
fb = pytest.importorskip("paper_2208_01239_b200")
from paper_2208_01239_b200 import frobinv as fbi  # noqa: E402

DEV = "cuda"
PAD = 4096  # bytes of canary on each side


def _canary_u8(nbytes):
    """uint8 buffer of nbytes + 2 PAD filled with 0xFF (a NaN pattern for doubles); returns (buf, inner)."""
    buf = torch.full((nbytes + 2 * PAD,), 0xFF, dtype=torch.uint8, device=DEV)
    return buf, buf[PAD:PAD + nbytes]


def _intact(buf, nbytes):
    head, tail = buf[:PAD], buf[PAD + nbytes:]
    return bool((head == 0xFF).all()) and bool((tail == 0xFF).all())


@pytest.mark.parametrize("n,ldx_pad", [(1, 0), (37, 3), (300, 5), (1100, 8), (4100, 4)])
@pytest.mark.parametrize("mode", ["auto", "fused", "device_auto"])
def test_frob_inv_writes_stay_in_bounds(n, ldx_pad, mode):
    L = fbi.load()
    z = synth.config2(n, seed=n + 11)
    zt = torch.from_numpy(z).to(DEV)
    ldx = n + ldx_pad
    xbytes = ((n - 1) * ldx + n) * 16
    xbuf, xin = _canary_u8(xbytes)
    wsb = L.frob_inv_workspace_bytes(n)
    wbuf, win = _canary_u8(wsb)
    opts = {"auto": 0, "fused": fbi.OPT_FUSED_FIRST_STEP, "device_auto": fbi.OPT_DEVICE_AUTO}[mode]
    st = L.frob_inv_opts(n, fbi._p(zt), n, fbi._p(xin), ldx, 0, opts, fbi._p(win), wsb, fbi._stream(), None)
    torch.cuda.synchronize()
    assert st == 0
    assert _intact(xbuf, xbytes), "write outside X"
    assert _intact(wbuf, wsb), "write outside the workspace"
    x = torch.as_strided(xin.view(torch.complex128), (n, n), (ldx, 1))
    if ldx_pad:  # gap columns between rows untouched
        full = xin[: (n - 1) * ldx * 16].view(torch.complex128).reshape(n - 1, ldx)
        gap = torch.view_as_real(full[:, n:]).contiguous().view(torch.uint8)
        assert bool((gap == 0xFF).all()), "write into the leading-dimension gap"
    ref, _ = oracle.zinv_gj(z) if n <= 1100 else (None, None)
    xs = x.cpu().numpy()
    if ref is not None:
        assert oracle.rel_fro(xs, ref) <= 1e-10 * max(1.0, np.linalg.cond(z) / 1e4)
    else:
        r = torch.linalg.norm(zt @ x - torch.eye(n, dtype=torch.complex128, device=DEV))
        assert float(r) <= 1e-11 * n * 2


@pytest.mark.parametrize("n,count", [(1, 3), (17, 5), (32, 7), (50, 9), (64, 3), (100, 4), (128, 5)])
def test_batched_writes_stay_in_bounds(n, count):
    L = fbi.load()
    zs = synth.batch(n, count, seed=n, shift=8.0)
    zt = torch.from_numpy(zs).to(DEV)
    xbytes = count * n * n * 16
    xbuf, xin = _canary_u8(xbytes)
    ibuf, iin = _canary_u8(count * 4)
    bbuf, bin_ = _canary_u8(count)
    st = L.frob_inv_batched(n, count, fbi._p(zt), n * n, fbi._p(xin), n * n, 0, fbi._p(iin), fbi._p(bin_), None, 0,
                            fbi._stream())
    torch.cuda.synchronize()
    assert st == 0
    assert _intact(xbuf, xbytes) and _intact(ibuf, count * 4) and _intact(bbuf, count)
    x = xin.view(torch.complex128).reshape(count, n, n).cpu().numpy()
    for i in range(count):
        ref, _ = oracle.zinv_gj(zs[i])
        assert oracle.rel_fro(x[i], ref) <= 1e-10 * max(1.0, np.linalg.cond(zs[i]) / 1e4)
    # the complex comparator too
    xbuf2, xin2 = _canary_u8(xbytes)
    st = L.zinv_lu_batched(n, count, fbi._p(zt), n * n, fbi._p(xin2), n * n, fbi._p(iin), None, 0, fbi._stream())
    torch.cuda.synchronize()
    assert st == 0 and _intact(xbuf2, xbytes)


@pytest.mark.parametrize("n", [5, 300, 1100])
def test_zinv_and_hpd_writes_stay_in_bounds(n):
    L = fbi.load()
    z = synth.config2(n, seed=3)
    zt = torch.from_numpy(z).to(DEV)
    xbytes = n * n * 16
    for fn, wsfn, inp in (("zinv_lu", "zinv_lu_workspace_bytes", zt),
                          ("frob_hpd_inv", "frob_hpd_inv_workspace_bytes", torch.from_numpy(synth.hpd(n, seed=n)).to(DEV)),
                          ("zhpd_inv_chol", "zhpd_inv_chol_workspace_bytes", torch.from_numpy(synth.hpd(n, seed=n)).to(DEV))):
        xbuf, xin = _canary_u8(xbytes)
        wsb = getattr(L, wsfn)(n)
        wbuf, win = _canary_u8(wsb)
        st = getattr(L, fn)(n, fbi._p(inp), n, fbi._p(xin), n, fbi._p(win), wsb, fbi._stream(), None)
        torch.cuda.synchronize()
        assert st == 0, fn
        assert _intact(xbuf, xbytes) and _intact(wbuf, wsb), fn
        x = xin.view(torch.complex128).reshape(n, n)
        r = float(torch.linalg.norm(inp @ x - torch.eye(n, dtype=torch.complex128, device=DEV)))
        assert math.isfinite(r) and r <= 1e-8 * n, (fn, r)
