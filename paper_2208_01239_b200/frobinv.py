"""Thin Python binding of libfrobinv.so (include/frobinv.h) -- argument marshalling only.

Every step of the method runs in the CUDA kernels behind the C ABI; this module only
allocates torch tensors for outputs / workspaces, passes device pointers and the
current CUDA stream, and maps status codes to exceptions.  There is no CPU fallback:
if the library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfrobinv.so")

STATUS = {0: "ok", 1: "singular", 2: "both_singular", 3: "not_converged", 4: "invalid_arg",
          5: "nonfinite", 6: "workspace", 7: "cuda"}
BRANCH = {"auto": 0, "a": 1, "b": 2}
METHOD = {"frobenius": 0, "frob": 0, "zlu": 1}

# header declarations (name -> (restype, argtypes)); tests check every one is exported
_vp, _dp, _ip = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
_ll, _i, _sz, _d = ctypes.c_longlong, ctypes.c_int, ctypes.c_size_t, ctypes.c_double


OPT_FUSED_FIRST_STEP = 1
OPT_DEVICE_AUTO = 2


class DevStatus(ctypes.Structure):
    """frob_dev_status (include/frobinv.h): the device-side status record of frob_inv_dev."""
    _fields_ = [("status", ctypes.c_int), ("info", ctypes.c_int), ("branch_used", ctypes.c_int),
                ("nonfinite", ctypes.c_int), ("rho_a", ctypes.c_double), ("rho_b", ctypes.c_double),
                ("rho_m", ctypes.c_double), ("kappa_a", ctypes.c_double), ("kappa_b", ctypes.c_double)]


DEV_STATUS_BYTES = ctypes.sizeof(DevStatus)


class FrobInfo(ctypes.Structure):
    _fields_ = [("info", ctypes.c_int), ("branch_used", ctypes.c_int), ("rho_a", ctypes.c_double),
                ("rho_b", ctypes.c_double), ("rho_m", ctypes.c_double), ("kappa_a", ctypes.c_double),
                ("kappa_b", ctypes.c_double)]

    def as_dict(self):
        return {"info": self.info, "branch_used": self.branch_used, "rho_a": self.rho_a,
                "rho_b": self.rho_b, "rho_m": self.rho_m, "kappa_a": self.kappa_a, "kappa_b": self.kappa_b}


_FIP = ctypes.POINTER(FrobInfo)
SIGNATURES = {
    "frob_inv_workspace_bytes": (_sz, [_i]),
    "frob_inv": (_i, [_i, _vp, _ll, _vp, _ll, _i, _vp, _sz, _vp, _FIP]),
    "frob_inv_opts": (_i, [_i, _vp, _ll, _vp, _ll, _i, _i, _vp, _sz, _vp, _FIP]),
    "frob_inv_rand": (_i, [_i, _vp, _ll, _vp, _ll, _d, _vp, _sz, _vp, _FIP]),
    "frob_inv_host_workspace_bytes": (_sz, [_i]),
    "frob_inv_host": (_i, [_i, _vp, _vp, _i, _vp, _sz, _vp, _FIP]),
    "frob_inv_host_many_workspace_bytes": (_sz, [_i]),
    "frob_inv_host_many": (_i, [_i, _i, _vp, _vp, _i, _vp, _vp, _sz, _vp]),
    "frob_inv_dev": (_i, [_i, _vp, _ll, _vp, _ll, _i, _i, _vp, _vp, _sz, _vp]),
    "frob_dtrmm": (_i, [_i, _i, _i, _d, _vp, _ll, _vp, _ll, _vp, _ll, _vp]),
    "frob_inv_batched_host_workspace_bytes": (_sz, [_i, _i]),
    "frob_inv_batched_host": (_i, [_i, _i, _vp, _vp, _i, _vp, _i, _vp, _sz, _vp]),
    "zinv_lu_workspace_bytes": (_sz, [_i]),
    "zinv_lu": (_i, [_i, _vp, _ll, _vp, _ll, _vp, _sz, _vp, _ip]),
    "frob_inv_batched_workspace_bytes": (_sz, [_i, _i]),
    "frob_inv_batched": (_i, [_i, _i, _vp, _ll, _vp, _ll, _i, _vp, _vp, _vp, _sz, _vp]),
    "zinv_lu_batched_workspace_bytes": (_sz, [_i, _i]),
    "zinv_lu_batched": (_i, [_i, _i, _vp, _ll, _vp, _ll, _vp, _vp, _sz, _vp]),
    "frob_newton_workspace_bytes": (_sz, [_i, _i]),
    "frob_sign_newton": (_i, [_i, _vp, _vp, _d, _i, _i, _vp, _sz, _vp, _ip, _dp, _dp]),
    "frob_polar_newton": (_i, [_i, _vp, _vp, _vp, _d, _i, _i, _vp, _sz, _vp, _ip, _dp, _dp]),
    "frob_hpd_inv_workspace_bytes": (_sz, [_i]),
    "frob_hpd_inv": (_i, [_i, _vp, _ll, _vp, _ll, _vp, _sz, _vp, _ip]),
    "zhpd_inv_chol_workspace_bytes": (_sz, [_i]),
    "frob_dpoinv_workspace_bytes": (_sz, [_i]),
    "frob_dpoinv": (_i, [_i, _vp, _ll, _vp, _ll, _vp, _sz, _vp, _ip]),
    "zhpd_inv_chol": (_i, [_i, _vp, _ll, _vp, _ll, _vp, _sz, _vp, _ip]),
    "frob_sylvester_workspace_bytes": (_sz, [_i, _i, _i]),
    "frob_sylvester": (_i, [_i, _i, _vp, _vp, _vp, _vp, _d, _i, _i, _vp, _sz, _vp, _ip, _dp]),
    "frob_lyapunov": (_i, [_i, _vp, _vp, _vp, _d, _i, _i, _vp, _sz, _vp, _ip, _dp]),
    "frob_dgemm": (_i, [_i, _i, _i, _d, _vp, _ll, _vp, _ll, _d, _vp, _ll, _vp]),
    "frob_dinv_workspace_bytes": (_sz, [_i]),
    "frob_dinv": (_i, [_i, _vp, _ll, _vp, _ll, _vp, _sz, _vp, _FIP]),
    "frob_dgetrf_workspace_bytes": (_sz, [_i]),
    "frob_dgetrf": (_i, [_i, _vp, _ll, _vp, _vp, _sz, _vp, _FIP]),
    "frob_profile_enable": (None, [_i]),
    "frob_profile_read": (_i, [ctypes.c_char_p, _sz]),
    "frob_status_string": (ctypes.c_char_p, [_i]),
    "frob_last_cuda_error": (ctypes.c_char_p, []),
    "frob_version": (_i, []),
    "frob_launch_count": (ctypes.c_ulonglong, []),
}

_lib = None
_lock = threading.Lock()


class FrobError(RuntimeError):
    def __init__(self, fn, status, info=None):
        self.status = status
        self.name = STATUS.get(status, str(status))
        self.info = info
        msg = f"{fn}: {self.name}"
        if status == 7 and _lib is not None:
            msg += " (" + _lib.frob_last_cuda_error().decode() + ")"
        if info is not None:
            msg += f" info={info}"
        super().__init__(msg)


def load(path: str = LIB_PATH):
    """Load libfrobinv.so (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def profile_enable(on: bool = True):
    """Per-kernel CUDA-event timing inside the library (measurement passes only)."""
    load().frob_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kernel: {"launches", "total_ms", "flops"}} of the launches since profile_enable."""
    import json
    L = load()
    n = L.frob_profile_read(None, 0)
    if n < 0:
        raise RuntimeError("frob_profile_read failed")
    buf = ctypes.create_string_buffer(n + 1)
    L.frob_profile_read(buf, n + 1)
    return json.loads(buf.value.decode())


def launch_count() -> int:
    """Kernels launched through the library so far in this process."""
    return int(load().frob_launch_count())


def _need_cuda(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_ws_cache: dict = {}


def workspace(nbytes: int, device) -> torch.Tensor:
    """Cached device workspace (uint8) of at least nbytes on `device`."""
    key = (torch.device(device).index, torch.cuda.current_stream(device).cuda_stream)
    t = _ws_cache.get(key)
    if t is None or t.numel() < nbytes:
        t = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = t
    return t


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def _check(fn, st, info=None):
    if st != 0:
        raise FrobError(fn, st, info)


# ----------------------------------------------------------------------------- single matrix
def _check_out(x, z, name="out"):
    assert x.dtype == torch.complex128 and x.shape == z.shape and x.stride(1) == 1 and x.device == z.device, \
        f"{name}: complex128 {tuple(z.shape)} with unit column stride on {z.device} required"


def inv(z: torch.Tensor, branch: str = "auto", out: torch.Tensor | None = None, info: bool = False,
        fused: bool = False, device_auto: bool = False):
    """Z^{-1} by Frobenius inversion (Alg 1).  z: (n, n) complex128 CUDA tensor.
    fused=True: NEXT-1 first step C = U^{-1} (L^{-1} (P Y)) (FROB_OPT_FUSED_FIRST_STEP).
    device_auto=True: the AUTO branch decided on the device (FROB_OPT_DEVICE_AUTO; no host sync)."""
    L = load()
    _need_cuda(z, "z")
    assert z.dtype == torch.complex128 and z.dim() == 2 and z.shape[0] == z.shape[1]
    z = z if z.stride(1) == 1 else z.contiguous()
    n = z.shape[0]
    x = out if out is not None else torch.empty((n, n), dtype=torch.complex128, device=z.device)
    _check_out(x, z)
    ws = workspace(L.frob_inv_workspace_bytes(n), z.device)
    fi = FrobInfo()
    opts = (OPT_FUSED_FIRST_STEP if fused else 0) | (OPT_DEVICE_AUTO if device_auto else 0)
    st = L.frob_inv_opts(n, _p(z), z.stride(0), _p(x), x.stride(0), BRANCH[branch], opts,
                         _p(ws), ws.numel(), _stream(), ctypes.byref(fi) if info else None)
    _check("frob_inv", st, fi.as_dict() if info else None)
    return (x, fi.as_dict()) if info else x


def inv_dev(z: torch.Tensor, branch: str = "auto", out: torch.Tensor | None = None, fused: bool = False,
            device_auto: bool = False, status: torch.Tensor | None = None):
    """frob_inv_dev: like inv() but device-side errors land in a device status record (uint8 tensor
    of DEV_STATUS_BYTES on z's device) instead of a host synchronisation.  Returns (X, status);
    decode the record with dev_status(status) after the stream."""
    L = load()
    _need_cuda(z, "z")
    assert z.dtype == torch.complex128 and z.dim() == 2 and z.shape[0] == z.shape[1]
    z = z if z.stride(1) == 1 else z.contiguous()
    n = z.shape[0]
    x = out if out is not None else torch.empty((n, n), dtype=torch.complex128, device=z.device)
    _check_out(x, z)
    if status is None:
        status = torch.zeros(DEV_STATUS_BYTES, dtype=torch.uint8, device=z.device)
    assert status.is_cuda and status.dtype == torch.uint8 and status.numel() >= DEV_STATUS_BYTES
    ws = workspace(L.frob_inv_workspace_bytes(n), z.device)
    opts = (OPT_FUSED_FIRST_STEP if fused else 0) | (OPT_DEVICE_AUTO if device_auto else 0)
    st = L.frob_inv_dev(n, _p(z), z.stride(0), _p(x), x.stride(0), BRANCH[branch], opts, _p(status), _p(ws),
                        ws.numel(), _stream())
    _check("frob_inv_dev", st)
    return x, status


def dev_status(status: torch.Tensor) -> dict:
    """Decode a frob_dev_status record (synchronises through the device->host copy)."""
    raw = bytes(status[:DEV_STATUS_BYTES].cpu().numpy().tobytes())
    r = DevStatus.from_buffer_copy(raw)
    return {"status": STATUS.get(r.status, str(r.status)), "code": r.status, "info": r.info,
            "branch_used": r.branch_used, "nonfinite": r.nonfinite, "rho_a": r.rho_a, "rho_b": r.rho_b,
            "rho_m": r.rho_m, "kappa_a": r.kappa_a, "kappa_b": r.kappa_b}


def draw_mu(seed: int) -> float:
    """Alg 5 line 1: mu uniform in [0, 1] from a seeded counter-based generator (Philox)."""
    import numpy as np
    return float(np.random.Generator(np.random.Philox(key=seed)).random())


def inv_rand(z: torch.Tensor, mu: float | None = None, seed: int = 0, out: torch.Tensor | None = None,
             info: bool = False):
    """Randomized Frobenius inversion (Alg 5).  mu in [0, 1]; drawn from `seed` if None."""
    L = load()
    _need_cuda(z, "z")
    assert z.dtype == torch.complex128 and z.dim() == 2 and z.shape[0] == z.shape[1]
    z = z if z.stride(1) == 1 else z.contiguous()
    n = z.shape[0]
    mu = draw_mu(seed) if mu is None else float(mu)
    x = out if out is not None else torch.empty((n, n), dtype=torch.complex128, device=z.device)
    ws = workspace(L.frob_inv_workspace_bytes(n), z.device)
    fi = FrobInfo()
    st = L.frob_inv_rand(n, _p(z), z.stride(0), _p(x), x.stride(0), mu, _p(ws), ws.numel(), _stream(),
                         ctypes.byref(fi) if info else None)
    _check("frob_inv_rand", st, fi.as_dict() if info else None)
    return (x, fi.as_dict()) if info else x


def _check_host_out(x_host, z_host):
    assert (x_host.shape == z_host.shape and x_host.dtype == torch.complex128 and x_host.is_contiguous()
            and not x_host.is_cuda), "x_host: contiguous CPU complex128 of z_host's shape required"


def inv_host(z_host: torch.Tensor, x_host: torch.Tensor | None = None, branch: str = "auto",
             device="cuda"):
    """End-to-end call with HOST buffers (pinned recommended): H2D, invert, D2H."""
    L = load()
    assert z_host.dtype == torch.complex128 and not z_host.is_cuda and z_host.is_contiguous()
    n = z_host.shape[0]
    assert z_host.dim() == 2 and z_host.shape[0] == z_host.shape[1]
    x_host = x_host if x_host is not None else torch.empty_like(z_host).pin_memory()
    _check_host_out(x_host, z_host)
    ws = workspace(L.frob_inv_host_workspace_bytes(n), device)
    st = L.frob_inv_host(n, _p(z_host), _p(x_host), BRANCH[branch], _p(ws), ws.numel(), _stream(), None)
    _check("frob_inv_host", st)
    return x_host


def inv_host_many(z_host: torch.Tensor, x_host: torch.Tensor | None = None, branch: str = "auto",
                  device="cuda", status: bool = False):
    """count matrices (count, n, n) in pinned HOST memory, pipelined: the copies of matrices
    i + 1 (in) and i - 1 (out) overlap the inversion of matrix i (frob_inv_host_many).
    status=True: return (x_host, per-matrix status int32[count]) and do not raise on a failing
    matrix (its status code says which)."""
    L = load()
    assert z_host.dtype == torch.complex128 and not z_host.is_cuda and z_host.is_contiguous() and z_host.dim() == 3
    count, n = z_host.shape[0], z_host.shape[1]
    assert z_host.shape[2] == n
    x_host = x_host if x_host is not None else torch.empty_like(z_host).pin_memory()
    _check_host_out(x_host, z_host)
    codes = torch.empty(count, dtype=torch.int32).pin_memory()
    ws = workspace(L.frob_inv_host_many_workspace_bytes(n), device)
    st = L.frob_inv_host_many(n, count, _p(z_host), _p(x_host), BRANCH[branch], _p(codes), _p(ws), ws.numel(),
                              _stream())
    if status:
        if st not in STATUS or st in (4, 6, 7):
            _check("frob_inv_host_many", st)
        return x_host, codes
    _check("frob_inv_host_many", st)
    return x_host


def inv_batched_host(z_host: torch.Tensor, x_host: torch.Tensor | None = None, branch: str = "auto",
                     chunk: int | None = None, device="cuda"):
    """Batched Frobenius inversion (n <= 128) with pinned HOST buffers (batch, n, n), pipelined in
    chunks (frob_inv_batched_host).  Returns (x_host, info int32 tensor [batch])."""
    L = load()
    assert z_host.dtype == torch.complex128 and not z_host.is_cuda and z_host.is_contiguous() and z_host.dim() == 3
    batch, n = z_host.shape[0], z_host.shape[1]
    assert z_host.shape[2] == n
    x_host = x_host if x_host is not None else torch.empty_like(z_host).pin_memory()
    _check_host_out(x_host, z_host)
    info = torch.empty(batch, dtype=torch.int32).pin_memory()  # pageable memory would stall the pipeline
    chunk = chunk or max(1, min(batch, (256 << 20) // (16 * n * n)))
    ws = workspace(L.frob_inv_batched_host_workspace_bytes(n, chunk), device)
    st = L.frob_inv_batched_host(n, batch, _p(z_host), _p(x_host), BRANCH[branch], _p(info), chunk, _p(ws),
                                 ws.numel(), _stream())
    _check("frob_inv_batched_host", st)
    return x_host, info


def zinv(z: torch.Tensor, out: torch.Tensor | None = None):
    """Complex-LU inversion (Alg 3 over C), the comparator."""
    L = load()
    _need_cuda(z, "z")
    assert z.dtype == torch.complex128 and z.dim() == 2
    z = z if z.stride(1) == 1 else z.contiguous()
    n = z.shape[0]
    x = out if out is not None else torch.empty((n, n), dtype=torch.complex128, device=z.device)
    ws = workspace(L.zinv_lu_workspace_bytes(n), z.device)
    st = L.zinv_lu(n, _p(z), z.stride(0), _p(x), x.stride(0), _p(ws), ws.numel(), _stream(), None)
    _check("zinv_lu", st)
    return x


# ----------------------------------------------------------------------------- batched
def inv_batched(z: torch.Tensor, branch: str = "auto", out: torch.Tensor | None = None):
    """Batched Frobenius inversion, z: (batch, n, n) complex128 contiguous, n <= 128.
    Returns (X, info int32[batch], branch_used uint8[batch])."""
    L = load()
    _need_cuda(z, "z")
    assert z.dtype == torch.complex128 and z.dim() == 3 and z.is_contiguous()
    b, n, _ = z.shape
    x = out if out is not None else torch.empty_like(z)
    info = torch.empty(b, dtype=torch.int32, device=z.device)
    bu = torch.empty(b, dtype=torch.uint8, device=z.device)
    st = L.frob_inv_batched(n, b, _p(z), n * n, _p(x), n * n, BRANCH[branch], _p(info), _p(bu), None, 0,
                            _stream())
    _check("frob_inv_batched", st)
    return x, info, bu


def zinv_batched(z: torch.Tensor, out: torch.Tensor | None = None):
    """Batched complex-LU comparator (complex Gauss-Jordan), n <= 128 (64 < n: a 2-CTA cluster per
    matrix).  Returns (X, info int32[batch])."""
    L = load()
    _need_cuda(z, "z")
    assert z.dtype == torch.complex128 and z.dim() == 3 and z.is_contiguous()
    b, n, _ = z.shape
    x = out if out is not None else torch.empty_like(z)
    info = torch.empty(b, dtype=torch.int32, device=z.device)
    st = L.zinv_lu_batched(n, b, _p(z), n * n, _p(x), n * n, _p(info), None, 0, _stream())
    _check("zinv_lu_batched", st)
    return x, info


# ----------------------------------------------------------------------------- Newton drivers
def sign(z: torch.Tensor, tol: float = 1e-12, max_iter: int = 50, method: str = "frobenius",
         trace: bool = False):
    """Matrix sign by Newton.  Returns (S, iters, final_delta[, deltas])."""
    L = load()
    _need_cuda(z, "z")
    z = z.contiguous()
    n = z.shape[0]
    s = torch.empty_like(z)
    ws = workspace(L.frob_newton_workspace_bytes(n, METHOD[method]), z.device)
    it = ctypes.c_int(0)
    fd = ctypes.c_double(0.0)
    tr = (ctypes.c_double * max_iter)()
    st = L.frob_sign_newton(n, _p(z), _p(s), tol, max_iter, METHOD[method], _p(ws), ws.numel(), _stream(),
                            ctypes.byref(it), ctypes.byref(fd), tr)
    if st not in (0, 3):
        _check("frob_sign_newton", st)
    out = (s, it.value, fd.value)
    return out + ([tr[i] for i in range(it.value)],) if trace else out


def polar(a: torch.Tensor, tol: float = 1e-12, max_iter: int = 50, method: str = "frobenius"):
    """Polar decomposition A = U H by Newton.  Returns (U, H, iters, final_delta)."""
    L = load()
    _need_cuda(a, "a")
    a = a.contiguous()
    n = a.shape[0]
    u = torch.empty_like(a)
    h = torch.empty_like(a)
    ws = workspace(L.frob_newton_workspace_bytes(n, METHOD[method]), a.device)
    it = ctypes.c_int(0)
    fd = ctypes.c_double(0.0)
    st = L.frob_polar_newton(n, _p(a), _p(u), _p(h), tol, max_iter, METHOD[method], _p(ws), ws.numel(),
                             _stream(), ctypes.byref(it), ctypes.byref(fd), None)
    if st not in (0, 3):
        _check("frob_polar_newton", st)
    return u, h, it.value, fd.value


# ----------------------------------------------------------------------------- real blocks
def _hpd_call(fn, wsfn, z, out, check):
    L = load()
    _need_cuda(z, "z")
    assert z.dtype == torch.complex128 and z.dim() == 2 and z.shape[0] == z.shape[1]
    z = z if z.stride(1) == 1 else z.contiguous()
    n = z.shape[0]
    x = out if out is not None else torch.empty((n, n), dtype=torch.complex128, device=z.device)
    ws = workspace(getattr(L, wsfn)(n), z.device)
    info = ctypes.c_int(0)
    st = getattr(L, fn)(n, _p(z), z.stride(0), _p(x), x.stride(0), _p(ws), ws.numel(), _stream(),
                        ctypes.byref(info) if check else None)
    _check(fn, st, {"info": info.value} if check else None)
    return x


def hpd_inv(z: torch.Tensor, out: torch.Tensor | None = None, check: bool = True):
    """HPD inversion by the Cholesky-based Frobenius variant (Alg 6)."""
    return _hpd_call("frob_hpd_inv", "frob_hpd_inv_workspace_bytes", z, out, check)


def zhpd_inv(z: torch.Tensor, out: torch.Tensor | None = None, check: bool = True):
    """HPD inversion by complex Cholesky (Alg 8 over C), the comparator."""
    return _hpd_call("zhpd_inv_chol", "zhpd_inv_chol_workspace_bytes", z, out, check)


def dpoinv(a: torch.Tensor, out: torch.Tensor | None = None, check: bool = True):
    """Real SPD inversion (Alg 8 over R): Thm 6.2's T_pinv operation.  a: (n, n) float64 CUDA."""
    L = load()
    _need_cuda(a, "a")
    assert a.dtype == torch.float64 and a.dim() == 2 and a.shape[0] == a.shape[1] and a.stride(1) == 1
    n = a.shape[0]
    x = out if out is not None else torch.empty((n, n), dtype=torch.float64, device=a.device)
    ws = workspace(L.frob_dpoinv_workspace_bytes(n), a.device)
    info = ctypes.c_int(0)
    st = L.frob_dpoinv(n, _p(a), a.stride(0), _p(x), x.stride(0), _p(ws), ws.numel(), _stream(),
                       ctypes.byref(info) if check else None)
    _check("frob_dpoinv", st, {"info": info.value} if check else None)
    return x


def sylvester(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, tol: float = 1e-12, max_iter: int = 50,
              method: str = "frobenius"):
    """A X + X B = C via the sign of [[A, -C], [0, -B]].  Returns (X, iters, delta)."""
    L = load()
    for t, nm in ((a, "a"), (b, "b"), (c, "c")):
        _need_cuda(t, nm)
        assert t.dtype == torch.complex128
    a, b, c = a.contiguous(), b.contiguous(), c.contiguous()
    m, n = a.shape[0], b.shape[0]
    assert c.shape == (m, n)
    x = torch.empty((m, n), dtype=torch.complex128, device=a.device)
    ws = workspace(L.frob_sylvester_workspace_bytes(m, n, METHOD[method]), a.device)
    it, d = ctypes.c_int(0), ctypes.c_double(0.0)
    st = L.frob_sylvester(m, n, _p(a), _p(b), _p(c), _p(x), tol, max_iter, METHOD[method], _p(ws), ws.numel(),
                          _stream(), ctypes.byref(it), ctypes.byref(d))
    if st not in (0, 3):
        _check("frob_sylvester", st)
    return x, it.value, d.value


def lyapunov(a: torch.Tensor, c: torch.Tensor, tol: float = 1e-12, max_iter: int = 50, method: str = "frobenius"):
    """A X + X A^* = C.  Returns (X, iters, delta)."""
    L = load()
    _need_cuda(a, "a")
    _need_cuda(c, "c")
    a, c = a.contiguous(), c.contiguous()
    n = a.shape[0]
    x = torch.empty((n, n), dtype=torch.complex128, device=a.device)
    ws = workspace(L.frob_sylvester_workspace_bytes(n, n, METHOD[method]), a.device)
    it, d = ctypes.c_int(0), ctypes.c_double(0.0)
    st = L.frob_lyapunov(n, _p(a), _p(c), _p(x), tol, max_iter, METHOD[method], _p(ws), ws.numel(), _stream(),
                         ctypes.byref(it), ctypes.byref(d))
    if st not in (0, 3):
        _check("frob_lyapunov", st)
    return x, it.value, d.value


def dgemm(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor | None = None, alpha: float = 1.0,
          beta: float = 0.0):
    L = load()
    _need_cuda(a, "a")
    m, k = a.shape
    k2, n = b.shape
    assert k == k2 and a.dtype == b.dtype == torch.float64
    if c is None:
        c = torch.empty((m, n), dtype=torch.float64, device=a.device)
        beta = 0.0
    st = L.frob_dgemm(m, n, k, alpha, _p(a), a.stride(0), _p(b), b.stride(0), beta, _p(c), c.stride(0),
                      _stream())
    _check("frob_dgemm", st)
    return c


def dtrmm(t: torch.Tensor, b: torch.Tensor, uplo: str = "lower", alpha: float = 1.0,
          c: torch.Tensor | None = None):
    """C = alpha tri(T) B on the GEMM engine (T's other strict triangle must be zero)."""
    L = load()
    _need_cuda(t, "t")
    n, m = b.shape
    assert t.shape == (n, n) and t.dtype == b.dtype == torch.float64
    c = c if c is not None else torch.empty((n, m), dtype=torch.float64, device=b.device)
    st = L.frob_dtrmm(1 if uplo == "upper" else 2, n, m, alpha, _p(t), t.stride(0), _p(b), b.stride(0), _p(c),
                      c.stride(0), _stream())
    _check("frob_dtrmm", st)
    return c


def dinv(a: torch.Tensor, out: torch.Tensor | None = None, info: bool = False):
    L = load()
    _need_cuda(a, "a")
    n = a.shape[0]
    x = out if out is not None else torch.empty_like(a)
    ws = workspace(L.frob_dinv_workspace_bytes(n), a.device)
    fi = FrobInfo()
    st = L.frob_dinv(n, _p(a), a.stride(0), _p(x), x.stride(0), _p(ws), ws.numel(), _stream(),
                     ctypes.byref(fi) if info else None)
    _check("frob_dinv", st, fi.as_dict() if info else None)
    return (x, fi.as_dict()) if info else x


def dgetrf(a: torch.Tensor):
    """In-place LU of a copy: returns (LU, perm) with (P A)[i] = A[perm[i]]."""
    L = load()
    _need_cuda(a, "a")
    lu = a.clone()
    n = a.shape[0]
    perm = torch.empty(n, dtype=torch.int32, device=a.device)
    ws = workspace(L.frob_dgetrf_workspace_bytes(n), a.device)
    fi = FrobInfo()
    st = L.frob_dgetrf(n, _p(lu), lu.stride(0), _p(perm), _p(ws), ws.numel(), _stream(), ctypes.byref(fi))
    if st not in (0, 1):
        _check("frob_dgetrf", st)
    return lu, perm, fi.as_dict()
