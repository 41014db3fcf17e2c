"""CPU oracle for Frobenius inversion -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  The product path
(``paper_2208_01239_b200``) never imports it and shares no code with it.

The arithmetic lives in ``frob_oracle.c`` (plain loops, fp64, no BLAS, no FMA
contraction); this module compiles it with gcc and marshals numpy arrays.  The
Newton drivers below follow the paper's iterations step by step in numpy
(P:L1108-1111 sign, P:L1231-1233 polar), calling the C inversions.

Pins: tests/test_oracle_pins.py checks every function here against closed forms,
exact rational brute force, invariants and the paper's printed special cases.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "frob_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

BRANCH = {"auto": 0, "a": 1, "b": 2}
KAPPA_SWITCH = 2.5e4  # DESIGN.md reading R1': AUTO switch test on kappa_inf(A) / sqrt(n), kappa_inf = ||A||_inf ||A^-1||_inf


def build(force: bool = False) -> str:
    """Compile frob_oracle.c -> liboracle.so (gcc, -O2, OpenMP, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            dp = ctypes.POINTER(ctypes.c_double)
            ip = ctypes.POINTER(ctypes.c_int)
            L.or_dgetrf.argtypes = [ctypes.c_int, dp, ip]
            L.or_dtrtri_upper.argtypes = [ctypes.c_int, dp, dp]
            L.or_dgetri_solve.argtypes = [ctypes.c_int, dp, dp, dp]
            L.or_dinv.argtypes = [ctypes.c_int, dp, dp, dp]
            L.or_dgemm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp]
            L.or_frob_inv.argtypes = [ctypes.c_int, dp, dp, dp, dp, ctypes.c_int, ctypes.c_double, ip, dp]
            L.or_frob_inv_rand.argtypes = [ctypes.c_int, dp, dp, ctypes.c_double, dp, dp, ctypes.c_double,
                                           ip, dp]
            L.or_dpotrf_upper.argtypes = [ctypes.c_int, dp, dp]
            L.or_hpd_frob_inv.argtypes = [ctypes.c_int, dp, dp, dp, dp, ip]
            L.or_zhpd_inv_chol.argtypes = [ctypes.c_int, dp, dp, dp, dp]
            L.or_zinv_gj.argtypes = [ctypes.c_int, dp, dp]
            L.or_zinv_lu.argtypes = [ctypes.c_int, dp, dp, dp, dp]
            L.or_zgetrf.argtypes = [ctypes.c_int, dp, dp, ip]
            L.or_zgetrs.argtypes = [ctypes.c_int, dp, dp, ip, ctypes.c_int, ctypes.c_int, dp, dp]
            L.or_zgetrs.restype = None
            L.or_frob_inv_many.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, ctypes.c_int,
                                           ctypes.c_double, ip, dp, ip]
            for f in ("or_dgetrf", "or_dtrtri_upper", "or_dinv", "or_frob_inv", "or_frob_inv_rand", "or_zinv_gj",
                      "or_dpotrf_upper", "or_hpd_frob_inv", "or_zhpd_inv_chol",
                      "or_zinv_lu", "or_num_threads", "or_zgetrf", "or_frob_inv_many"):
                getattr(L, f).restype = ctypes.c_int
            L.or_dgetri_solve.restype = None
            L.or_dgemm.restype = None
            L.or_set_threads.argtypes = [ctypes.c_int]
            L.or_set_threads.restype = None
            _lib = L
    return _lib


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_threads(t: int) -> None:
    """OpenMP thread count of the oracle's loops (timing control; results do not depend on it)."""
    lib().or_set_threads(int(t))


def _p(a: np.ndarray, ct=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ real kernels
def dgetrf(a):
    """Alg 3 line 1. Returns (lu, ipiv, info); P A = L U with LAPACK ipiv order."""
    lu = _f64(a).copy()
    n = lu.shape[0]
    ipiv = np.zeros(max(n, 1), dtype=np.int32)
    info = lib().or_dgetrf(n, _p(lu), _p(ipiv, ctypes.c_int))
    return lu, ipiv[:n], info


def dtrtri_upper(lu):
    """Alg 3 line 2: inverse of the upper triangle of lu (zeros below)."""
    lu = _f64(lu)
    n = lu.shape[0]
    x = np.empty_like(lu)
    info = lib().or_dtrtri_upper(n, _p(lu), _p(x))
    return x, info


def dgetri_solve(lu, w):
    """Alg 3 line 3: X with X L = W (L = unit lower triangle of lu)."""
    lu, w = _f64(lu), _f64(w)
    x = np.empty_like(w)
    lib().or_dgetri_solve(lu.shape[0], _p(lu), _p(w), _p(x))
    return x


def dinv(a):
    """Alg 3: real inverse via LU.  Returns (ainv, info, rho)."""
    a = _f64(a)
    n = a.shape[0]
    x = np.zeros_like(a)
    rho = ctypes.c_double(0.0)
    info = lib().or_dinv(n, _p(a), _p(x), ctypes.byref(rho))
    return x, info, rho.value


def dgemm(a, b):
    """m_{n,R}: plain triple-loop product."""
    a, b = _f64(a), _f64(b)
    m, k = a.shape
    k2, n = b.shape
    assert k == k2
    c = np.empty((m, n), dtype=np.float64)
    lib().or_dgemm(m, n, k, _p(a), _p(b), _p(c))
    return c


# --------------------------------------------------------------- complex inverses
def split(z):
    z = np.asarray(z)
    return _f64(z.real), _f64(z.imag)


def frob_inv(z, branch: str = "auto", kappa_sw: float = KAPPA_SWITCH):
    """Alg 1.  Returns (X complex128, status, info dict).

    status: 0 ok, 1 singular (info['info'] = 1-based column), 2 both parts singular.
    """
    a, b = split(z)
    n = a.shape[0]
    xr = np.zeros_like(a)
    xi = np.zeros_like(a)
    out = np.zeros(2, dtype=np.int32)
    rho = np.zeros(4, dtype=np.float64)
    st = lib().or_frob_inv(n, _p(a), _p(b), _p(xr), _p(xi), BRANCH[branch], float(kappa_sw),
                           _p(out, ctypes.c_int), _p(rho))
    x = xr + 1j * xi
    return x, st, {"info": int(out[0]), "branch_used": int(out[1]), "rho_a": float(rho[0]), "rho_b": float(rho[1]),
                   "kappa_a": float(rho[2]), "kappa_b": float(rho[3])}


def frob_inv_rand(z, mu: float, kappa_sw: float = KAPPA_SWITCH):
    """Alg 5 with the random mu given: Z^{-1} = (1 + mu i) (Z (1 + mu i))^{-1}.

    Returns (X complex128, status, info dict) as frob_inv (status of the inner Alg 1 call).
    """
    a, b = split(z)
    n = a.shape[0]
    xr = np.zeros_like(a)
    xi = np.zeros_like(a)
    out = np.zeros(2, dtype=np.int32)
    rho = np.zeros(4, dtype=np.float64)
    st = lib().or_frob_inv_rand(n, _p(a), _p(b), float(mu), _p(xr), _p(xi), float(kappa_sw),
                                _p(out, ctypes.c_int), _p(rho))
    return xr + 1j * xi, st, {"info": int(out[0]), "branch_used": int(out[1]), "rho_a": float(rho[0]),
                              "rho_b": float(rho[1]), "kappa_a": float(rho[2]), "kappa_b": float(rho[3])}


def dpotrf_upper(a):
    """Alg 10: A = U^T U, U upper.  Returns (U, info)."""
    a = _f64(a)
    u = np.zeros_like(a)
    info = lib().or_dpotrf_upper(a.shape[0], _p(a), _p(u))
    return u, info


def hpd_frob_inv(z):
    """Alg 6 for Hermitian positive definite Z.  Returns (X, status, col)."""
    a, b = split(z)
    xr = np.zeros_like(a)
    xi = np.zeros_like(a)
    col = np.zeros(1, dtype=np.int32)
    st = lib().or_hpd_frob_inv(a.shape[0], _p(a), _p(b), _p(xr), _p(xi), _p(col, ctypes.c_int))
    return xr + 1j * xi, st, int(col[0])


def zhpd_inv_chol(z):
    """Alg 8 over C: complex Cholesky inversion X = U^{-1} U^{-H}.  Returns (X, info)."""
    re, im = split(z)
    xr = np.zeros_like(re)
    xi = np.zeros_like(im)
    info = lib().or_zhpd_inv_chol(re.shape[0], _p(re), _p(im), _p(xr), _p(xi))
    return xr + 1j * xi, info


def zinv_gj(z):
    """Complex inverse by Gauss-Jordan with partial pivoting (the plain definition)."""
    re, im = split(z)
    re, im = re.copy(), im.copy()
    info = lib().or_zinv_gj(re.shape[0], _p(re), _p(im))
    return re + 1j * im, info


def zinv_lu(z):
    """Alg 3 over C (the paper's comparator)."""
    re, im = split(z)
    xr = np.zeros_like(re)
    xi = np.zeros_like(im)
    info = lib().or_zinv_lu(re.shape[0], _p(re), _p(im), _p(xr), _p(xi))
    return xr + 1j * xi, info


def zgetrf(z):
    """Alg 3 line 1 over C: P Z = L U.  Returns (lu_re, lu_im, ipiv, info), planar."""
    re, im = split(z)
    re, im = re.copy(), im.copy()
    n = re.shape[0]
    ipiv = np.zeros(max(n, 1), dtype=np.int32)
    info = lib().or_zgetrf(n, _p(re), _p(im), _p(ipiv, ctypes.c_int))
    return re, im, ipiv[:n], info


def zgetrs(fac, r, trans: bool = False):
    """Y = Z^{-1} R (trans=False) or Z^{-H} R (trans=True) from zgetrf's factors; R (n, k) or (n,)."""
    lr, li, ipiv, _ = fac
    r = np.asarray(r)
    vec = r.ndim == 1
    r2 = r.reshape(r.shape[0], -1)
    yr, yi = _f64(r2.real).copy(), _f64(np.imag(r2)).copy()
    n, k = yr.shape
    lib().or_zgetrs(n, _p(lr), _p(li), _p(np.ascontiguousarray(ipiv, dtype=np.int32), ctypes.c_int),
                    1 if trans else 0, k, _p(yr), _p(yi))
    y = yr + 1j * yi
    return y[:, 0] if vec else y


def zsolve(z, r):
    """Z^{-1} R by Gaussian elimination with partial pivoting (or_zgetrf + or_zgetrs)."""
    fac = zgetrf(z)
    if fac[3]:
        raise np.linalg.LinAlgError(f"singular at column {fac[3]}")
    return zgetrs(fac, r)


def kappa2(z, fac=None, iters: int = 30, block: int = 16, seed: int = 12345):
    """Estimate of kappa_2(Z) = sigma_max / sigma_min (reading R10 / SURVEY G7).

    Block subspace iteration with Rayleigh-Ritz (block size `block`): sigma_max^2 = largest
    eigenvalue of Z^H Z (numpy matvecs), 1 / sigma_min^2 = largest eigenvalue of
    (Z^H Z)^{-1} = Z^{-1} Z^{-H} (applied through zgetrs).  A block converges at the rate of the
    ratio to the (block+1)-th singular value, so the clustered small singular values of random
    matrices do not stall it.  Ritz values approach from below: the returned kappa is (up to
    convergence) a lower bound of the true one.  Returns (kappa, sigma_max, sigma_min)."""
    z = np.asarray(z, dtype=np.complex128)
    n = z.shape[0]
    k = max(1, min(block, n))
    fac = fac if fac is not None else zgetrf(z)
    rng = np.random.default_rng(seed)

    def top_eig(apply):
        q, _ = np.linalg.qr(rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k)))
        for _ in range(iters):
            q, _ = np.linalg.qr(apply(q))
        t = q.conj().T @ apply(q)
        return float(np.linalg.eigvalsh(0.5 * (t + t.conj().T)).max())

    smax = math.sqrt(top_eig(lambda v: z.conj().T @ (z @ v)))
    lam = top_eig(lambda v: zgetrs(fac, zgetrs(fac, v, trans=True)))
    smin = 1.0 / math.sqrt(lam) if lam > 0 else 0.0
    return (smax / smin if smin > 0 else float("inf")), smax, smin


def frob_inv_many(zs, branch: str = "auto", kappa_sw: float = KAPPA_SWITCH):
    """or_frob_inv on each matrix of zs (count, n, n), in parallel over matrices.

    Returns (X (count, n, n), status int32[count], info int32[count], branch_used int32[count],
    rho (count, 4) = (rho_A, rho_B, kappa_inf(A), kappa_inf(B)))."""
    zs = np.asarray(zs)
    count, n = zs.shape[0], zs.shape[1]
    a, b = _f64(zs.real), _f64(zs.imag)
    xr = np.zeros_like(a)
    xi = np.zeros_like(a)
    out = np.zeros((count, 2), dtype=np.int32)
    rho = np.zeros((count, 4), dtype=np.float64)
    st = np.zeros(count, dtype=np.int32)
    lib().or_frob_inv_many(count, n, _p(a), _p(b), _p(xr), _p(xi), BRANCH[branch], float(kappa_sw),
                           _p(out, ctypes.c_int), _p(rho), _p(st, ctypes.c_int))
    return xr + 1j * xi, st, out[:, 0].copy(), out[:, 1].copy(), rho


def inverse(z, method: str = "frobenius"):
    if method in ("frobenius", "frob"):
        x, st, _ = frob_inv(z)
        if st:
            raise np.linalg.LinAlgError(f"frob_inv status {st}")
        return x
    x, info = zinv_lu(z) if method == "zlu" else zinv_gj(z)
    if info:
        raise np.linalg.LinAlgError(f"singular at column {info}")
    return x


# --------------------------------------------------------------- Newton drivers
def sign_newton(z, tol: float = 1e-12, max_iter: int = 50, method: str = "frobenius"):
    """X_{t+1} = (X_t + X_t^{-1})/2, X_0 = Z.

    Stop when delta_t = ||X_{t+1}-X_t||_F / ||X_{t+1}||_F < tol (BASELINE config 4,
    DESIGN.md reading R6) or after max_iter steps; at least one step.
    Returns (S, iters, deltas).
    """
    x = np.array(z, dtype=np.complex128)
    deltas = []
    for _ in range(max_iter):
        xn = 0.5 * (x + inverse(x, method))
        d = np.linalg.norm(xn - x) / np.linalg.norm(xn)
        deltas.append(float(d))
        x = xn
        if d < tol:
            break
    return x, len(deltas), deltas


def polar_newton(a, tol: float = 1e-12, max_iter: int = 50, method: str = "frobenius"):
    """X_{t+1} = (X_t + X_t^{-*})/2, X_0 = A; H = (U^H A + (U^H A)^H)/2."""
    x = np.array(a, dtype=np.complex128)
    deltas = []
    for _ in range(max_iter):
        xn = 0.5 * (x + inverse(x, method).conj().T)
        d = np.linalg.norm(xn - x) / np.linalg.norm(xn)
        deltas.append(float(d))
        x = xn
        if d < tol:
            break
    h = x.conj().T @ np.asarray(a, dtype=np.complex128)
    h = 0.5 * (h + h.conj().T)
    return x, h, len(deltas), deltas


def sylvester_sign(a, b, c, tol: float = 1e-12, max_iter: int = 50, method: str = "frobenius"):
    """A X + X B = C via the matrix sign function: for sign(A) = I, sign(B) = I,
    sign([[A, -C], [0, -B]]) = [[I, -2X], [0, -I]].  Newton X_{t+1} = (X_t + X_t^{-1})/2 from
    X_0 = [[A, -C], [0, -B]] (sign_newton above); X = -S_12 / 2.  Returns (X, iters, deltas)."""
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    c = np.asarray(c, dtype=np.complex128)
    m, n = a.shape[0], b.shape[0]
    t = np.zeros((m + n, m + n), dtype=np.complex128)
    t[:m, :m] = a
    t[:m, m:] = -c
    t[m:, m:] = -b
    s, it, d = sign_newton(t, tol=tol, max_iter=max_iter, method=method)
    return -0.5 * s[:m, m:], it, d


def lyapunov_sign(a, c, tol: float = 1e-12, max_iter: int = 50, method: str = "frobenius"):
    """A X + X A^* = C: the Sylvester solver with B = A^*."""
    a = np.asarray(a, dtype=np.complex128)
    return sylvester_sign(a, a.conj().T, c, tol, max_iter, method)


# --------------------------------------------------------------- metrics
def max_norm(z) -> float:
    """||A + iB||_max = max(||A||_max, ||B||_max)."""
    z = np.asarray(z)
    return float(max(np.abs(z.real).max(initial=0.0), np.abs(z.imag).max(initial=0.0)))


def res_lr(z, x):
    """Left/right relative residuals in the max norm."""
    z = np.asarray(z, dtype=np.complex128)
    x = np.asarray(x, dtype=np.complex128)
    n = z.shape[0]
    eye = np.eye(n)
    den = max_norm(z) * max_norm(x)
    return max_norm(x @ z - eye) / den, max_norm(z @ x - eye) / den


def rel_fro(x, ref) -> float:
    return float(np.linalg.norm(np.asarray(x) - np.asarray(ref)) / np.linalg.norm(ref))


def residual_fro(z, x) -> float:
    z = np.asarray(z, dtype=np.complex128)
    return float(np.linalg.norm(z @ np.asarray(x) - np.eye(z.shape[0])))
