"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Tolerances (BASELINE north_star):
  ||X_gpu - X_oracle||_F / ||X_oracle||_F <= 1e-10   and   ||Z X_gpu - I||_F <= 1e-11 n
for kappa_2(Z) <= 1e4.  GEMM / LU building blocks are checked tighter (rounding order
differs only through FMA and blocking).  Bitwise invariants: conj(Z) -> conj(X),
2Z -> X/2, B = 0 -> real inverse, repeat-run determinism.
"""
import math

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
fb = pytest.importorskip("paper_2208_01239_b200")

REL = 1e-10
DEV = "cuda"


def _t(z):
    return torch.from_numpy(np.ascontiguousarray(z)).to(DEV)


def _np(t):
    return t.cpu().numpy()


def _resid(z, x):
    # independent library GEMM (torch complex128 matmul), not our kernels
    zt, xt = _t(z), _t(x)
    e = zt @ xt - torch.eye(z.shape[0], dtype=torch.complex128, device=DEV)
    return float(torch.linalg.norm(e))


def _check_inverse(z, x, ref=None, rel=REL):
    n = z.shape[0]
    if ref is None:
        ref, info = oracle.zinv_gj(z)
        assert info == 0
    r = oracle.rel_fro(x, ref)
    res = _resid(z, x)
    assert r <= rel, f"rel {r:.3e}"
    assert res <= 1e-11 * n, f"residual {res:.3e}"
    return r, res


# ------------------------------------------------------------------ building blocks
@pytest.mark.parametrize("mnk", [(1, 1, 1), (7, 5, 3), (37, 53, 29), (64, 64, 64), (130, 70, 200),
                                 (257, 129, 65), (512, 512, 512)])
def test_dgemm(mnk):
    m, n, k = mnk
    rng = np.random.default_rng(m * 7 + n)
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((k, n))
    c0 = rng.standard_normal((m, n))
    ref = oracle.dgemm(a, b)
    c = _np(fb.dgemm(_t(a), _t(b)))
    assert np.abs(c - ref).max() <= 1e-14 * k * np.abs(a).max() * np.abs(b).max() + 1e-300
    ct = _t(c0)
    fb.dgemm(_t(a), _t(b), ct, alpha=-0.5, beta=2.0)
    np.testing.assert_allclose(_np(ct), 2.0 * c0 - 0.5 * ref, rtol=0, atol=1e-13 * k)


def test_dgemm_exact_integers():
    rng = np.random.default_rng(1)
    a = rng.integers(-64, 64, size=(200, 300)).astype(float)
    b = rng.integers(-64, 64, size=(300, 150)).astype(float)
    assert np.array_equal(_np(fb.dgemm(_t(a), _t(b))), oracle.dgemm(a, b))


@pytest.mark.parametrize("n", [1, 2, 5, 33, 100, 257, 1000, 1536, 2100])
def test_dgetrf_reconstruction(n):
    # n = 1536 / 2100 (16-byte aligned rows): the blocked getrf with lu2's 32-column panel kernels
    # (one CTA, then clusters of up to 4 CTAs), single-level and two-level (n >= 2048)
    a, _ = synth.gauss_pair(n, seed=n, shift=0.0)
    lu, perm, info = fb.dgetrf(_t(a))
    lu, perm = _np(lu), _np(perm)
    assert sorted(perm.tolist()) == list(range(n))
    l = np.tril(lu, -1) + np.eye(n)
    u = np.triu(lu)
    assert np.abs(l).max() <= 1.0 + 1e-15  # partial pivoting: |l_ij| <= 1
    err = np.abs(a[perm] - l @ u).max()
    assert err <= 20 * n * 2.0 ** -53 * np.abs(a).max() * max(1.0, np.abs(u).max() / np.abs(a).max())
    # same pivots as the oracle (LAPACK order) when no near-ties: compare U diagonals
    lo, ipiv, _ = oracle.dgetrf(a)
    np.testing.assert_allclose(np.abs(np.diag(u)), np.abs(np.diag(lo)), rtol=1e-9)


@pytest.mark.parametrize("n", [1, 7, 64, 100, 255, 512])
def test_dinv(n):
    a, _ = synth.gauss_pair(n, seed=n + 1, shift=math.sqrt(n))
    ref, info, _ = oracle.dinv(a)
    x = _np(fb.dinv(_t(a)))
    assert oracle.rel_fro(x, ref) <= 1e-12 * max(1.0, np.linalg.cond(a))


# ------------------------------------------------------------------ frob_inv (single)
@pytest.mark.parametrize("n", [1, 2, 3, 16, 17, 64, 100, 256, 511, 512, 513, 1000, 1025])
@pytest.mark.parametrize("branch", ["auto", "a", "b"])
def test_frob_inv_small(n, branch):
    z = synth.shifted_complex(n, seed=100 + n, shift=math.sqrt(n) + 2.0)
    if branch == "b":
        z = z.imag * 0.5 + 1j * (z.real)  # make B the well-conditioned part
    x, info = fb.inv(_t(z), branch=branch, info=True)
    _check_inverse(z, _np(x))
    if branch != "auto":
        assert info["branch_used"] == (1 if branch == "a" else 2)


def test_config1_all_paths():
    """BASELINE config 1: n=64, both branches, AUTO, complex LU, batched kernel."""
    z = synth.config1()
    ref, _ = oracle.zinv_gj(z)
    for br in ("auto", "a", "b"):
        _check_inverse(z, _np(fb.inv(_t(z), branch=br)), ref)
        xb, inf, bu = fb.inv_batched(_t(z[None]), branch=br)
        assert int(inf[0]) == 0
        _check_inverse(z, _np(xb)[0], ref)
    _check_inverse(z, _np(fb.zinv(_t(z))), ref)
    xz, inf = fb.zinv_batched(_t(z[None]))
    _check_inverse(z, _np(xz)[0], ref)


def test_config2_full_size():
    """BASELINE config 2: n=1024 at full size, in the launch configuration bench.py times."""
    z = synth.config2(1024)
    ref, _ = oracle.zinv_gj(z)
    x, info = fb.inv(_t(z), info=True)
    _check_inverse(z, _np(x), ref)
    assert info["branch_used"] == 1 and info["info"] == 0
    _check_inverse(z, _np(fb.zinv(_t(z))), ref)
    # the oracle's Frobenius (Alg 1 literally) agrees too
    xo, st, _ = oracle.frob_inv(z)
    assert oracle.rel_fro(_np(x), xo) <= REL


@pytest.mark.parametrize("n", [1, 5, 8, 9, 31, 64, 129, 300, 513, 1000, 1025])
def test_zinv_lu(n):
    z = synth.shifted_complex(n, seed=7 * n, shift=3.0 + math.sqrt(n))
    _check_inverse(z, _np(fb.zinv(_t(z))))


@pytest.mark.parametrize("n", [1100, 1537, 2048])
def test_cluster_panel_sizes(n):
    """n > 1024: lu2 steps with more than 512 rows take the cluster panel (2..4 CTAs, DSMEM pivot
    exchange) and the look-ahead pipeline; Frobenius and complex LU against the oracle."""
    z = synth.shifted_complex(n, seed=31 * n, shift=math.sqrt(n) + 2.0)
    ref, _ = oracle.zinv_gj(z)
    x, info = fb.inv(_t(z), info=True)
    assert info["info"] == 0
    _check_inverse(z, _np(x), ref)
    _check_inverse(z, _np(fb.zinv(_t(z))), ref)


# ------------------------------------------------------------------ NEXT-1 fused first step
@pytest.mark.parametrize("n", [1, 2, 33, 256, 513, 1024, 2048])
@pytest.mark.parametrize("branch", ["auto", "b"])
def test_frob_inv_fused_first_step(n, branch):
    """C = U^{-1}(L^{-1}(P Y)) instead of X^{-1} Y: same oracle, same bounds; both LU paths."""
    z = synth.shifted_complex(n, seed=900 + n, shift=math.sqrt(n) + 2.0)
    if branch == "b":
        z = z.imag * 0.5 + 1j * z.real
    x, info = fb.inv(_t(z), branch=branch, info=True, fused=True)
    x = _np(x)
    if n <= 1024:
        _check_inverse(z, x)
    else:
        xo, st, _ = oracle.frob_inv(z, branch)
        assert st == 0 and oracle.rel_fro(x, xo) <= REL
        assert _resid(z, x) <= 1e-11 * n
    x_lit = _np(fb.inv(_t(z), branch=branch))
    assert oracle.rel_fro(x, x_lit) <= 1e-11  # two roundings of the same Alg 1 (kappa ~ 2e3 at n = 2048)


# ------------------------------------------------------------------ Alg 5 (randomized)
@pytest.mark.parametrize("n", [1, 7, 64, 300, 1024])
def test_frob_inv_rand_vs_oracle(n):
    """Alg 5 on the GPU vs the oracle's Alg 5 with the same mu, and vs the definition."""
    z = synth.shifted_complex(n, seed=500 + n, shift=math.sqrt(n) + 2.0)
    mu = fb.draw_mu(n)
    x = _np(fb.inv_rand(_t(z), mu=mu))
    xo, st, _ = oracle.frob_inv_rand(z, mu)
    assert st == 0
    assert oracle.rel_fro(x, xo) <= REL
    _check_inverse(z, x)


def test_frob_inv_rand_both_parts_singular():
    """DFT/sqrt(n): Alg 1 fails in both branches, Alg 5 returns Z^{-1} = Z^H."""
    for n in (16, 64, 256):
        z = synth.dft_unitary(n)
        with pytest.raises(fb.FrobError):
            fb.inv(_t(z))
        x = _np(fb.inv_rand(_t(z), seed=n))
        _check_inverse(z, x, ref=z.conj().T)


def test_frob_inv_rand_mu_zero_and_invalid():
    z = synth.shifted_complex(80, seed=8, shift=10.0)
    assert np.array_equal(_np(fb.inv_rand(_t(z), mu=0.0)), _np(fb.inv(_t(z))))
    with pytest.raises(fb.FrobError) as e:
        fb.inv_rand(_t(z), mu=1.5)
    assert e.value.name == "invalid_arg"


# ------------------------------------------------------------------ bitwise invariants
@pytest.mark.parametrize("n", [513, 1500, 2048])
def test_repeat_runs_bitwise_pipeline(n):
    """The look-ahead pipeline (cluster panels, NEXT / BULK updates synchronised by flags and
    programmatic launches) and the split-K GEMMs are deterministic: repeated calls agree bitwise
    (a race in the pipeline would not)."""
    zt = _t(synth.config2(n, seed=n))
    for f in (fb.inv, fb.zinv):
        ref = f(zt)
        for _ in range(3):
            assert torch.equal(f(zt), ref), (f.__name__, n)


def test_bitwise_invariants():
    z = synth.shifted_complex(200, seed=3, shift=16.0)
    x = _np(fb.inv(_t(z), branch="a"))
    x2 = _np(fb.inv(_t(z), branch="a"))
    assert np.array_equal(x, x2), "repeat-run determinism"
    xc = _np(fb.inv(_t(np.conj(z)), branch="a"))
    assert np.array_equal(xc, np.conj(x)), "conj(Z) -> conj(X)"
    xs = _np(fb.inv(_t(2.0 * z), branch="a"))
    assert np.array_equal(xs, x / 2.0), "2Z -> X/2"


def test_b_zero_and_a_zero():
    a, b = synth.gauss_pair(96, seed=4, shift=10.0)
    x, info = fb.inv(_t(a + 0j), info=True)
    x = _np(x)
    assert info["branch_used"] == 1
    assert not np.any(x.imag)
    assert np.array_equal(x.real, _np(fb.dinv(_t(a))))
    y, info = fb.inv(_t(1j * a), info=True)
    y = _np(y)
    assert info["branch_used"] == 2
    assert not np.any(y.real)
    np.testing.assert_allclose(y.imag, -x.real, rtol=0, atol=0)


def test_auto_switches_and_both_singular():
    n = 48
    rng = np.random.default_rng(5)
    a = rng.standard_normal((n, n))
    a[:, 0] = a[:, 1] * (1 + 1e-9)
    b = rng.standard_normal((n, n)) + 6 * np.eye(n)
    z = a + 1j * b
    x, info = fb.inv(_t(z), info=True)
    assert info["branch_used"] == 2 and info["kappa_a"] > 1e6 and info["kappa_b"] < info["kappa_a"]
    _check_inverse(z, _np(x), rel=1e-8)
    with pytest.raises(fb.FrobError) as e:
        fb.inv(_t(synth.dft_unitary(16)))
    assert e.value.name == "both_singular"
    xb, inf, bu = fb.inv_batched(_t(np.stack([z, synth.dft_unitary(n)])))
    assert int(bu[0]) == 2 and int(inf[0]) == 0
    assert int(bu[1]) == 0 and int(inf[1]) != 0


def test_nonfinite_and_invalid():
    z = synth.shifted_complex(32, seed=1)
    z[3, 4] = np.nan
    with pytest.raises(fb.FrobError) as e:
        fb.inv(_t(z))
    assert e.value.name == "nonfinite"
    zt = _t(synth.shifted_complex(32, seed=1))
    with pytest.raises(fb.FrobError) as e:
        fb.inv(zt, out=zt)
    assert e.value.name == "invalid_arg"


# ------------------------------------------------------------------ batched
@pytest.mark.parametrize("n", [1, 2, 17, 32, 50, 64, 65, 100, 128])
@pytest.mark.parametrize("branch", ["auto", "a", "b"])
def test_batched(n, branch):
    cnt = 24
    z = synth.batch(n, cnt, seed=9, shift=8.0)
    if branch == "b":
        z = z.imag * 0.5 + 1j * z.real
    x, inf, bu = fb.inv_batched(_t(z), branch=branch)
    x, inf, bu = _np(x), _np(inf), _np(bu)
    zinv_ok = n <= 128
    if zinv_ok:
        xz, infz = fb.zinv_batched(_t(z))
        xz = _np(xz)
    for i in range(cnt):
        ref, _ = oracle.zinv_gj(z[i])
        assert inf[i] == 0
        if branch != "auto":
            assert bu[i] == (1 if branch == "a" else 2)
        _check_inverse(z[i], x[i], ref)
        if zinv_ok:
            _check_inverse(z[i], xz[i], ref)


def test_batched_config3_n128_sample():
    """Config 3 (n=128 half): 2048 matrices checked by residual, a sample vs oracle; AUTO switches seen."""
    z = synth.batch(128, 2048, seed=0)
    x, inf, bu = fb.inv_batched(_t(z))
    zt = _t(z)
    e = torch.matmul(zt, x) - torch.eye(128, dtype=torch.complex128, device=DEV)
    res = torch.linalg.norm(e, dim=(1, 2)).cpu().numpy()
    bu = _np(bu)
    xs = _np(x)
    for i in range(0, 2048, 256):
        ref, _ = oracle.zinv_gj(z[i])
        assert oracle.rel_fro(xs[i], ref) <= REL
    assert int(inf.abs().sum()) == 0
    # kappa(A) is heavy-tailed at shift 8, n=128: residual bound on the well-posed ones
    kz = np.linalg.cond(z[:256])
    ok = kz <= 1e4
    assert np.all(res[:256][ok] <= 1e-11 * 128)


def test_batched_config3_n32_sample():
    """Config 3 (n=32 half) at full batch: every output checked via residual, a sample vs oracle."""
    z = synth.batch(32, 65536, seed=0)
    x, inf, bu = fb.inv_batched(_t(z))
    assert int(inf.abs().sum()) == 0
    zt = _t(z)
    e = torch.matmul(zt, x) - torch.eye(32, dtype=torch.complex128, device=DEV)
    res = torch.linalg.norm(e, dim=(1, 2))
    assert float(res.max()) <= 1e-11 * 32
    xs = _np(x[::4096])
    for k, i in enumerate(range(0, 65536, 4096)):
        ref, _ = oracle.zinv_gj(z[i])
        assert oracle.rel_fro(xs[k], ref) <= REL


# ------------------------------------------------------------------ Newton drivers
def test_sign_small_and_closed_form():
    z, s, lam, sinv = synth.sign_instance(64, seed=0)
    ref = (s * np.sign(lam.real)[None, :]) @ sinv
    for m in ("frobenius", "zlu"):
        st, it, d = fb.sign(_t(z), tol=1e-12, max_iter=50, method=m)
        st = _np(st)
        assert d < 1e-12 and it < 50
        assert oracle.rel_fro(st, ref) <= 1e-11
        so, ito, _ = oracle.sign_newton(z, method=m)
        assert oracle.rel_fro(st, so) <= 1e-11
        assert abs(it - ito) <= 1


def test_polar_small():
    n = 40
    rng = np.random.default_rng(2)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    c = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h0 = c.conj().T @ c + n * np.eye(n)
    a = q @ h0
    u, h, it, d = fb.polar(_t(a), tol=1e-13)
    u, h = _np(u), _np(h)
    assert oracle.rel_fro(u, q) <= 1e-11 and oracle.rel_fro(h, h0) <= 1e-11


# ------------------------------------------------------------------ full-size configs 4 and 5
def test_config4_sign_full_size():
    """BASELINE config 4 at full size (n=2048): Newton sign with Frobenius and with complex LU,
    against the closed form S sign(Re lambda) S^{-1} built from the generator's own S^{-1}."""
    z, s, lam, sinv = synth.sign_instance(2048, seed=0)
    ref = _t((s * np.sign(lam.real)[None, :]) @ sinv)
    zt = _t(z)
    eye = torch.eye(2048, dtype=torch.complex128, device=DEV)
    for m in ("frobenius", "zlu"):
        st, it, d = fb.sign(zt, tol=1e-12, max_iter=50, method=m)
        rel = float(torch.linalg.norm(st - ref) / torch.linalg.norm(ref))
        assert it < 50 and d < 1e-12, (m, it, d)
        assert rel <= 1e-10, (m, rel)
        # invariants with independent library GEMMs: S^2 = I, S Z = Z S
        assert float(torch.linalg.norm(st @ st - eye)) <= 1e-9
        assert float(torch.linalg.norm(st @ zt - zt @ st) / torch.linalg.norm(zt)) <= 1e-10


# config 5 at full size (n = 2048 ... 16384) against the oracle: tests/test_gpu_fullsize.py


# ------------------------------------------------------------------ Sylvester / Lyapunov (NEXT-3)
@pytest.mark.parametrize("mn", [(1, 1), (5, 3), (40, 24), (96, 96)])
@pytest.mark.parametrize("method", ["frobenius", "zlu"])
def test_sylvester_vs_oracle(mn, method):
    m, n = mn
    rng = np.random.default_rng(m * 100 + n)
    # spectra well inside the right half plane (complex Gaussian disc radius ~ sqrt(2 m)):
    # sign(A) = I, sign(B) = I as the block-sign formula requires
    a = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m)) + (3 + 2 * math.sqrt(2 * m)) * np.eye(m)
    b = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) + (3 + 2 * math.sqrt(2 * n)) * np.eye(n)
    c = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    x, it, d = fb.sylvester(_t(a), _t(b), _t(c), method=method)
    x = _np(x)
    xo, ito, _ = oracle.sylvester_sign(a, b, c, method="frobenius" if method == "frobenius" else "zlu")
    assert oracle.rel_fro(x, xo) <= REL
    assert np.linalg.norm(a @ x + x @ b - c) <= 1e-11 * np.linalg.norm(c) * max(m, n)
    assert abs(it - ito) <= 1


def test_lyapunov_gpu():
    n = 64
    rng = np.random.default_rng(64)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) + (3 + 2 * math.sqrt(2 * n)) * np.eye(n)
    c = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    c = c + c.conj().T
    x, it, d = fb.lyapunov(_t(a), _t(c))
    x = _np(x)
    xo, _, _ = oracle.lyapunov_sign(a, c)
    assert oracle.rel_fro(x, xo) <= REL
    assert np.linalg.norm(a @ x + x @ a.conj().T - c) <= 1e-11 * np.linalg.norm(c) * n
    assert np.linalg.norm(x - x.conj().T) <= 1e-11 * np.linalg.norm(x)


# ------------------------------------------------------------------ HPD (NEXT-4)
@pytest.mark.parametrize("n", [1, 2, 17, 64, 65, 100, 257, 1000])
def test_hpd_inv_vs_oracle(n):
    """Alg 6 and Alg 8 on the GPU vs the oracle's Alg 6 / Alg 8 and the definition."""
    z = synth.hpd(n, seed=n)
    ref, _ = oracle.zinv_gj(z)
    x6 = _np(fb.hpd_inv(_t(z)))
    x8 = _np(fb.zhpd_inv(_t(z)))
    _check_inverse(z, x6, ref)
    _check_inverse(z, x8, ref)
    if n <= 257:
        xo6, st, _ = oracle.hpd_frob_inv(z)
        xo8, st8 = oracle.zhpd_inv_chol(z)
        assert st == 0 and st8 == 0
        assert oracle.rel_fro(x6, xo6) <= REL and oracle.rel_fro(x8, xo8) <= REL


def test_hpd_not_positive_definite():
    z = synth.hpd(40, seed=4)
    z[7, 7] = -3.0
    for f in (fb.hpd_inv, fb.zhpd_inv):
        with pytest.raises(fb.FrobError) as e:
            f(_t(z))
        assert e.value.name == "singular"


@pytest.mark.parametrize("n", [1, 63, 64, 65, 200, 1000, 2100])
def test_dpoinv_vs_oracle(n):
    """Real SPD inversion (Alg 8 over R, T_pinv of Thm 6.2) vs the oracle's real inverse; the
    Cholesky's symmetric trailing update skips the tiles below the diagonal."""
    rng = np.random.default_rng(n)
    g = rng.standard_normal((n, n)) / math.sqrt(n)
    a = g @ g.T + 0.5 * np.eye(n)
    ref, info, _ = oracle.dinv(a)
    assert info == 0
    x = _np(fb.dpoinv(_t(a)))
    assert oracle.rel_fro(x, ref) <= 1e-12 * max(1.0, np.linalg.cond(a))
    a[n // 2, n // 2] = -1.0
    with pytest.raises(fb.FrobError) as e:
        fb.dpoinv(_t(a))
    assert e.value.name == "singular"


# ------------------------------------------------------------------ the paper's own generators
@pytest.mark.parametrize("n", [64, 512, 1024])
def test_paper_speed_generator_uniform(n):
    """E1's inputs: A, B with iid U(0,1) entries (no diagonal shift: kappa grows with n),
    AUTO Frobenius, NEXT-1 and complex LU against the oracle's Gauss-Jordan inverse; the bound is
    kappa-scaled (R10)."""
    rng = np.random.default_rng(1055 + n)
    z = rng.uniform(0.0, 1.0, (n, n)) + 1j * rng.uniform(0.0, 1.0, (n, n))
    ref, info = oracle.zinv_gj(z)
    assert info == 0
    kf = max(1.0, np.linalg.cond(z) / 1e4)
    zt = _t(z)
    for name, x in (("auto", fb.inv(zt)), ("fused", fb.inv(zt, fused=True)), ("zinv", fb.zinv(zt))):
        rel = oracle.rel_fro(_np(x), ref)
        assert rel <= 1e-10 * kf, (name, rel, kf)
        assert _resid(z, _np(x)) <= 1e-11 * n * kf


@pytest.mark.parametrize("n", [64, 256, 1024])
def test_paper_accuracy_generator_hadamard(n):
    """E2's inputs: A, B = H D H^T / ||.||_F with kappa = 10 (synth.hadamard_kappa),
    the paper's left / right residuals of GPU Frobenius vs GPU complex LU: both at
    rounding level, as the paper reports ("difference is so small")."""
    z = synth.hadamard_kappa(n, 10.0, seed=1) + 1j * synth.hadamard_kappa(n, 10.0, seed=2)
    ref, _ = oracle.zinv_gj(z)
    zt = _t(z)
    xf, xz = _np(fb.inv(zt)), _np(fb.zinv(zt))
    assert oracle.rel_fro(xf, ref) <= 1e-12 and oracle.rel_fro(xz, ref) <= 1e-12
    lf, rf = oracle.res_lr(z, xf)
    lz, rz = oracle.res_lr(z, xz)
    assert max(lf, rf, lz, rz) <= 1e-13 * n


@pytest.mark.parametrize("n", [300, 1030])
def test_alg5_both_singular_structured_large(n):
    """Alg 5 on a unitary Z = DFT/sqrt(n) at larger n (real and imaginary parts singular): Z^{-1} = Z^H;
    AUTO Alg 1 reports both parts singular."""
    z = synth.dft_unitary(n)
    zt = _t(z)
    with pytest.raises(fb.FrobError) as e:
        fb.inv(zt)
    assert e.value.name == "both_singular"
    x = _np(fb.inv_rand(zt, seed=7))
    assert oracle.rel_fro(x, z.conj().T) <= 1e-11
