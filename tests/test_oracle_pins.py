"""Pins for the CPU oracle (oracle/): it is checked against things other than itself.

- exact rational brute force over Q(i) (tests/golden/exact_inverses.json, written by
  tests/golden/make_golden.py from oracle/exact.py),
- closed forms (n=1 reduction P:L218, 2x2 adjugate, diagonal, unitary inputs,
  SPEC trivial cases in tests/golden/closed_forms.json),
- structural special cases (B=0, A=0, both parts singular),
- invariants (P A = L U, Z X = I, two-branch agreement, branch-B rotation),
- LAPACK (numpy) as an independent library reference for the real kernels.
A plausible slip (dropped term, wrong sign, transposed operand, wrong branch output
order, wrong pivot un-swap) fails at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import exact

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U = 2.0 ** -53


def _dec(m):
    from fractions import Fraction
    return np.array([[complex(float(Fraction(a)), float(Fraction(b))) for a, b in r] for r in m])


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _cm(rows):
    return np.array([[complex(a, b) for a, b in r] for r in rows])


# ------------------------------------------------------------------ exact brute force
@pytest.mark.parametrize("case", _gold("exact_inverses.json")["cases"],
                         ids=lambda c: f"n{c['n']}")
def test_exact_golden(case):
    z = np.array(case["re"], float) + 1j * np.array(case["im"], float)
    ref = _dec(case["inv"])
    kap = np.linalg.cond(z)
    tol = 50 * case["n"] * U * kap * max(1.0, kap)
    x, info = oracle.zinv_gj(z)
    assert info == 0
    assert oracle.rel_fro(x, ref) <= tol
    xl, info = oracle.zinv_lu(z)
    assert info == 0 and oracle.rel_fro(xl, ref) <= tol
    for br in ("a", "b"):
        if case["frob_" + br] is None:
            continue
        # Lemma 4.1 in exact arithmetic: Alg 1 equals the exact inverse exactly.
        assert case["frob_" + br] == case["inv"]
        xf, st, inf = oracle.frob_inv(z, br)
        if st == 0:
            kx = np.linalg.cond(z.real if br == "a" else z.imag)
            assert oracle.rel_fro(xf, ref) <= 100 * case["n"] * U * kap * kx * kx + tol


def test_exact_alg1_matches_definition_random():
    """Alg 1 over Q(i), both branches, equals Gauss-Jordan over Q(i) (fresh draws)."""
    rng = np.random.default_rng(7)
    for n in (2, 3, 4):
        re = rng.integers(-3, 4, size=(n, n))
        im = rng.integers(-3, 4, size=(n, n))
        z = exact.from_ints(re.tolist(), im.tolist())
        try:
            zi = exact.inv_exact(z)
            fa = exact.frobenius_exact(z, "a")
            fb = exact.frobenius_exact(z, "b")
        except ZeroDivisionError:
            continue
        assert fa == zi and fb == zi


# ------------------------------------------------------------------ closed forms
def test_closed_forms_golden():
    g = _gold("closed_forms.json")
    for c in g["complex_inverse"]:
        z, ref = _cm(c["z"]), _cm(c["inv"])
        for fn in (lambda q: oracle.zinv_gj(q)[0], lambda q: oracle.zinv_lu(q)[0],
                   lambda q: oracle.frob_inv(q)[0]):
            np.testing.assert_allclose(fn(z), ref, rtol=0, atol=1e-15, err_msg=c["cite"])
    for c in g["upper_triangular_inverse"]:
        x, info = oracle.dtrtri_upper(np.array(c["u"], float))
        np.testing.assert_allclose(x, np.array(c["inv"]), rtol=1e-15, atol=0)


def test_n1_reduction_all_branches():
    """for n = 1, Alg 1 is the scalar (a+ib)^{-1} = (a-ib)/(a^2+b^2)."""
    for a, b in [(3.0, 4.0), (-1.5, 0.25), (1e-3, 7.0), (2.0, -2.0)]:
        ref = complex(a, -b) / (a * a + b * b)
        z = np.array([[complex(a, b)]])
        for br in ("a", "b", "auto"):
            x, st, _ = oracle.frob_inv(z, br)
            assert st == 0
            assert abs(x[0, 0] - ref) <= 4 * U * abs(ref)


def test_2x2_adjugate():
    rng = np.random.default_rng(3)
    for _ in range(20):
        z = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
        det = z[0, 0] * z[1, 1] - z[0, 1] * z[1, 0]
        ref = np.array([[z[1, 1], -z[0, 1]], [-z[1, 0], z[0, 0]]]) / det
        kap = np.linalg.cond(z)
        for x in (oracle.zinv_gj(z)[0], oracle.zinv_lu(z)[0], oracle.frob_inv(z, "auto")[0]):
            assert oracle.rel_fro(x, ref) <= 1e-13 * kap * kap


def test_diagonal():
    d = np.array([1 + 2j, -3 + 0.5j, 0.25 - 4j, 5 + 5j, -2 - 1j])
    z = np.diag(d)
    ref = np.diag(1 / d)
    for x in (oracle.zinv_gj(z)[0], oracle.zinv_lu(z)[0], oracle.frob_inv(z, "a")[0],
              oracle.frob_inv(z, "b")[0]):
        np.testing.assert_allclose(x, ref, rtol=4e-16 * 8, atol=0)


def test_unitary_phase():
    """Z = Q e^{i theta} with Q real orthogonal: Z^{-1} = e^{-i theta} Q^T (both A, B invertible)."""
    n = 16
    q, _ = np.linalg.qr(np.random.default_rng(1).standard_normal((n, n)))
    for th in (0.3, 1.1, 2.5):
        z = q * np.exp(1j * th)
        ref = np.exp(-1j * th) * q.T
        for br in ("a", "b", "auto"):
            x, st, _ = oracle.frob_inv(z, br)
            assert st == 0
            assert oracle.rel_fro(x, ref) <= 1e-13 / min(abs(math.cos(th)), abs(math.sin(th))) ** 2
        assert oracle.rel_fro(oracle.zinv_gj(z)[0], ref) <= 1e-14


# ------------------------------------------------------------------ special structure
def test_b_zero_is_real_inverse_bitwise():
    a, _ = synth.gauss_pair(24, seed=5)
    z = a + 0j
    x, st, info = oracle.frob_inv(z, "auto")
    ainv, i2, _ = oracle.dinv(a)
    assert st == 0 and info["branch_used"] == 1
    assert np.array_equal(x.real, ainv)
    assert not np.any(x.imag)


def test_a_zero_takes_branch_b():
    _, b = synth.gauss_pair(24, seed=6)
    z = 1j * b
    x, st, info = oracle.frob_inv(z, "auto")
    binv, _, _ = oracle.dinv(b)
    assert st == 0 and info["branch_used"] == 2
    assert not np.any(x.real)
    assert np.array_equal(x.imag, -binv)


def test_both_parts_singular_dft():
    z = synth.dft_unitary(8)
    _, st, _ = oracle.frob_inv(z, "auto")
    assert st == 2
    x, info = oracle.zinv_gj(z)
    assert info == 0 and oracle.rel_fro(x, z.conj().T) <= 1e-14


def test_branch_b_is_rotated_branch_a():
    """S2 output (K - iJ) equals -i * S1-Alg1 applied to (B, -A) bitwise."""
    z = synth.shifted_complex(20, seed=11, shift=6.0)
    xb, st, _ = oracle.frob_inv(z, "b")
    xa_rot, st2, _ = oracle.frob_inv(z.imag - 1j * z.real, "a")
    assert st == 0 and st2 == 0
    assert np.array_equal(xb, -1j * xa_rot)


# ------------------------------------------------------------------ Alg 5 (randomized)
def test_exact_alg5_matches_definition_including_both_singular():
    """Alg 5 over Q(i) with rational mu equals the exact inverse, also where Alg 1 cannot run:
    Z = [[1, i], [i, 1]] has A = I but B = [[0,1],[1,0]]; Z = [[1+i, 1-i],[1-i, 1+i]] has A and B
    both singular (rank 1) while Z is invertible (det = 4i) -- Lemma 5.4."""
    cases = [([[1, 0], [0, 1]], [[0, 1], [1, 0]]), ([[1, 1], [1, 1]], [[1, -1], [-1, 1]])]
    rng = np.random.default_rng(5)
    for n in (3, 4):
        cases.append((rng.integers(-3, 4, size=(n, n)).tolist(), rng.integers(-3, 4, size=(n, n)).tolist()))
    from fractions import Fraction
    for re, im in cases:
        z = exact.from_ints(re, im)
        try:
            zi = exact.inv_exact(z)
        except ZeroDivisionError:
            continue
        for mu in (Fraction(1, 3), Fraction(5, 7)):
            assert exact.frobenius_rand_exact(z, mu) == zi
    # the both-singular example really defeats Alg 1 in both branches
    z = exact.from_ints(cases[1][0], cases[1][1])
    for br in ("a", "b"):
        with pytest.raises(ZeroDivisionError):
            exact.frobenius_exact(z, br)


def test_alg5_dft_both_singular_gives_unitary_inverse():
    """DFT/sqrt(n): A, B singular (AUTO Alg 1 -> status 2) but Alg 5 returns Z^{-1} = Z^H."""
    z = synth.dft_unitary(16)
    _, st, _ = oracle.frob_inv(z, "auto")
    assert st == 2
    x, st, info = oracle.frob_inv_rand(z, 0.6180339887)
    assert st == 0
    assert oracle.rel_fro(x, z.conj().T) <= 1e-13


def test_alg5_mu_zero_is_alg1_bitwise():
    z = synth.shifted_complex(24, seed=3, shift=6.0)
    x0, st0, _ = oracle.frob_inv(z, "auto")
    xr, st1, _ = oracle.frob_inv_rand(z, 0.0)
    assert st0 == 0 and st1 == 0
    assert np.array_equal(x0, xr)


def test_alg5_residual_and_rotation_identity():
    """Z X = I, and X equals (1 + mu i) times Alg 1 applied to (1 + mu i) Z (line 5)."""
    z = synth.shifted_complex(40, seed=9, shift=7.0)
    mu = 0.41
    x, st, _ = oracle.frob_inv_rand(z, mu)
    assert st == 0
    assert oracle.residual_fro(z, x) <= 1e-12 * 40
    w, st2, _ = oracle.frob_inv((1 + 1j * mu) * z, "auto")
    assert st2 == 0
    assert oracle.rel_fro(x, (1 + 1j * mu) * w) <= 1e-14


# ------------------------------------------------------------------ real kernels
def test_dgetrf_reconstruction_and_lapack_pivots():
    a, _ = synth.gauss_pair(40, seed=2, shift=0.0)
    lu, ipiv, info = oracle.dgetrf(a)
    assert info == 0
    n = a.shape[0]
    l = np.tril(lu, -1) + np.eye(n)
    u = np.triu(lu)
    pa = a.copy()
    for k in range(n):
        pa[[k, ipiv[k]]] = pa[[ipiv[k], k]]
    assert np.abs(pa - l @ u).max() <= 10 * n * U * np.abs(a).max() * 4
    assert np.abs(l).max() <= 1.0
    import scipy.linalg as sla
    lu2, piv2 = sla.lu_factor(a)
    assert np.array_equal(piv2, ipiv)
    np.testing.assert_allclose(lu, lu2, rtol=0, atol=1e-12)


def test_dgetrf_swap_example():
    lu, ipiv, info = oracle.dgetrf(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert list(ipiv) == [1, 1] and np.array_equal(lu, np.eye(2))


def test_dinv_3x3_adjugate_and_lapack():
    m = np.array([[4.0, -2.0, 1.0], [3.0, 6.0, -4.0], [2.0, 1.0, 8.0]])
    c = np.zeros((3, 3))
    for i in range(3):
        for j in range(3):
            minor = np.delete(np.delete(m, i, 0), j, 1)
            c[i, j] = (-1) ** (i + j) * (minor[0, 0] * minor[1, 1] - minor[0, 1] * minor[1, 0])
    det = float(np.dot(m[0], c[0]))
    adj = c.T / det
    x, info, rho = oracle.dinv(m)
    assert info == 0
    np.testing.assert_allclose(x, adj, rtol=1e-14, atol=1e-16)
    a, _ = synth.gauss_pair(50, seed=4)
    np.testing.assert_allclose(oracle.dinv(a)[0], np.linalg.inv(a), rtol=0, atol=1e-13)


def test_dgetri_solve_and_trtri():
    a, _ = synth.gauss_pair(30, seed=9)
    lu, ipiv, _ = oracle.dgetrf(a)
    w, info = oracle.dtrtri_upper(lu)
    assert info == 0
    np.testing.assert_allclose(w @ np.triu(lu), np.eye(30), atol=1e-13)
    assert not np.any(np.tril(w, -1))
    x = oracle.dgetri_solve(lu, w)
    l = np.tril(lu, -1) + np.eye(30)
    np.testing.assert_allclose(x @ l, w, atol=1e-13)


def test_dgemm_exact_integers():
    rng = np.random.default_rng(0)
    a = rng.integers(-50, 50, size=(13, 17)).astype(float)
    b = rng.integers(-50, 50, size=(17, 11)).astype(float)
    ref = (a.astype(np.int64) @ b.astype(np.int64)).astype(float)
    assert np.array_equal(oracle.dgemm(a, b), ref)


# ------------------------------------------------------------------ whole-method invariants
@pytest.mark.parametrize("n", [33, 64, 130])
def test_frob_vs_definition_config_style(n):
    z = synth.shifted_complex(n, seed=n, shift=8.0)
    xg, info = oracle.zinv_gj(z)
    assert info == 0
    for br in ("a", "b", "auto"):
        xf, st, _ = oracle.frob_inv(z, br)
        assert st == 0
        assert oracle.rel_fro(xf, xg) <= 1e-10
        assert oracle.residual_fro(z, xf) <= 1e-11 * n
    xl, info = oracle.zinv_lu(z)
    assert oracle.rel_fro(xl, xg) <= 1e-12
    np.testing.assert_allclose(xg, np.linalg.inv(z), rtol=0, atol=1e-12 * np.abs(xg).max())


def test_auto_switch_on_bad_a():
    """A nearly singular (kappa_inf(A) huge) -> AUTO takes branch B (R1')."""
    n = 12
    rng = np.random.default_rng(5)
    a = rng.standard_normal((n, n))
    a[:, 0] = a[:, 1] * (1 + 1e-9)
    b = rng.standard_normal((n, n)) + 4 * np.eye(n)
    x, st, info = oracle.frob_inv(a + 1j * b, "auto")
    assert st == 0 and info["branch_used"] == 2 and info["kappa_a"] > oracle.KAPPA_SWITCH * math.sqrt(n)
    assert info["kappa_b"] < info["kappa_a"]
    assert oracle.rel_fro(x, np.linalg.inv(a + 1j * b)) <= 1e-9


def test_auto_rule_kappa_inf_exact_and_switch_point():
    """R1': kappa_inf(X) = ||X||_inf ||X^{-1}||_inf of the part (checked against numpy's inverse);
    AUTO keeps S1 at or below the threshold and compares both parts above it."""
    z = synth.shifted_complex(40, seed=3, shift=9.0)
    x, st, info = oracle.frob_inv(z)
    ka = np.abs(z.real).sum(1).max() * np.abs(np.linalg.inv(z.real)).sum(1).max()
    assert st == 0 and info["branch_used"] == 1 and abs(info["kappa_a"] - ka) <= 1e-12 * ka
    assert np.isnan(info["kappa_b"])                      # B untouched below the threshold
    x2, st2, info2 = oracle.frob_inv(z, kappa_sw=0.5 * ka / math.sqrt(40))  # force the comparison
    kb = np.abs(z.imag).sum(1).max() * np.abs(np.linalg.inv(z.imag)).sum(1).max()
    assert abs(info2["kappa_b"] - kb) <= 1e-12 * kb
    assert info2["branch_used"] == (2 if kb < ka else 1)
    xb, _, _ = oracle.frob_inv(z, "b")
    assert np.array_equal(x2, xb if kb < ka else x)


def test_auto_rule_fixes_ill_conditioned_a_with_small_pivot_ratio():
    """Config-3 matrix 7639 (n = 128, seed 0 + index): LU(A)'s pivot ratio is only 230 (the round-1
    rule kept S1) but kappa_2(A) = 5.9e5, kappa_2(M) = 3.9e7 and S1's result is 2.2e-10 off the
    definition; R1' switches to S2 (kappa_inf(B) ~ 1e4), which is accurate."""
    z = synth.batch(128, 1, seed=0, start=7639)[0]
    ref, _ = oracle.zinv_gj(z)
    x, st, info = oracle.frob_inv(z)
    assert st == 0 and info["branch_used"] == 2 and info["kappa_a"] > oracle.KAPPA_SWITCH * math.sqrt(128)
    assert oracle.rel_fro(x, ref) <= 1e-11
    xa, _, _ = oracle.frob_inv(z, "a")
    assert oracle.rel_fro(xa, ref) > 1e-10


def test_paper_accuracy_generator_residuals():
    """P:L1076-1077 kappa=10 generator; Frobenius residuals stay within 50x of complex LU."""
    n = 64
    a = synth.hadamard_kappa(n, 10.0, seed=1)
    b = synth.hadamard_kappa(n, 10.0, seed=2)
    z = a + 1j * b
    xf, st, _ = oracle.frob_inv(z)
    xl, _ = oracle.zinv_lu(z)
    rf = max(oracle.res_lr(z, xf))
    rl = max(oracle.res_lr(z, xl))
    assert st == 0 and rf <= max(50 * rl, 1e-14)


# ------------------------------------------------------------------ Newton drivers
def test_sign_closed_forms():
    g = _gold("closed_forms.json")
    for c in g["sign"]:
        for m in ("frobenius", "zlu"):
            s, it, _ = oracle.sign_newton(np.array(c["z"], complex), method=m)
            np.testing.assert_allclose(s, np.array(c["s"], complex), atol=1e-15)
    for c in g["polar"]:
        u, h, it, _ = oracle.polar_newton(np.array(c["a"], complex))
        np.testing.assert_allclose(u, np.array(c["u"]), atol=1e-15)
        np.testing.assert_allclose(h, np.array(c["h"]), atol=1e-15)


def test_sign_newton_config4_small():
    z, s, lam, sinv = synth.sign_instance(48, seed=0)
    ref = (s * np.sign(lam.real)[None, :]) @ sinv
    for m in ("frobenius", "zlu"):
        x, it, d = oracle.sign_newton(z, tol=1e-12, max_iter=50, method=m)
        assert it < 50 and d[-1] < 1e-12
        assert oracle.rel_fro(x, ref) <= 1e-12
        assert np.abs(x @ x - np.eye(48)).max() <= 1e-11
        assert np.abs(x @ z - z @ x).max() <= 1e-10 * np.abs(z).max()


def test_polar_planted():
    n = 24
    rng = np.random.default_rng(2)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    c = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h0 = c.conj().T @ c + n * np.eye(n)
    a = q @ h0
    u, h, it, _ = oracle.polar_newton(a, tol=1e-13)
    assert oracle.rel_fro(u, q) <= 1e-12 and oracle.rel_fro(h, h0) <= 1e-12
    assert np.abs(u.conj().T @ u - np.eye(n)).max() <= 1e-13


# ------------------------------------------------------------------ Sylvester / Lyapunov (NEXT-3)
def test_sylvester_diagonal_closed_form():
    """Diagonal A, B: X_ij = C_ij / (a_i + b_j) (textbook closed form)."""
    rng = np.random.default_rng(21)
    m, n = 5, 4
    a = np.diag(1.0 + rng.random(m) + 1j * rng.standard_normal(m))
    b = np.diag(2.0 + rng.random(n) - 1j * rng.standard_normal(n))
    c = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    x, it, _ = oracle.sylvester_sign(a, b, c)
    ref = c / (np.diag(a)[:, None] + np.diag(b)[None, :])
    assert np.abs(x - ref).max() <= 1e-13 * np.abs(ref).max()


def test_sylvester_vs_kronecker_and_scipy():
    """Dense A, B with spectra in the right half plane: the sign-based X equals the
    Kronecker solve vec(X) = (I (x) A + B^T (x) I)^{-1} vec(C) and scipy's Bartels-Stewart."""
    import scipy.linalg as sla
    rng = np.random.default_rng(22)
    m, n = 6, 7
    a = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m)) + 6 * np.eye(m)
    b = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) + 6 * np.eye(n)
    c = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    x, it, _ = oracle.sylvester_sign(a, b, c)
    k = np.kron(np.eye(n), a) + np.kron(b.T, np.eye(m))
    xk = np.linalg.solve(k, c.reshape(-1, order="F")).reshape((m, n), order="F")
    assert oracle.rel_fro(x, xk) <= 1e-12
    assert oracle.rel_fro(x, sla.solve_sylvester(a, b, c)) <= 1e-12
    assert np.linalg.norm(a @ x + x @ b - c) <= 1e-12 * np.linalg.norm(c)
    x2, _, _ = oracle.sylvester_sign(a, b, c, method="zlu")
    assert oracle.rel_fro(x, x2) <= 1e-12


def test_lyapunov_hermitian_solution():
    """A X + X A^* = C with Hermitian C has a Hermitian solution (uniqueness)."""
    rng = np.random.default_rng(23)
    n = 8
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) + 7 * np.eye(n)
    c = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    c = c + c.conj().T
    x, _, _ = oracle.lyapunov_sign(a, c)
    assert np.linalg.norm(x - x.conj().T) <= 1e-12 * np.linalg.norm(x)
    assert np.linalg.norm(a @ x + x @ a.conj().T - c) <= 1e-12 * np.linalg.norm(c)


# ------------------------------------------------------------------ HPD (NEXT-4)
def test_dpotrf_vs_lapack_and_reconstruction():
    z = synth.hpd(40, seed=1)
    a = z.real.copy()
    u, info = oracle.dpotrf_upper(a)
    assert info == 0
    assert np.all(u[np.tril_indices(40, -1)] == 0.0)
    np.testing.assert_allclose(u, np.linalg.cholesky(a).T, rtol=1e-12, atol=1e-13)
    assert np.linalg.norm(u.T @ u - a) <= 1e-14 * np.linalg.norm(a)
    bad = a.copy()
    bad[5, 5] = -1.0
    assert oracle.dpotrf_upper(bad)[1] != 0


def test_hpd_2x2_closed_form():
    """Z = [[a, i b], [-i b, c]] (Hermitian): Z^{-1} = [[c, -i b], [i b, a]] / (a c - b^2)."""
    a, b, c = 3.0, 1.25, 2.0
    z = np.array([[a, 1j * b], [-1j * b, c]])
    ref = np.array([[c, -1j * b], [1j * b, a]]) / (a * c - b * b)
    for x, st in (oracle.hpd_frob_inv(z)[:2], oracle.zhpd_inv_chol(z)):
        assert st == 0
        assert np.abs(x - ref).max() <= 1e-15


def test_hpd_variants_vs_definition_and_alg1():
    """Alg 6 and Alg 8 against complex Gauss-Jordan, LAPACK and the LU-based Alg 1; lemma 6.1:
    A symmetric positive definite, B skew-symmetric."""
    for n in (3, 17, 64):
        z = synth.hpd(n, seed=n)
        assert np.array_equal(z.real, z.real.T) and np.array_equal(z.imag, -z.imag.T)
        ref, _ = oracle.zinv_gj(z)
        x6, st, _ = oracle.hpd_frob_inv(z)
        x8, st8 = oracle.zhpd_inv_chol(z)
        x1, st1, _ = oracle.frob_inv(z, "a")
        assert st == 0 and st8 == 0 and st1 == 0
        kap = np.linalg.cond(z)
        for x in (x6, x8, x1):
            assert oracle.rel_fro(x, ref) <= 1e-15 * kap * kap * n
            assert oracle.rel_fro(x, np.linalg.inv(z)) <= 1e-15 * kap * kap * n
        assert np.linalg.norm(x6 - x6.conj().T) <= 1e-12 * np.linalg.norm(x6)


def test_hpd_rejects_indefinite():
    z = synth.hpd(12, seed=3)
    z[0, 0] = -5.0
    _, st, col = oracle.hpd_frob_inv(z)
    assert st == 1 and col == 1
    assert oracle.zhpd_inv_chol(z)[1] == 1


# ------------------------------------------------------------------ solves used by sketch parity
def test_zgetrf_lapack_pivots_and_reconstruction():
    """or_zgetrf vs LAPACK zgetrf (scipy): same izamax (|re|+|im|) pivots, same factors to
    rounding, and P Z = L U."""
    import scipy.linalg as sl
    rng = np.random.default_rng(11)
    for n in (1, 2, 7, 64, 301):
        z = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        lr, li, ipiv, info = oracle.zgetrf(z)
        assert info == 0
        lu, piv = sl.lu_factor(z)
        assert np.array_equal(ipiv, piv)
        f = lr + 1j * li
        assert np.abs(f - lu).max() <= 1e-13 * n * np.abs(lu).max()
        lo = np.tril(f, -1) + np.eye(n)
        up = np.triu(f)
        pz = z.copy()
        for k in range(n):
            pz[[k, ipiv[k]]] = pz[[ipiv[k], k]]
        assert np.abs(lo @ up - pz).max() <= 1e-13 * n * np.abs(z).max()


def test_zgetrf_zero_pivot():
    z = np.array([[0, 0], [0, 1j]], dtype=np.complex128)
    assert oracle.zgetrf(z)[3] == 1


def test_zgetrs_closed_forms():
    """Diagonal: Y = R / d elementwise (one complex division per entry, exact up to the
    division's rounding); a permutation times a diagonal of powers of two (and i): exact."""
    rng = np.random.default_rng(3)
    n, k = 9, 4
    d = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    r = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    y = oracle.zgetrs(oracle.zgetrf(np.diag(d)), r)
    assert np.abs(y - r / d[:, None]).max() <= 4 * U * np.abs(r / d[:, None]).max()
    perm = rng.permutation(n)
    scal = (2.0 ** rng.integers(-3, 4, size=n)) * np.array([1, 1j, -1, -1j])[rng.integers(0, 4, size=n)]
    p = np.zeros((n, n), dtype=np.complex128)
    p[np.arange(n), perm] = scal
    # P Y = R  =>  Y[perm[i]] = R[i] / scal[i]
    y = oracle.zgetrs(oracle.zgetrf(p), r)
    ref = np.empty_like(r)
    ref[perm] = r / scal[:, None]
    assert np.array_equal(y, ref)
    yh = oracle.zgetrs(oracle.zgetrf(p), r, trans=True)
    assert np.array_equal(yh, np.linalg.solve(p.conj().T, r))  # exact: powers of two, permutation


def test_zgetrs_vs_gauss_jordan_and_residuals():
    """Y = Z^{-1} R agrees with the (independently pinned) Gauss-Jordan inverse times R, and both
    Z Y = R and Z^H Y' = R hold to rounding; also the exact rational inverse on an integer Z."""
    rng = np.random.default_rng(5)
    n, k = 120, 7
    z = synth.shifted_complex(n, 7, 0, 3.0 * math.sqrt(n))
    r = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    fac = oracle.zgetrf(z)
    y = oracle.zgetrs(fac, r)
    x, _ = oracle.zinv_gj(z)
    assert np.linalg.norm(y - x @ r) <= 1e-12 * np.linalg.norm(y)
    assert np.linalg.norm(z @ y - r) <= 1e-12 * np.linalg.norm(r)
    yh = oracle.zgetrs(fac, r, trans=True)
    assert np.linalg.norm(z.conj().T @ yh - r) <= 1e-12 * np.linalg.norm(r)
    assert np.linalg.norm(yh - x.conj().T @ r) <= 1e-12 * np.linalg.norm(yh)
    case = _gold("exact_inverses.json")["cases"][-1]
    ze = np.array(case["re"], float) + 1j * np.array(case["im"], float)
    ref = _dec(case["inv"])
    ye = oracle.zsolve(ze, np.eye(ze.shape[0]))
    kap = np.linalg.cond(ze)
    assert np.abs(ye - ref).max() <= 50 * ze.shape[0] * U * kap * max(1.0, kap) * np.abs(ref).max()


def test_kappa2_estimate_closed_forms():
    """kappa_2 of Q diag(s) W^H (Q, W unitary) is s_max / s_min; of a diagonal, max|d|/min|d|."""
    rng = np.random.default_rng(9)
    n = 80
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    w, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    s = np.linspace(1.0, 2.0, n)
    s[0], s[-1] = 0.01, 50.0      # isolated extremes: power iterations converge fast
    z = (q * s[None, :]) @ w.conj().T
    kap, smax, smin = oracle.kappa2(z)
    assert abs(smax - 50.0) <= 1e-6 * 50.0 and abs(smin - 0.01) <= 1e-6 * 0.01
    assert abs(kap - 5000.0) <= 1e-5 * 5000.0
    d = np.array([3.0, -0.5j, 2 + 2j, 7.0])
    assert abs(oracle.kappa2(np.diag(d))[0] - 14.0) <= 1e-9


def test_frob_inv_many_matches_single_calls_bitwise():
    zs = synth.batch(16, 12, seed=4)
    zs[3] = 0.0
    zs[3].imag = np.eye(16)             # A = 0: branch B
    x, st, info, bu, rho = oracle.frob_inv_many(zs)
    for i in range(zs.shape[0]):
        xi, sti, inf = oracle.frob_inv(zs[i])
        assert st[i] == sti and info[i] == inf["info"] and bu[i] == inf["branch_used"]
        assert np.array_equal(x[i], xi)
    assert bu[3] == 2


def test_auto_rule_threshold_from_the_error_calibration():
    """R1' threshold 2.5e4 (kappa_inf(A) / sqrt(n)): S1's error is up to ~2.6 u kappa_inf(A), so every
    part kept must have kappa_inf(A) <= 1e-10 / (2.6 u) = 3.5e5 at n = 128.  Config-3 matrix 487
    (kappa_2(Z) = 678, kappa_inf(A) = 6.2e5) sits between the old (8.8e4 sqrt(n) = 1.0e6) and the new
    switch point: AUTO now takes S2, which is accurate; S1 carries u kappa_inf(A)-sized error."""
    n = 128
    z = synth.batch(n, 1, seed=0, start=487)[0]
    ref, _ = oracle.zinv_gj(z)
    x, st, info = oracle.frob_inv(z)
    assert 1e-10 / (2.6 * 2.0 ** -53) > oracle.KAPPA_SWITCH * math.sqrt(n)
    assert st == 0 and info["branch_used"] == 2
    assert oracle.KAPPA_SWITCH * math.sqrt(n) < info["kappa_a"] < 8.8e4 * math.sqrt(n)
    assert oracle.rel_fro(x, ref) <= 1e-12
    xa, _, _ = oracle.frob_inv(z, "a")
    assert oracle.rel_fro(xa, ref) > 1e-12
