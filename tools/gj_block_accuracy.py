"""Which blocked form the batched n = 128 sweep may use: numpy emulation of the exchange-form Gauss-Jordan
sweep unblocked and blocked (8-column panels swept in exchange form, or factored in LU form and
turned into the swept panel via U11^-1 L11^-1, then one rank-8 update of every other column), fed
to Alg 1 (S1) on the config-3 matrices with an ill-conditioned A, against the oracle's definition.
    python tools/gj_block_accuracy.py"""
import sys
import numpy as np

sys.path.insert(0, ".")
import oracle
import synth


def unscramble(a, piv):
    n = len(a)
    pos = np.empty(n, int)
    pos[np.array(piv)] = np.arange(n)
    inv = np.empty_like(a)
    inv[np.ix_(pos, np.array(piv))] = a
    return inv


def sweep_unblocked(A):
    a = A.copy()
    n = len(a)
    used = np.zeros(n, bool)
    piv = []
    for k in range(n):
        cand = np.where(~used)[0]
        p = cand[np.argmax(np.abs(a[cand, k]))]
        used[p] = True
        piv.append(p)
        ip = 1.0 / a[p, k]
        rp = a[p] * ip
        rp[k] = ip
        ck = a[:, k].copy()
        a[:, k] = 0
        a -= np.outer(ck, rp)
        a[p] = rp
    return unscramble(a, piv)


def sweep_blocked(A, w=8, luform=False):
    a = A.copy()
    n = len(a)
    used = np.zeros(n, bool)
    piv = []
    for k0 in range(0, n, w):
        K = list(range(k0, k0 + w))
        P = a[:, K].copy()
        rows = []
        if luform:
            pm = np.zeros(n, bool)
            for c in range(w):
                cand = np.where(~used)[0]
                p = cand[np.argmax(np.abs(P[cand, c]))]
                used[p] = pm[p] = True
                rows.append(p)
                u = P[p].copy()
                m = np.where(~pm, P[:, c] / u[c], 0.0)
                P[~pm, c] = m[~pm]
                P[:, c + 1:] -= np.outer(m, u[c + 1:])
            lu = P[rows]
            Linv = np.linalg.inv(np.tril(lu, -1) + np.eye(w))
            Pn = -P @ Linv
            Pn[rows] = np.linalg.inv(np.triu(lu)) @ Linv
        else:
            for c in range(w):
                cand = np.where(~used)[0]
                p = cand[np.argmax(np.abs(P[cand, c]))]
                used[p] = True
                rows.append(p)
                ip = 1.0 / P[p, c]
                rp = P[p] * ip
                rp[c] = ip
                ck = P[:, c].copy()
                P[:, c] = 0
                P -= np.outer(ck, rp)
                P[p] = rp
            Pn = P
        piv += rows
        J = [j for j in range(n) if j not in K]
        T = a[rows][:, J].copy()
        a[np.array(rows)[:, None], J] = 0
        a[:, J] += Pn @ T
        a[:, K] = Pn
    return unscramble(a, piv)


def sweep_blocked_subst(A, w=8):
    """The kernel's form: the other columns by substitution (W = L11^-1 T, V = U11^-1 W,
    A_IJ -= L21 W, A_RJ = V); the panel columns by the products with L11^-1 / U11^-1."""
    a = A.copy()
    n = len(a)
    used = np.zeros(n, bool)
    piv = []
    for k0 in range(0, n, w):
        K = list(range(k0, k0 + w))
        P = a[:, K].copy()
        rows = []
        pm = np.zeros(n, bool)
        for c in range(w):
            cand = np.where(~used)[0]
            p = cand[np.argmax(np.abs(P[cand, c]))]
            used[p] = pm[p] = True
            rows.append(p)
            u = P[p].copy()
            m = np.where(~pm, P[:, c] / u[c], 0.0)
            P[~pm, c] = m[~pm]
            P[:, c + 1:] -= np.outer(m, u[c + 1:])
        lu = P[rows]
        L = np.tril(lu, -1) + np.eye(w)
        U = np.triu(lu)
        J = [j for j in range(n) if j not in K]
        T = a[rows][:, J].copy()
        W = np.zeros_like(T)
        for c in range(w):
            W[c] = T[c] - L[c, :c] @ W[:c]
        V = np.zeros_like(W)
        for c in reversed(range(w)):
            V[c] = (W[c] - U[c, c + 1:] @ V[c + 1:]) / U[c, c]
        nonp = ~pm
        a[np.ix_(nonp, J)] -= P[nonp] @ W
        a[np.ix_(rows, J)] = V
        Linv = np.linalg.inv(L)
        newK = np.zeros((n, w))
        newK[nonp] = -P[nonp] @ Linv
        newK[rows] = np.linalg.inv(U) @ Linv
        a[:, K] = newK
        piv += rows
    return unscramble(a, piv)


def frob_s1(z, inv):
    A, B = z.real.copy(), z.imag.copy()
    C = inv(A) @ B
    Re = inv(A + B @ C)
    return Re - 1j * (C @ Re)


zz = synth.batch(128, 16384, seed=0)
print("matrix  kappa2(Z)  kappa_inf(A)  | S1 error vs the definition: oracle  unblocked  blocked(exchange)  "
      "blocked(LU form, products)  blocked(substitution form: the kernel)")
for idx in (487, 3568, 14129):
    z = zz[idx]
    ref, _ = oracle.zinv_gj(z)
    xo, _, info = oracle.frob_inv(z, "a")
    errs = [oracle.rel_fro(frob_s1(z, f), ref) for f in
            (sweep_unblocked, sweep_blocked, lambda A: sweep_blocked(A, luform=True), sweep_blocked_subst)]
    print(f"{idx:6d} {np.linalg.cond(z):10.1e} {info['kappa_a']:12.2e}  | {oracle.rel_fro(xo, ref):.2e}  "
          + "  ".join(f"{e:.2e}" for e in errs))
