"""Exact rational arithmetic over Q and Q(i) -- TEST INFRASTRUCTURE ONLY.

Brute-force references for tiny integer inputs: exact Gauss-Jordan inverse over
Q(i) (the definition of Z^{-1}) and Alg 1 evaluated in exact
arithmetic, which must equal it *exactly* (Lemma 4.1).  Used to pin
the fp64 oracle (frob_oracle.c) and to write tests/golden/ fixtures.
Elements of Q(i) are pairs (Fraction re, Fraction im).
"""
from __future__ import annotations

from fractions import Fraction as Fr

ZERO = (Fr(0), Fr(0))
ONE = (Fr(1), Fr(0))


def cadd(a, b):
    return (a[0] + b[0], a[1] + b[1])


def csub(a, b):
    return (a[0] - b[0], a[1] - b[1])


def cmul(a, b):
    return (a[0] * b[0] - a[1] * b[1], a[0] * b[1] + a[1] * b[0])


def cinv(a):
    d = a[0] * a[0] + a[1] * a[1]
    if d == 0:
        raise ZeroDivisionError("singular")
    return (a[0] / d, -a[1] / d)


def from_ints(re, im):
    n = len(re)
    return [[(Fr(int(re[i][j])), Fr(int(im[i][j]))) for j in range(n)] for i in range(n)]


def inv_exact(m):
    """Gauss-Jordan over Q(i) (any nonzero pivot is exact).  Raises on singular."""
    n = len(m)
    a = [row[:] + [ONE if i == j else ZERO for j in range(n)] for i, row in enumerate(m)]
    for k in range(n):
        p = next((i for i in range(k, n) if a[i][k] != ZERO), None)
        if p is None:
            raise ZeroDivisionError("singular")
        a[k], a[p] = a[p], a[k]
        iv = cinv(a[k][k])
        a[k] = [cmul(v, iv) for v in a[k]]
        for i in range(n):
            if i != k and a[i][k] != ZERO:
                f = a[i][k]
                a[i] = [csub(v, cmul(f, w)) for v, w in zip(a[i], a[k])]
    return [row[n:] for row in a]


def matmul(x, y):
    n, k, m = len(x), len(y), len(y[0])
    out = []
    for i in range(n):
        row = []
        for j in range(m):
            s = ZERO
            for q in range(k):
                s = cadd(s, cmul(x[i][q], y[q][j]))
            row.append(s)
        out.append(row)
    return out


def madd(x, y):
    return [[cadd(a, b) for a, b in zip(r, s)] for r, s in zip(x, y)]


def real_part(m):
    return [[(v[0], Fr(0)) for v in r] for r in m]


def imag_part(m):
    return [[(v[1], Fr(0)) for v in r] for r in m]


def frobenius_exact(m, branch: str = "a"):
    """Alg 1 over Q(i) with tau = 1: returns J - iK (S1) or K - iJ (S2), exactly."""
    a, b = real_part(m), imag_part(m)
    x, y = (a, b) if branch == "a" else (b, a)
    xinv = inv_exact(x)
    f = matmul(xinv, y)
    mm = madd(x, matmul(y, f))
    j = inv_exact(mm)
    k = matmul(f, j)
    mi = (Fr(0), Fr(-1))  # -i
    if branch == "a":
        return [[cadd(jv, cmul(mi, kv)) for jv, kv in zip(jr, kr)] for jr, kr in zip(j, k)]
    return [[cadd(kv, cmul(mi, jv)) for jv, kv in zip(jr, kr)] for jr, kr in zip(j, k)]


def frobenius_rand_exact(m, mu):
    """Alg 5 over Q(i) for a rational mu: X = A - mu B, Y = mu A + B,
    W = Alg 1 (X + iY) (branch S1), return (W1 - mu W2) + i (mu W1 + W2)."""
    mu = Fr(mu)
    rot = [[(v[0] - mu * v[1], mu * v[0] + v[1]) for v in r] for r in m]
    w = frobenius_exact(rot, "a")
    return [[(v[0] - mu * v[1], mu * v[0] + v[1]) for v in r] for r in w]


def to_complex(m):
    import numpy as np
    return np.array([[complex(float(v[0]), float(v[1])) for v in r] for r in m])
