"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no Frobenius step, no LU, no
GEMM of the method).  It only draws random numbers and assembles the workloads
named in BASELINE.json ``configs``.  Both the
CPU oracle (``oracle/``) and the CUDA path consume the exact same bytes, which
are generated on the host.

Random numbers: numpy's counter-based Philox4x32-10 bit generator keyed with
``seed + (index << 64)`` (one independent stream per matrix index), normal
deviates from numpy's ``standard_normal``.  The key layout lets every rank of a
multi-GPU run generate only its own shard (configs 3-5) from (seed, global index).
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "rng_for", "gauss_pair", "shifted_complex", "config1", "config2", "batch",
    "sign_instance", "dft_unitary", "hadamard_kappa", "rademacher",
]


def rng_for(seed: int, index: int = 0, stream: int = 0) -> np.random.Generator:
    """Independent Philox stream for (seed, matrix index, sub-stream)."""
    key = (int(seed) & ((1 << 64) - 1)) | ((int(index) & ((1 << 48) - 1)) << 64) \
        | ((int(stream) & 0xFFFF) << 112)
    return np.random.Generator(np.random.Philox(key=key))


def gauss_pair(n: int, seed: int, index: int = 0, shift: float | None = 8.0):
    """A = G1 + shift*I, B = G2 with G1, G2 iid N(0,1) (BASELINE configs 1-3, 5).

    Returns two C-contiguous float64 (n, n) arrays.
    """
    rng = rng_for(seed, index)
    g1 = rng.standard_normal((n, n))
    g2 = rng.standard_normal((n, n))
    if shift:
        g1[np.diag_indices(n)] += shift
    return g1, g2


def shifted_complex(n: int, seed: int, index: int = 0, shift: float | None = 8.0) -> np.ndarray:
    """Z = A + iB as interleaved complex128 (row-major, the ABI layout)."""
    a, b = gauss_pair(n, seed, index, shift)
    z = np.empty((n, n), dtype=np.complex128)
    z.real = a
    z.imag = b
    return z


def config1() -> np.ndarray:
    """BASELINE config 1: n=64, A = G1 + 8I, B = G2, seed 0."""
    return shifted_complex(64, 0, 0, 8.0)


def config2(n: int = 1024, seed: int = 0) -> np.ndarray:
    """BASELINE configs 2 and 5: A = G1 + sqrt(n) I, B = G2."""
    return shifted_complex(n, seed, 0, math.sqrt(n))


def batch(n: int, count: int, seed: int = 0, start: int = 0, shift: float = 8.0) -> np.ndarray:
    """BASELINE config 3: matrices start..start+count-1, each 'as in config 1' from seed+index.

    Returns a C-contiguous complex128 array of shape (count, n, n).
    """
    out = np.empty((count, n, n), dtype=np.complex128)
    diag = np.diag_indices(n)
    for i in range(count):
        rng = rng_for(seed, start + i)
        g = rng.standard_normal((2, n, n))
        g[0][diag] += shift
        out[i].real = g[0]
        out[i].imag = g[1]
    return out


def sign_instance(n: int, seed: int = 0, index: int = 0):
    """BASELINE config 4 input: Z = S diag(lam) S^-1, S = I + 0.1 (G3 + i G4)/sqrt(n).

    Half of lam has real parts in -U[0.1, 10], half in +U[0.1, 10]; imaginary
    parts U[-5, 5].  Returns (Z, S, lam, Sinv).  S^-1 is obtained with numpy's
    LAPACK solver: it is input construction (identical bytes reach the oracle and
    the GPU), not the method under test, and kappa(S) ~ 1.5 keeps it exact to
    ~1e-15 (input recipe).
    """
    rng = rng_for(seed, index, stream=1)
    g3 = rng.standard_normal((n, n))
    g4 = rng.standard_normal((n, n))
    s = np.eye(n, dtype=np.complex128) + 0.1 * (g3 + 1j * g4) / math.sqrt(n)
    h = n // 2
    re = rng.uniform(0.1, 10.0, size=n)
    re[:h] *= -1.0
    im = rng.uniform(-5.0, 5.0, size=n)
    lam = re + 1j * im
    sinv = np.linalg.solve(s, np.eye(n, dtype=np.complex128))
    z = (s * lam[None, :]) @ sinv
    return np.ascontiguousarray(z), s, lam, sinv


def hpd(n: int, seed: int = 0, delta: float = 0.01) -> np.ndarray:
    """Hermitian positive definite test matrix in the style of the paper's HPD experiment
    ((A+iB)(A+iB)^* + 0.01 I): W = (G1 + i G2)/sqrt(n), Z = W W^* + delta I."""
    g = np.random.Generator(np.random.Philox(key=[seed, 0xB1D]))
    w = (g.standard_normal((n, n)) + 1j * g.standard_normal((n, n))) / math.sqrt(n)
    z = w @ w.conj().T + delta * np.eye(n)
    return 0.5 * (z + z.conj().T)


def dft_unitary(n: int) -> np.ndarray:
    """F/sqrt(n): unitary, with singular real and imaginary parts for n > 2."""
    j = np.arange(n)
    return np.exp(-2j * np.pi * np.outer(j, j) / n) / math.sqrt(n)


def hadamard_kappa(n: int, kappa: float = 10.0, seed: int = 0) -> np.ndarray:
    """The paper's accuracy generator: H D H^T scaled to unit Frobenius norm.

    n must be a power of two (Sylvester Hadamard).  D holds 1, kappa and n-2
    integers drawn from 1..kappa-1.
    """
    assert n >= 2 and (n & (n - 1)) == 0
    h = np.array([[1.0]])
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    rng = rng_for(seed, 0, stream=2)
    d = np.concatenate([[1.0, kappa], rng.integers(1, int(kappa), size=n - 2).astype(float)])
    m = (h * d[None, :]) @ h.T
    return m / np.linalg.norm(m)


def rademacher(n: int, k: int, seed: int = 0) -> np.ndarray:
    """+-1 sketch matrix (n, k) used for sketch parity at large n."""
    rng = rng_for(seed, 0, stream=3)
    return (rng.integers(0, 2, size=(n, k)) * 2 - 1).astype(np.float64)
