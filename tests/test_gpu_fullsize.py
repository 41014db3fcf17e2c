"""Full-size oracle parity for BASELINE configs 3 and 5 (the sizes bench.py times).

Bar (BASELINE north_star): ||X_gpu - X_oracle||_F / ||X_oracle||_F <= 1e-10 and
||Z X_gpu - I||_F <= 1e-11 n for kappa_2(Z) <= 1e4.  Above 1e4 the north star is silent; the
reading taken (R10) scales both bounds by kappa_2(Z) / 1e4, i.e.
rel <= 1e-14 kappa_2(Z).  kappa_2(Z) per instance: config 5 from the committed oracle script
(tests/golden/make_sketch.py: power / inverse-power iteration through the oracle's LU),
config 3 from torch.linalg.svdvals (cuSOLVER, an independent library; it only picks the bound).

- config 5, n = 2048 / 4096: element by element against the oracle's complex Gauss-Jordan inverse
  (oracle.zinv_gj, the plain definition) computed in-test on the host cores;
- config 5, n = 8192 / 16384: sketch parity -- X_gpu R against X_oracle R, R the
  +-1 matrix synth.rademacher(n, 64), X_oracle R stored by tests/golden/make_sketch.py, which calls
  only oracle/ and synth/ (Gaussian elimination on the augmented system);
- the residual ||Z X - I||_F <= 1e-11 n (x kappa factor) with torch's complex GEMM, and sampled
  columns ||Z x_j - e_j|| in fp64 on the host (their RMS x sqrt(n) estimates the same residual);
- config 3: EVERY matrix (65536 x n=32, 16384 x n=128) against the oracle's Alg 1
  (oracle.frob_inv_many, the same AUTO rule R1), and the branch each side took.
The GPU calls are the bench's launch configuration (frob_inv AUTO / frob_inv_batched AUTO).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
fb = pytest.importorskip("paper_2208_01239_b200")

DEV = "cuda"
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _kfac(kappa):
    return max(1.0, kappa / 1e4)


def _sketch_meta():
    with open(os.path.join(GOLD, "sketch_config5.json")) as f:
        return json.load(f)


def _residuals(z, zt, x_dev, n, kf, seed):
    """The north-star residual ||Z X - I||_F <= 1e-11 n (x kappa factor), with an independent library
    GEMM (torch complex128), plus sampled columns ||Z x_j - e_j|| in fp64 on the host: their RMS
    times sqrt(n) estimates the same Frobenius residual (checked with a 1.5x sampling allowance)."""
    eye = torch.eye(n, dtype=torch.complex128, device=DEV)
    res = float(torch.linalg.norm(zt @ x_dev - eye))
    del eye
    assert res <= 1e-11 * n * kf, (n, res, 1e-11 * n * kf)
    rng = np.random.default_rng(seed)
    cols = rng.choice(n, size=8, replace=False)
    xs = x_dev[:, torch.from_numpy(cols).to(DEV)].cpu().numpy()
    rs = []
    for k, j in enumerate(cols):
        r = z @ xs[:, k]
        r[j] -= 1.0
        rs.append(float(np.linalg.norm(r)))
    est = math.sqrt(n * np.mean(np.square(rs)))
    assert est <= 1.5 * 1e-11 * n * kf, (n, est, rs)
    return res, max(rs)


@pytest.mark.parametrize("n", [2048, 4096])
def test_config5_elementwise_vs_oracle(n):
    """Element-wise parity against oracle.zinv_gj at n = 2048 / 4096 (config-5 generator, seed 0),
    for Frobenius (AUTO, the bench call), the NEXT-1 option and the complex-LU comparator."""
    z = synth.config2(n, seed=0)
    zt = torch.from_numpy(z).to(DEV)
    ref, info = oracle.zinv_gj(z)
    assert info == 0
    meta = _sketch_meta()
    kappa = meta[str(n)]["kappa2_est"] if str(n) in meta else float(np.linalg.cond(z))
    kf = _kfac(kappa)
    for name, f in (("frob", lambda: fb.inv(zt)), ("frob_fused", lambda: fb.inv(zt, fused=True)),
                    ("zinv_lu", lambda: fb.zinv(zt))):
        x = f()
        rel = oracle.rel_fro(x.cpu().numpy(), ref)
        assert rel <= 1e-10 * kf, (name, rel, kappa)
        _residuals(z, zt, x, n, kf, seed=n)


@pytest.mark.parametrize("n", [8192, 16384])
def test_config5_sketch_parity(n):
    """Sketch parity at n = 8192 / 16384: E||(X_gpu - X_or) R||_F^2 / k = ||X_gpu - X_or||_F^2 for a
    Rademacher R (k = 64), so ||(X_gpu - X_or) R||_F / ||X_or R||_F estimates the relative
    Frobenius error; X_or R comes from the committed oracle script."""
    meta = _sketch_meta().get(str(n))
    if meta is None:
        pytest.skip(f"no committed oracle sketch for n={n} (tests/golden/make_sketch.py {n})")
    yor = np.load(os.path.join(GOLD, meta["file"]))
    kappa = meta["kappa2_est"]
    kf = _kfac(kappa)
    z = synth.config2(n, seed=0)
    zt = torch.from_numpy(z).to(DEV)
    r = torch.from_numpy(synth.rademacher(n, meta["k"], seed=0)).to(DEV).to(torch.complex128)
    yo = torch.from_numpy(yor).to(DEV)
    for name, f in (("frob", lambda: fb.inv(zt)), ("zinv_lu", lambda: fb.zinv(zt))):
        x = f()
        y = x @ r  # independent library GEMM (torch complex128)
        rel = float(torch.linalg.norm(y - yo) / torch.linalg.norm(yo))
        assert rel <= 1e-10 * kf, (name, n, rel, kappa)
        _residuals(z, zt, x, n, kf, seed=n + 1)
        del x, y
        torch.cuda.empty_cache()


def _config3_part(n, total, chunk):
    z_all = synth.batch(n, total, seed=0)
    zt = torch.from_numpy(z_all).to(DEV)
    x, inf, bu = fb.inv_batched(zt)  # the bench's launch: the whole sub-batch in one call
    assert int((inf != 0).sum()) == 0
    sv = torch.linalg.svdvals(zt)  # descending
    kap = (sv[:, 0] / sv[:, -1]).cpu().numpy()
    del sv
    bu = bu.cpu().numpy()
    worst, mism, switched = 0.0, [], int((bu == 2).sum())
    for s in range(0, total, chunk):
        e = min(total, s + chunk)
        xo, st, info, buo, rho = oracle.frob_inv_many(z_all[s:e])
        assert np.all(st == 0)
        xg = x[s:e].cpu().numpy()
        num = np.linalg.norm((xg - xo).reshape(e - s, -1), axis=1)
        den = np.linalg.norm(xo.reshape(e - s, -1), axis=1)
        rel = num / den
        bound = 1e-10 * np.maximum(1.0, kap[s:e] / 1e4)
        same = bu[s:e] == buo
        # branch decision: identical except where kappa_inf(A) sits within rounding of the switch point
        near = (np.abs(rho[:, 2] / (oracle.KAPPA_SWITCH * math.sqrt(n)) - 1.0) < 1e-6) | (np.abs(rho[:, 3] / rho[:, 2] - 1.0) < 1e-6)
        bad_branch = np.nonzero(~same & ~near)[0]
        assert bad_branch.size == 0, (n, s + bad_branch[:8], rho[bad_branch[:8]])
        for i in np.nonzero(~same)[0]:      # rounding-level ties: judge against the definition
            ref, _ = oracle.zinv_gj(z_all[s + i])
            rel[i] = oracle.rel_fro(xg[i], ref)
            mism.append(s + i)
        assert np.all(rel <= bound), (n, s + np.argmax(rel / bound), rel.max())
        worst = max(worst, float((rel / bound).max()))
    return {"n": n, "count": total, "branch_b": switched, "tie_mismatch": mism, "worst_rel_over_bound": worst}


def test_config3_full_set_vs_oracle():
    """Every config-3 matrix (65536 x n=32 and 16384 x n=128, seed 0 + index, shift 8) against the
    oracle's Alg 1, element by element, and the AUTO branch against the oracle's."""
    r32 = _config3_part(32, 65536, 16384)
    r128 = _config3_part(128, 16384, 2048)
    assert r128["branch_b"] > 0  # the kappa(A) tail exercises the switch
    print(json.dumps({"config3": [r32, r128]}))
