"""GPU parity of the LU pipeline variants that are selected by environment switches (A/B aids,
read once per process, so each runs in its own subprocess): lu2's look-ahead modes
(FROB_LU2_LOOKAHEAD = 0 none, 1 separate NEXT kernel, 2 fused into the panel), and the blocked
getrf with lu2's in-place panels (FROB_LU2_MAX=1024 routes n > 1024 to getrf) against the same
oracle and bounds as tests/test_gpu_parity.py."""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIZES = (300, 1100)

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import synth, paper_2208_01239_b200 as fb
out = {{}}
for n in {sizes!r}:
    z = synth.shifted_complex(n, seed=77 * n, shift=n ** 0.5 + 2.0)
    zt = torch.from_numpy(z).cuda()
    out[f"frob{{n}}"] = fb.inv(zt).cpu().numpy()
    out[f"zinv{{n}}"] = fb.zinv(zt).cpu().numpy()
np.savez({path!r}, **out)
"""


@pytest.fixture(scope="module")
def refs():
    r = {}
    for n in SIZES:
        z = synth.shifted_complex(n, seed=77 * n, shift=math.sqrt(n) + 2.0)
        x, info = oracle.zinv_gj(z)
        assert info == 0
        r[n] = (z, x)
    return r


@pytest.mark.parametrize("env", [{"FROB_LU2_LOOKAHEAD": "0"}, {"FROB_LU2_LOOKAHEAD": "1"},
                                 {"FROB_LU2_LOOKAHEAD": "2"}, {"FROB_LU2_MAX": "1024"}],
                         ids=["lookahead0", "lookahead1", "lookahead2", "getrf"])
def test_pipeline_mode(env, refs, tmp_path):
    path = str(tmp_path / "out.npz")
    code = CHILD.format(root=ROOT, sizes=SIZES, path=path)
    e = dict(os.environ, **env)
    p = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    got = np.load(path)
    for n in SIZES:
        z, ref = refs[n]
        for k in ("frob", "zinv"):
            x = got[f"{k}{n}"]
            assert oracle.rel_fro(x, ref) <= 1e-10, (env, k, n)
            r = np.linalg.norm(z @ x - np.eye(n))
            assert r <= 1e-11 * n, (env, k, n, r)


P2C_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import synth, paper_2208_01239_b200 as fb
n = {n}
a, _ = synth.gauss_pair(n, seed=31, shift=n ** 0.5 + 2.0)
lu, perm, info = fb.dgetrf(torch.from_numpy(a).cuda())
np.savez({path!r}, lu=lu.cpu().numpy(), perm=perm.cpu().numpy())
"""


def test_blocked_lu_wide_cluster_panels(tmp_path):
    """The blocked getrf's panels for 4096 < m <= 8192 rows run on 9..16-CTA clusters (non-portable
    cluster size; FROB_P2C_MAX=8 keeps them on the older 16-column cluster panel).  n = 4700: panels
    of 4700 .. 4097 rows (10-CTA clusters, ragged last CTA).  Both must give P A = L U to rounding,
    and the same pivots (identical argmax rule, well separated pivots for this shifted Gaussian)."""
    n = 4700
    got = []
    for env in ({"FROB_P2C_MAX": "8"}, {}):
        path = str(tmp_path / f"lu{len(got)}.npz")
        p = subprocess.run([sys.executable, "-c", P2C_CHILD.format(root=ROOT, n=n, path=path)],
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        got.append(np.load(path))
    a, _ = synth.gauss_pair(n, seed=31, shift=math.sqrt(n) + 2.0)
    for g in got:
        lu, perm = g["lu"], g["perm"].astype(np.int64)
        assert sorted(perm.tolist()) == list(range(n))
        L = np.tril(lu, -1) + np.eye(n)
        U = np.triu(lu)
        r = np.linalg.norm(a[perm] - L @ U) / np.linalg.norm(a)
        assert r <= 1e-14 * math.sqrt(n), r
    assert np.array_equal(got[0]["perm"], got[1]["perm"])
    assert np.abs(got[0]["lu"] - got[1]["lu"]).max() <= 1e-10 * np.abs(got[0]["lu"]).max()


@pytest.mark.parametrize("n", [2048, 4352])
def test_blocked_lu_lu2_tail(n, tmp_path):
    """The real blocked getrf hands its last trailing matrix to lu2 (FROB_GETRF_TAIL=0: blocked to
    the end): n = 2048 -> one 256-column block + lu2 on 1792 rows; n = 4352 -> lu2 on exactly 4096
    rows (its maximum).  Both give P A = L U to rounding and the same pivots."""
    got = []
    for env in ({"FROB_GETRF_TAIL": "0"}, {}):
        path = str(tmp_path / f"tail{len(got)}.npz")
        p = subprocess.run([sys.executable, "-c", P2C_CHILD.format(root=ROOT, n=n, path=path)],
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        got.append(np.load(path))
    a, _ = synth.gauss_pair(n, seed=31, shift=math.sqrt(n) + 2.0)
    for g in got:
        lu, perm = g["lu"], g["perm"].astype(np.int64)
        assert sorted(perm.tolist()) == list(range(n))
        L = np.tril(lu, -1) + np.eye(n)
        U = np.triu(lu)
        r = np.linalg.norm(a[perm] - L @ U) / np.linalg.norm(a)
        assert r <= 1e-14 * math.sqrt(n), r
    assert np.array_equal(got[0]["perm"], got[1]["perm"])
    assert np.abs(got[0]["lu"] - got[1]["lu"]).max() <= 1e-10 * np.abs(got[0]["lu"]).max()
