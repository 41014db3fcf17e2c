"""Write the config-5 sketch-parity fixtures: X_oracle R for R = synth.rademacher(n, 64).

Calls only ``oracle/`` (Gaussian elimination with partial pivoting: or_zgetrf + or_zgetrs,
the plain definition of Z^{-1} R -- Lemma 4.1, says Frobenius inversion reaches
Z^{-1} exactly) and ``synth/`` (the BASELINE config-5 generator, A = G1 + sqrt(n) I,
B = G2, seed 0).  Also records kappa_2(Z) (power / inverse-power iteration, oracle.kappa2)
so the GPU test can pick the north-star bound (kappa_2 <= 1e4) or the kappa-scaled reading
(R10 / SURVEY G7).

    python tests/golden/make_sketch.py 4096 8192 16384

Outputs tests/golden/sketch_config5_n{n}.npy (complex128, n x 64) and merges one record per n
into tests/golden/sketch_config5.json.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
import synth  # noqa: E402

K = 64
META = os.path.join(HERE, "sketch_config5.json")


def one(n: int) -> dict:
    z = synth.config2(n, seed=0)
    r = synth.rademacher(n, K, seed=0)
    t0 = time.time()
    fac = oracle.zgetrf(z)
    t_lu = time.time() - t0
    assert fac[3] == 0, f"singular at {fac[3]}"
    t0 = time.time()
    y = oracle.zgetrs(fac, r)
    t_s = time.time() - t0
    res = float(np.linalg.norm(z @ y - r) / np.linalg.norm(r))
    t0 = time.time()
    kap, smax, smin = oracle.kappa2(z, fac=fac, iters=40)
    t_k = time.time() - t0
    np.save(os.path.join(HERE, f"sketch_config5_n{n}.npy"), y)
    return {"n": n, "k": K, "seed": 0, "generator": "synth.config2(n, seed=0); R = synth.rademacher(n, 64, seed=0)",
            "file": f"sketch_config5_n{n}.npy", "fro_XR": float(np.linalg.norm(y)),
            "oracle_residual_ZY_minus_R_rel": res, "kappa2_est": kap, "sigma_max_est": smax,
            "sigma_min_est": smin, "oracle_threads": oracle.num_threads(),
            "seconds": {"zgetrf": t_lu, "zgetrs": t_s, "kappa2": t_k},
            "cite": "Lemma 4.1 (P:L175-188); sketch parity SURVEY 8(c); kappa reading DESIGN R10"}


def main(ns):
    meta = {}
    if os.path.exists(META):
        with open(META) as f:
            meta = json.load(f)
    for n in ns:
        rec = one(int(n))
        meta[str(n)] = rec
        with open(META, "w") as f:
            json.dump(meta, f, indent=1, sort_keys=True)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["4096", "8192", "16384"])
