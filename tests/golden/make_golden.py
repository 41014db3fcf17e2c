"""Writes tests/golden/exact_inverses.json using ONLY oracle.exact (exact Q(i) arithmetic).

Each case: small integer complex matrix Z = A + iB and its exact inverse over Q(i),
plus the exact Alg 1 value for both branches where that branch's preconditions hold
(Lemma 4.1: the two must agree exactly).  Re-run:
    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from oracle import exact  # noqa: E402


def enc(m):
    return [[[str(v[0]), str(v[1])] for v in r] for r in m]


def main():
    rng = np.random.default_rng(20220802)
    cases = []
    for n in (1, 2, 3, 4, 5):
        made = 0
        while made < 3:
            re = rng.integers(-4, 5, size=(n, n))
            im = rng.integers(-4, 5, size=(n, n))
            z = exact.from_ints(re.tolist(), im.tolist())
            try:
                zinv = exact.inv_exact(z)
            except ZeroDivisionError:
                continue
            case = {"n": n, "re": re.tolist(), "im": im.tolist(), "inv": enc(zinv)}
            for br in ("a", "b"):
                try:
                    fr = exact.frobenius_exact(z, br)
                except ZeroDivisionError:
                    fr = None
                case["frob_" + br] = enc(fr) if fr is not None else None
            cases.append(case)
            made += 1
    out = {
        "source": "oracle/exact.py (exact Gauss-Jordan over Q(i)); Lemma 4.1 P:L175-188",
        "cases": cases,
    }
    path = os.path.join(os.path.dirname(__file__), "exact_inverses.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path, len(cases), "cases")


if __name__ == "__main__":
    main()
