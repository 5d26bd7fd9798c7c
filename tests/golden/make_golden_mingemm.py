"""Golden vectors for the kernel plug-point module, produced by the REFERENCE
(propsim.mingemm): mgemm_blocked / mgemm_naive, column_sums, xj_columns,
pair_numerators, triple_min_numerators, pack_bits, mgemm_bitpacked.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_mingemm.py

Writes tests/golden/mingemm.json (inputs and outputs as IEEE bit patterns).
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from propsim import mingemm as M  # noqa: E402

OUT = Path(__file__).resolve().parent / "mingemm.json"


def bits(a) -> list[str]:
    a = np.asarray(a)
    u = np.asfortranarray(a).ravel(order="F").view(np.uint64 if a.dtype.itemsize == 8
                                                    else np.uint32)
    return [format(int(x), "x") for x in u]


def matrix(rng, n_f, n, dt, zeros=False):
    X = rng.random((n_f, n)).astype(dt)
    if zeros:  # signed zeros and exact ties exercise the min rule
        X[rng.random((n_f, n)) < 0.2] = dt(0.0)
        X[rng.random((n_f, n)) < 0.2] = -dt(0.0)
        X[rng.random((n_f, n)) < 0.1] = dt(0.5)
    return np.asfortranarray(X)


def main():
    rng = np.random.default_rng(1705)
    cases = []
    for dt, name in ((np.float64, "double"), (np.float32, "single")):
        for n_f, m, n, zeros in ((37, 5, 7, False), (150, 40, 33, True), (1, 3, 2, False),
                                 (129, 20, 1, True)):
            W, V = matrix(rng, n_f, m, dt, zeros), matrix(rng, n_f, n, dt, zeros)
            vj = matrix(rng, n_f, 1, dt, zeros)[:, 0]
            cases.append({
                "precision": name, "n_f": n_f, "m": m, "n": n,
                "W": bits(W), "V": bits(V), "vj": bits(vj),
                "mgemm": bits(M.mgemm_blocked(W, V)),
                "naive_equals_blocked": bits(M.mgemm_naive(W, V)) == bits(M.mgemm_blocked(W, V)),
                "column_sums": bits(M.column_sums(V)),
                "xj_columns": bits(M.xj_columns(V, vj)),
                "pair_numerators": bits(M.pair_numerators(V)),
                "triple_min_numerators": bits(M.triple_min_numerators(V)),
            })
    bit_cases = []
    for n_f, m, n in ((100, 9, 6), (64, 3, 4), (31, 5, 5), (257, 70, 3)):
        A = (rng.random((n_f, m)) < 0.5).astype(np.float64)
        B = (rng.random((n_f, n)) < 0.3).astype(np.float64)
        pa, pb = M.pack_bits(A), M.pack_bits(B)
        bit_cases.append({
            "n_f": n_f, "m": m, "n": n, "A": A.T.astype(int).tolist(), "B": B.T.astype(int).tolist(),
            "words_A": [[format(int(x), "x") for x in col] for col in pa.words.T],
            "counts": M.mgemm_bitpacked(pa, pb).T.tolist(),
        })
    OUT.write_text(json.dumps({"dense": cases, "bits": bit_cases}, indent=0))
    print(f"wrote {OUT} ({len(cases)} dense, {len(bit_cases)} bit cases)")


if __name__ == "__main__":
    main()
