"""Golden runs of the REFERENCE at the benchmarked configurations' shapes.

Run in the build container (the reference exists only here):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_configs.py

Writes tests/golden/configs.json. Each case keeps a BASELINE config's field
count, precision, bits and decomposition, with n_v reduced so that
propsim.run_2way / run_3way (the reference's own entry points) finish in
seconds (SURVEY 8d "Parity at full size": reduced-n_v runs compare full
checksums). Every checksum and value bit in the file comes from
/root/reference/pkg/src/propsim, never from this repository's code.
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from propsim import DecompGrid, Problem, run_2way, run_3way  # noqa: E402
from propsim.core import field_range, vector_range  # noqa: E402
from propsim.verify import _mix64_u64, gen_random_exact, value_bits  # noqa: E402

OUT = Path(__file__).resolve().parent / "configs.json"
SEED = 2026


def grid_dict(g):
    return {"n_pf": g.n_pf, "n_pv": g.n_pv, "n_pr": g.n_pr, "n_st": g.n_st}


class ArraySource:
    """In-memory source (reference tests/conftest.py:17-26 shape)."""

    def __init__(self, matrix):
        self.matrix = matrix

    def local_block(self, problem, grid, coords):
        f0, f1 = field_range(grid, coords.p_f, problem.n_f)
        v0, v1 = vector_range(grid, coords.p_v, problem.n_v)
        return self.matrix[f0:f1, v0:v1]


def uniform(seed, n_f, n_v, precision):
    """General-FP input, same formula as psim_gen_uniform (the reference's
    vectorised mix64, verify.py:47-55)."""
    q = np.arange(n_f, dtype=np.uint64)[:, None]
    i = np.arange(n_v, dtype=np.uint64)[None, :]
    h = _mix64_u64((q * np.uint64(n_v) + i) ^ np.uint64(seed))
    if precision == "double":
        return np.asfortranarray((h >> np.uint64(11)).astype(np.float64) * 2.0**-53)
    return np.asfortranarray((h >> np.uint64(40)).astype(np.float32) * np.float32(2.0**-24))


_UNIFORM = {}


def case(cfg, arity, precision, n_f, n_v, bits, grid, sample_bits=64, kind="random-exact"):
    t0 = time.perf_counter()
    if kind == "uniform":
        key = (n_f, n_v, precision)
        if key not in _UNIFORM:
            _UNIFORM[key] = uniform(SEED, n_f, n_v, precision)
        src = ArraySource(_UNIFORM[key])
    else:
        src = gen_random_exact(SEED, n_f, n_v, bits)
    prob = Problem(arity, n_f, n_v, src, precision)
    res = run_2way(prob, grid) if arity == 2 else run_3way(prob, grid)
    recs = res.records
    step = max(1, len(recs) // sample_bits)
    out = {
        "config": cfg, "kind": kind, "arity": arity, "precision": precision,
        "n_f": n_f, "n_v": n_v, "seed": SEED, "bits": bits, "grid": grid_dict(grid),
        "records": len(recs), "degenerate": res.degenerate_count, "checksum": res.checksum.hex,
        # a spread of individual records: canonical position -> value bits
        "sample": {str(p): format(value_bits(recs[p].value), "x")
                   for p in list(range(0, len(recs), step)) + [len(recs) - 1]},
    }
    print(f"{cfg} {arity}-way {precision} {n_f}x{n_v} grid={grid_dict(grid)} "
          f"{res.checksum.hex} ({time.perf_counter() - t0:.1f} s)", flush=True)
    return out


def main():
    cases = []
    # cfg2: 2-way FP64, n_f = 20000, bits 20 (1 GPU; also its circulant splits)
    for g in (DecompGrid(), DecompGrid(n_pv=2), DecompGrid(n_pv=4), DecompGrid(n_pv=8)):
        cases.append(case("cfg2", 2, "double", 20000, 192, 20, g))
    # cfg3: 2-way FP32, n_f = 50000, bits 6, circulant n_pv = 1 / 2 / 4 / 8
    for g in (DecompGrid(), DecompGrid(n_pv=2), DecompGrid(n_pv=4), DecompGrid(n_pv=8)):
        cases.append(case("cfg3", 2, "single", 50000, 192, 6, g))
    # cfg4: 3-way FP64, n_f = 10000, bits 20, tetrahedral n_pv = 1 / 2 / 4 / 8
    for g in (DecompGrid(), DecompGrid(n_pv=2), DecompGrid(n_pv=4), DecompGrid(n_pv=8)):
        cases.append(case("cfg4", 3, "double", 10000, 96, 20, g))
    # cfg5: 2-way FP64, n_f = 2,000,000, bits 20, field split n_pf = 8 (the
    # ordered fold of engine.py:197-216), plus n_pf = 2 / 4 and n_pf = 1
    for g in (DecompGrid(n_pf=8), DecompGrid(n_pf=4), DecompGrid(n_pf=2), DecompGrid()):
        cases.append(case("cfg5", 2, "double", 2_000_000, 48, 20, g))
    # general FP data at cfg5's field depth: the n_pf fold order changes bits
    # (SURVEY Appendix A), so these pin the ascending-p_f fold itself
    for g in (DecompGrid(n_pf=8), DecompGrid(n_pf=2), DecompGrid()):
        cases.append(case("cfg5", 2, "double", 2_000_000, 48, 0, g, kind="uniform"))
    # general FP data at cfg3's field width in FP32 (sequential FP32 sums)
    cases.append(case("cfg3", 2, "single", 50000, 192, 0, DecompGrid(n_pv=4), kind="uniform"))
    OUT.write_text(json.dumps({"seed": SEED, "cases": cases}, indent=0))
    print(f"wrote {OUT} ({len(cases)} cases)")


if __name__ == "__main__":
    main()
