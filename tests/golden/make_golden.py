"""Generate golden fixtures by running the REFERENCE itself (propsim).

Run in the build container (the reference exists only here):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes tests/golden/golden.json. Every number in it was produced by
/root/reference/pkg/src/propsim (run_2way / run_3way / verify.*), never by
this repository's code; the GPU tests and the oracle tests compare against
it on the GPU box, where the reference is absent.
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
from propsim import DecompGrid, Problem, run_2way, run_3way  # noqa: E402
from propsim.core import field_range, vector_range  # noqa: E402
from propsim.verify import (  # noqa: E402
    Checksum128, checksum, dense_matrix, gen_analytic, gen_random_exact, mix64, oracle_2way,
    oracle_3way, value_bits,
)

OUT = Path(__file__).resolve().parent / "golden.json"


class ArraySource:
    """In-memory source (reference tests/conftest.py:17-26 shape)."""

    def __init__(self, matrix):
        self.matrix = np.asarray(matrix)

    def local_block(self, problem, grid, coords):
        f0, f1 = field_range(grid, coords.p_f, problem.n_f)
        v0, v1 = vector_range(grid, coords.p_v, problem.n_v)
        return self.matrix[f0:f1, v0:v1]


def uniform(seed, n_f, n_v, precision):
    """Same formula as psim_gen_uniform / oracle.propsim_np.uniform."""
    q = np.arange(n_f, dtype=np.uint64)[:, None]
    i = np.arange(n_v, dtype=np.uint64)[None, :]
    h = np.vectorize(mix64, otypes=[object])((q * np.uint64(n_v) + i) ^ np.uint64(seed))
    h = h.astype(np.uint64)
    if precision == "double":
        return np.asfortranarray((h >> np.uint64(11)).astype(np.float64) * 2.0**-53)
    return np.asfortranarray((h >> np.uint64(40)).astype(np.float32) * np.float32(2.0**-24))


def grid_dict(g):
    return {"n_pf": g.n_pf, "n_pv": g.n_pv, "n_pr": g.n_pr, "n_st": g.n_st}


def record_bits(res):
    return [format(value_bits(r.value), "x") for r in res.records]


def run_case(kind, arity, precision, n_f, n_v, grid, seed=0, bits=0, values=False, matrix=None):
    if kind == "random-exact":
        src = gen_random_exact(seed, n_f, n_v, bits)
    elif kind == "analytic":
        src = gen_analytic(seed, n_f, n_v)
    elif kind == "uniform":
        src = ArraySource(uniform(seed, n_f, n_v, precision))
    else:
        src = ArraySource(np.asfortranarray(np.asarray(matrix, dtype=np.float64)))
    prob = Problem(arity, n_f, n_v, src, precision)
    res = run_2way(prob, grid) if arity == 2 else run_3way(prob, grid)
    case = {
        "kind": kind, "arity": arity, "precision": precision, "n_f": n_f, "n_v": n_v,
        "seed": seed, "bits": bits, "grid": grid_dict(grid),
        "records": len(res.records), "degenerate": res.degenerate_count,
        "checksum": res.checksum.hex,
    }
    if matrix is not None:
        case["matrix"] = np.asarray(matrix, dtype=np.float64).tolist()
    if values:
        case["value_bits"] = record_bits(res)
        case["degenerate_flags"] = [bool(r.degenerate) for r in res.records]
    return case


def main():
    kat = {
        "mix64": {str(x): format(mix64(x), "x") for x in (0, 1, 2, (1 << 64) - 1, 12345)},
        "random_exact_42_4x3_b11": dense_matrix(gen_random_exact(42, 4, 3, 11)).tolist(),
        "oracle2_42_4x3_b11": {
            f"{r.id.indices[0]},{r.id.indices[1]}": float(r.value)
            for r in oracle_2way(dense_matrix(gen_random_exact(42, 4, 3, 11)))
        },
        "oracle3_42_4x3_b11": float(oracle_3way(dense_matrix(gen_random_exact(42, 4, 3, 11)))[0].value),
    }
    from propsim.core import MetricRecord, TupleId

    vals = [((0, 1), 0.8), ((0, 2), 2.0 / 3.0), ((1, 2), 0.75)]
    for name, dt in (("double", np.float64), ("single", np.float32)):
        recs = [MetricRecord(TupleId(ix), dt(v)) for ix, v in vals]
        kat[f"checksum_pairs_{name}"] = checksum(recs, 3).hex
    kat["empty_checksum"] = Checksum128().hex

    cases = []
    one = DecompGrid()
    # Appendix B configurations + the reference tests' specs
    cases.append(run_case("random-exact", 2, "double", 1000, 500, one, 2026, 20))
    cases.append(run_case("random-exact", 2, "double", 1000, 500, one, 2026, 8))
    cases.append(run_case("random-exact", 2, "single", 1000, 500, one, 2026, 8))
    cases.append(run_case("random-exact", 3, "double", 1000, 60, one, 2026, 20))
    cases.append(run_case("random-exact", 3, "single", 1000, 60, one, 2026, 8))
    cases.append(run_case("random-exact", 3, "double", 10000, 96, one, 2026, 20))
    for prec in ("double", "single"):
        cases.append(run_case("random-exact", 2, prec, 16, 12, one, 7, 8, values=True))
        cases.append(run_case("random-exact", 3, prec, 10, 6, one, 19, 6, values=True))
        cases.append(run_case("random-exact", 3, prec, 8, 12, one, 4, 5, values=True))
        cases.append(run_case("analytic", 2, prec, 24, 6, one, values=True))
        cases.append(run_case("analytic", 3, prec, 24, 6, one, values=True))
        # general floating-point data (bitwise parity beyond exact integers)
        cases.append(run_case("uniform", 2, prec, 777, 48, one, 11, values=True))
        cases.append(run_case("uniform", 3, prec, 200, 24, one, 13, values=True))
        cases.append(run_case("uniform", 2, prec, 3001, 130, one, 5))
    # field-split grids: the ordered p_f fold (bitwise on general FP data)
    cases.append(run_case("uniform", 2, "double", 1000, 120, DecompGrid(n_pf=8), 17, values=True))
    cases.append(run_case("uniform", 2, "single", 1000, 120, DecompGrid(n_pf=4, n_pv=2), 17,
                          values=True))
    cases.append(run_case("uniform", 3, "double", 200, 24, DecompGrid(n_pf=2), 23, values=True))
    cases.append(run_case("uniform", 3, "single", 300, 24, DecompGrid(n_pf=4, n_pv=2), 29,
                          values=True))
    cases.append(run_case("random-exact", 3, "double", 64, 24, DecompGrid(n_pf=2, n_pr=2), 402,
                          11))
    # edge cases from the reference tests
    m2 = np.zeros((4, 4))
    m2[:, 0] = [1, 2, 0, 1]
    m2[:, 2] = [0, 1, 1, 0]
    cases.append(run_case("matrix", 2, "double", 4, 4, one, matrix=m2, values=True))
    m3 = np.ones((6, 6))
    m3[:, 2] = m3[:, 4] = m3[:, 5] = 0.0
    cases.append(run_case("matrix", 3, "double", 6, 6, one, matrix=m3, values=True))
    cases.append(run_case("random-exact", 2, "double", 1, 7, one, 3, 4, values=True))
    cases.append(run_case("random-exact", 2, "double", 9, 2, one, 3, 4, values=True))
    cases.append(run_case("random-exact", 3, "double", 5, 6, one, 9, 0, values=True))
    # cross-grid (results must equal the 1-rank run, so checksums repeat)
    for g in (DecompGrid(n_pv=2), DecompGrid(n_pv=3, n_pr=2), DecompGrid(n_pf=2, n_pv=2),
              DecompGrid(n_pv=4)):
        cases.append(run_case("random-exact", 2, "double", 64, 24, g, 401, 11))
    for g in (DecompGrid(n_pv=2), DecompGrid(n_pv=2, n_pr=3), DecompGrid(n_st=2),
              DecompGrid(n_pv=4)):
        cases.append(run_case("random-exact", 3, "double", 64, 24, g, 402, 11))
    # Sorenson (metric="sorenson"): the reference's bit-packed kernel on 0/1 data
    for n_f, n_v, g, prec in ((1, 9, DecompGrid(), "double"), (63, 17, DecompGrid(), "double"),
                              (65, 40, DecompGrid(n_pv=2), "single"),
                              (1000, 130, DecompGrid(), "double"),
                              (777, 96, DecompGrid(n_pv=3, n_pr=2), "single")):
        spec = gen_random_exact(31, n_f, n_v, 1)
        prob = Problem(2, n_f, n_v, spec, prec, metric="sorenson")
        res = run_2way(prob, g)
        cases.append({
            "kind": "random-exact", "metric": "sorenson", "arity": 2, "precision": prec,
            "n_f": n_f, "n_v": n_v, "seed": 31, "bits": 1, "grid": grid_dict(g),
            "records": len(res.records), "degenerate": res.degenerate_count,
            "checksum": res.checksum.hex, "kernel": res.kernel,
        })
    spec = gen_random_exact(32, 90, 12, 1)
    res = run_3way(Problem(3, 90, 12, spec, "double", metric="sorenson"), DecompGrid())
    cases.append({"kind": "random-exact", "metric": "sorenson", "arity": 3, "precision": "double",
                  "n_f": 90, "n_v": 12, "seed": 32, "bits": 1, "grid": grid_dict(DecompGrid()),
                  "records": len(res.records), "degenerate": res.degenerate_count,
                  "checksum": res.checksum.hex, "kernel": res.kernel})
    # staged 3-way runs: one case per stage
    for s in range(2):
        spec = gen_random_exact(402, 64, 24, 11)
        prob = Problem(3, 64, 24, spec, "double")
        res = run_3way(prob, DecompGrid(n_pv=2, n_st=2), stage=s)
        cases.append({
            "kind": "random-exact", "arity": 3, "precision": "double", "n_f": 64, "n_v": 24,
            "seed": 402, "bits": 11, "grid": grid_dict(DecompGrid(n_pv=2, n_st=2)), "stage": s,
            "records": len(res.records), "degenerate": res.degenerate_count,
            "checksum": res.checksum.hex,
            "ids": [list(r.id.indices) for r in res.records],
        })
    OUT.write_text(json.dumps({"kat": kat, "cases": cases, "outputs": output_cases(),
                               "owners": owner_tables()}, indent=0))
    print(f"wrote {OUT} ({len(cases)} cases)")


def owner_tables():
    """Reference owns_pair / owns_triple for every tuple of small grids."""
    from propsim.schedule import owns_pair, owns_triple
    from propsim.core import iter_pairs, iter_triples

    out = []
    for n_v, g in ((24, DecompGrid(n_pv=3, n_pr=2)), (24, DecompGrid(n_pv=4, n_pr=3, n_pf=2)),
                   (30, DecompGrid(n_pv=5, n_pr=4)), (12, DecompGrid(n_pv=6))):
        out.append({"arity": 2, "n_v": n_v, "grid": grid_dict(g),
                    "rank": [owns_pair(i, j, n_v, g)[0] for i, j in iter_pairs(n_v)]})
    for n_v, g in ((24, DecompGrid(n_pv=2, n_pr=3)), (36, DecompGrid(n_pv=3, n_pr=5, n_st=2)),
                   (48, DecompGrid(n_pv=4, n_pr=7, n_pf=2)), (24, DecompGrid(n_st=2, n_pr=2))):
        own = [owns_triple(i, j, k, n_v, g) for i, j, k in iter_triples(n_v)]
        out.append({"arity": 3, "n_v": n_v, "grid": grid_dict(g),
                    "rank": [o[0] for o in own], "stage": [o[1] for o in own]})
    return out


def output_cases():
    """Reference run + write_run_output: per-file sha256 and the manifest."""
    import hashlib
    import tempfile

    from propsim.io import MetricOutputSpec, read_manifest, write_run_output

    specs = [
        ("uniform", 2, "double", 777, 48, DecompGrid(), 11, 0, None, "czekanowski"),
        ("random-exact", 2, "double", 64, 24, DecompGrid(n_pv=3, n_pr=2), 401, 11, None,
         "czekanowski"),
        ("uniform", 2, "single", 1000, 120, DecompGrid(n_pf=4, n_pv=2), 17, 0, None,
         "czekanowski"),
        ("random-exact", 3, "double", 64, 24, DecompGrid(n_pv=2, n_pr=3), 402, 11, None,
         "czekanowski"),
        ("random-exact", 3, "double", 64, 24, DecompGrid(n_pv=2, n_st=2), 402, 11, 1,
         "czekanowski"),
        ("uniform", 3, "single", 300, 24, DecompGrid(n_pf=4, n_pv=2), 29, 0, None,
         "czekanowski"),
        ("random-exact", 2, "single", 777, 96, DecompGrid(n_pv=3, n_pr=2), 31, 1, None,
         "sorenson"),
    ]
    out = []
    for kind, arity, prec, n_f, n_v, g, seed, bits, stage, metric in specs:
        if kind == "uniform":
            src = ArraySource(uniform(seed, n_f, n_v, prec))
        else:
            src = gen_random_exact(seed, n_f, n_v, bits)
        prob = Problem(arity, n_f, n_v, src, prec, metric=metric)
        res = run_2way(prob, g) if arity == 2 else run_3way(prob, g, stage=stage)
        for mode in ("full", "byte"):
            with tempfile.TemporaryDirectory() as d:
                write_run_output(res, MetricOutputSpec(d, mode), source={"kind": kind})
                files = {}
                for r in range(g.n_p):
                    blob = Path(d, f"metrics_{r}.bin").read_bytes()
                    files[str(r)] = [len(blob), hashlib.sha256(blob).hexdigest()]
                out.append({"kind": kind, "arity": arity, "precision": prec, "n_f": n_f,
                            "n_v": n_v, "grid": grid_dict(g), "seed": seed, "bits": bits,
                            "stage": stage, "metric": metric, "mode": mode, "files": files,
                            "manifest": read_manifest(Path(d, "manifest.txt"))})
    return out


if __name__ == "__main__":
    main()
