"""INTEGRATION.md section 3 exercised as written: integration/propsim_b200.py
(the reference-side ctypes binding -- numpy + ctypes, no torch) runs the
reference's golden problems through psim_run2 / psim_run3."""
import importlib.util
import math
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import cuda_available, golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

ROOT = Path(__file__).resolve().parent.parent


def _binding():
    spec = importlib.util.spec_from_file_location("propsim_b200",
                                                  ROOT / "integration" / "propsim_b200.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod  # dataclasses resolve annotations through sys.modules
    spec.loader.exec_module(mod)
    mod.lib(str(ROOT / "paper_1705_08210_b200" / "_lib" / "libpsim.so"))
    return mod


class Spec:
    """A reference SyntheticSpec's attributes (verify.py:113-147)."""

    def __init__(self, kind, seed, n_f, n_v, bits=0):
        self.kind, self.seed, self.n_f, self.n_v, self.bits = kind, seed, n_f, n_v, bits


class Prob:
    def __init__(self, arity, n_f, n_v, source, precision="double"):
        self.arity, self.n_f, self.n_v, self.source = arity, n_f, n_v, source
        self.precision, self.metric = precision, "czekanowski"


class Grid:
    def __init__(self, n_pf=1, n_pv=1, n_pr=1, n_st=1):
        self.n_pf, self.n_pv, self.n_pr, self.n_st = n_pf, n_pv, n_pr, n_st


class ArraySource:
    """reference tests/conftest.py:17-26"""

    def __init__(self, m):
        self.m = m

    def local_block(self, problem, grid, coords):
        w_f, w_v = problem.n_f // grid.n_pf, problem.n_v // grid.n_pv
        return self.m[coords.p_f * w_f:(coords.p_f + 1) * w_f,
                      coords.p_v * w_v:(coords.p_v + 1) * w_v]


def _case(**kw):
    for c in golden()["cases"]:
        if all(c.get(k) == v for k, v in kw.items()) and c["grid"]["n_pf"] == 1 \
                and c["grid"]["n_pv"] == 1 and "stage" not in c:
            return c
    raise KeyError(kw)


def test_binding_cfg1_and_values():
    B = _binding()
    c = _case(kind="random-exact", arity=2, precision="double", n_f=1000, n_v=500, bits=20)
    res = B.run_2way(Prob(2, 1000, 500, Spec("random-exact", 2026, 1000, 500, 20)), Grid())
    assert res.checksum_hex == c["checksum"] == "ea23ebab734aeaaefdc87babae741b72"
    assert res.count == c["records"] == math.comb(500, 2)
    assert res.degenerate_count == c["degenerate"]
    import paper_1705_08210_b200 as P

    want = P.run_2way(P.Problem(2, 1000, 500, P.gen_random_exact(2026, 1000, 500, 20)),
                      P.DecompGrid()).records.values
    assert (res.values.view(np.uint64) == want.view(np.uint64)).all()
    assert res.traffic == {}


def test_binding_generic_source_and_3way():
    B = _binding()
    from oracle import propsim_np as O

    c = _case(kind="uniform", arity=2, precision="double", n_f=777, n_v=48)
    m = O.uniform(c["seed"], 777, 48, np.float64)
    res = B.run_2way(Prob(2, 777, 48, ArraySource(m)), Grid())
    assert res.checksum_hex == c["checksum"]
    bits = [format(int(b), "x") for b in O.value_bits(res.values)]
    assert bits == c["value_bits"]
    c3 = _case(kind="random-exact", arity=3, precision="double", n_f=1000, n_v=60, bits=20)
    r3 = B.run_3way(Prob(3, 1000, 60, Spec("random-exact", 2026, 1000, 60, 20)), Grid())
    assert r3.checksum_hex == c3["checksum"] and r3.count == c3["records"]
    bad = m.copy()
    bad[5, 5] = np.nan
    with pytest.raises(ValueError):
        B.run_2way(Prob(2, 777, 48, ArraySource(bad)), Grid())
