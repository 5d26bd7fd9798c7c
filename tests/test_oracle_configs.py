"""The oracle against the reference's runs at the benchmarked configurations'
shapes (tests/golden/configs.json, written by make_golden_configs.py from
/root/reference): CPU only. 2-way cases without a field split are re-run
whole by the C restatement (checksum); every case's sampled records are
recomputed from their columns by the numpy restatement, bit for bit,
including the ascending-p_f fold of cfg5's field split."""
import itertools
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import c_oracle
from oracle import propsim_np as O

CASES = json.loads((Path(__file__).resolve().parent / "golden" / "configs.json")
                   .read_text())["cases"]


def _cols(c, cols):
    dt = np.float64 if c["precision"] == "double" else np.float32
    if c["kind"] == "uniform":
        return O.uniform_cols(c["seed"], c["n_f"], c["n_v"], cols, dt)
    return O.random_exact_cols(c["seed"], c["n_f"], c["n_v"], c["bits"], cols, dt)


def _tuples(arity, n_v):
    return list(itertools.combinations(range(n_v), arity))


@pytest.mark.parametrize("idx", range(len(CASES)),
                         ids=[f"{c['config']}-{c['kind']}-pf{c['grid']['n_pf']}"
                              f"pv{c['grid']['n_pv']}" for c in CASES])
def test_oracle_sampled_records(idx):
    c = CASES[idx]
    tuples = _tuples(c["arity"], c["n_v"])
    assert len(tuples) == c["records"]
    picks = [(int(p), tuples[int(p)]) for p in c["sample"]]
    cols = sorted({x for _, t in picks for x in t})
    at = {x: k for k, x in enumerate(cols)}
    V = _cols(c, cols)
    local = [tuple(at[x] for x in t) for _, t in picks]
    n_pf = c["grid"]["n_pf"]
    got = (O.pair_values_sampled_slabs(V, local, n_pf) if c["arity"] == 2
           else O.triple_values_sampled(V, local, n_pf))
    for (p, _), v in zip(picks, got):
        assert format(int(O.value_bits(np.asarray([v]))[0]), "x") == c["sample"][str(p)], p


@pytest.mark.parametrize("idx", [i for i, c in enumerate(CASES)
                                 if c["arity"] == 2 and c["grid"]["n_pf"] == 1
                                 and c["n_f"] <= 50000 and c["grid"]["n_pv"] == 1])
def test_oracle_whole_run_checksum(idx):
    c = CASES[idx]
    V = _cols(c, range(c["n_v"]))
    _, cks, deg = c_oracle.czek2(V)
    assert cks == c["checksum"]
    assert deg == c["degenerate"]


@pytest.mark.parametrize("idx", [i for i, c in enumerate(CASES) if c["arity"] == 3])
def test_triple_values_grid_matches_reference_samples(idx):
    """The grid recompute bench.py uses for its ~10^4-triple parity check of
    cfg4 (oracle.triple_values_grid) reproduces the reference's sampled 3-way
    values: every sampled triple of the golden case, as a 1 x 1 grid around
    its pivot, and the whole grid equals the per-triple recompute."""
    c = CASES[idx]
    tuples = _tuples(3, c["n_v"])
    n_pf = c["grid"]["n_pf"]
    for p, want in list(c["sample"].items())[:20]:
        i, j, k = tuples[int(p)]
        V = _cols(c, [i, j, k])
        got = O.triple_values_grid(V[:, :1], V[:, 1], V[:, 2:], n_pf)
        assert format(int(O.value_bits(got.ravel())[0]), "x") == want, p
    # a whole grid vs the per-triple restatement
    j = c["n_v"] // 2
    rows, cols = list(range(0, j, 7)), list(range(j + 1, c["n_v"], 5))
    V = _cols(c, rows + [j] + cols)
    a = len(rows)
    grid = O.triple_values_grid(V[:, :a], V[:, a], V[:, a + 1:], n_pf)
    per = O.triple_values_sampled(V, [(r, a, a + 1 + q) for r in range(a)
                                      for q in range(len(cols))], n_pf)
    assert (O.value_bits(grid.ravel()) == O.value_bits(per)).all()
