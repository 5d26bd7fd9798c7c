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
