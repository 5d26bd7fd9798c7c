"""Metric output directories (row f1, reference io.py): ownership tables and
the file writer against directories the REFERENCE wrote (golden sha256 per
file + manifest, tests/golden/make_golden.py). CPU only: the run results fed
to the writer are the oracle's values, which are pinned bitwise to the
reference's runs in test_oracle_golden.py."""
import hashlib
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import pytest

from conftest import golden
from oracle import propsim_np as O
from paper_1705_08210_b200 import output as OUT
from paper_1705_08210_b200.domain import DataError, DecompGrid, TupleId, triple_unindex_np
from paper_1705_08210_b200.synthetic import Checksum128

# fields a drop-in caller does not control: they name this engine, not the reference's
OURS_ONLY = {"transport", "kernel"}


@pytest.mark.parametrize("case", golden()["owners"], ids=lambda c: f"{c['arity']}w-{c['grid']}")
def test_owner_ranks_match_reference(case):
    grid = DecompGrid(**case["grid"])
    canon = np.arange(math.comb(case["n_v"], case["arity"]), dtype=np.int64)
    rank, stage = OUT.owner_ranks(case["arity"], canon, case["n_v"], grid)
    assert rank.tolist() == case["rank"]
    if case["arity"] == 3:
        assert stage.tolist() == case["stage"]


def test_owned_canonical_partitions_all_tuples():
    for arity, n_v, g in ((2, 30, DecompGrid(n_pv=5, n_pr=4)),
                          (3, 36, DecompGrid(n_pv=3, n_pr=5, n_st=2))):
        parts = [OUT.owned_canonical(r, arity=arity, n_v=n_v, grid=g, chunk=97)
                 for r in range(g.n_p)]
        allidx = np.concatenate(parts)
        assert np.array_equal(np.sort(allidx), np.arange(math.comb(n_v, arity)))
        assert all((np.diff(p) > 0).all() for p in parts)


def test_quantize_rules():
    assert [OUT.quantize_byte(v) for v in (-1.0, 0.0, 0.5 / 255, 0.5, 1.0, 7.0)] == \
        [0, 0, 1, 128, 255, 255]
    with pytest.raises(DataError):
        OUT.quantize_values(np.array([0.2, np.nan]))
    assert OUT.dequantize_byte(255) == 1.0
    assert OUT.dequantize_byte(51, "single") == np.float32(0.2)


def test_manifest_round_trip_and_errors(tmp_path):
    p = tmp_path / "m.txt"
    OUT.write_manifest(p, {"a": 1, "b": "x=y", "c": ""})
    assert OUT.read_manifest(p) == {"a": "1", "b": "x=y", "c": ""}
    with pytest.raises(DataError):
        OUT.write_manifest(p, {"a=b": 1})
    with pytest.raises(DataError):
        OUT.write_manifest(p, {"a": "x\ny"})
    p.write_text("ok=1\nbroken\n")
    with pytest.raises(DataError):
        OUT.read_manifest(p)


class _Records:
    """Host stand-in for LazyRecords: canonical indices + values."""

    def __init__(self, idx, vals):
        self.canonical_indices, self.values = idx, vals

    def __len__(self):
        return len(self.values)


@dataclass
class _Result:
    arity: int
    n_f: int
    n_v: int
    precision: str
    metric: str
    grid: object
    transport: str
    kernel: str
    records: object
    checksum: object
    degenerate_count: int
    stages: tuple | None


def oracle_result(case):
    """RunResult-shaped object holding the oracle's values for a golden case."""
    dt = np.float64 if case["precision"] == "double" else np.float32
    if case["kind"] == "uniform":
        V = O.uniform(case["seed"], case["n_f"], case["n_v"], dt)
    else:
        V = O.random_exact(case["seed"], case["n_f"], case["n_v"], case["bits"], dt)
    grid = DecompGrid(**case["grid"])
    vals, zero = O.values_field_split(V, case["arity"], grid.n_pf)
    idx = np.arange(len(vals), dtype=np.int64)
    stages = None
    if case["stage"] is not None:
        stages = (case["stage"],)
        _, st = OUT.triple_owner_ranks(*triple_unindex_np(idx, case["n_v"]), case["n_v"], grid)
        keep = st == case["stage"]
        idx, vals, zero = idx[keep], vals[keep], zero[keep]
    cks = Checksum128(O.checksum(idx, vals))
    return _Result(case["arity"], case["n_f"], case["n_v"], case["precision"], case["metric"],
                   grid, "local", "b200", _Records(idx, vals), cks, int(zero.sum()), stages)


def check_directory(directory, case):
    """Every metrics_<r>.bin byte-identical to the reference's; manifest equal
    except the engine-naming keys."""
    for r, (size, digest) in case["files"].items():
        blob = Path(directory, f"metrics_{r}.bin").read_bytes()
        assert len(blob) == size, (r, case["grid"])
        assert hashlib.sha256(blob).hexdigest() == digest, (r, case["grid"], case["mode"])
    got = OUT.read_manifest(Path(directory, "manifest.txt"))
    want = case["manifest"]
    assert {k: v for k, v in got.items() if k not in OURS_ONLY} == \
        {k: v for k, v in want.items() if k not in OURS_ONLY}
    assert set(got) == set(want)


@pytest.mark.parametrize("case", golden()["outputs"],
                         ids=lambda c: f"{c['arity']}w-{c['precision']}-{c['mode']}-{c['grid']}")
def test_writer_matches_reference_directory(case, tmp_path):
    res = oracle_result(case)
    OUT.write_run_output(res, OUT.MetricOutputSpec(str(tmp_path), case["mode"]),
                         source={"kind": case["kind"]})
    check_directory(tmp_path, case)
    entries, per_rank = OUT.read_run_output(tmp_path)
    got = sorted((rec.id.canonical_index(case["n_v"]), rec.value)
                 for recs in per_rank.values() for rec in recs)
    assert [g[0] for g in got] == res.records.canonical_indices.tolist()
    vals = np.array([g[1] for g in got])
    if case["mode"] == "full":
        assert np.array_equal(vals, res.records.values)
    else:
        dt = res.records.values.dtype.type
        assert np.array_equal(vals, OUT.quantize_values(res.records.values).astype(dt) / dt(255))
    _, idx, arr = OUT.read_run_values(tmp_path)
    assert np.array_equal(idx, res.records.canonical_indices)
    assert np.allclose(arr, vals)


def test_reconstruct_index_and_write_metrics(tmp_path):
    g = DecompGrid(n_pv=2, n_pr=3)
    owned = list(OUT.owned_tuples(4, arity=3, n_v=24, grid=g))
    assert OUT.reconstruct_index(4, 0, arity=3, n_v=24, grid=g) == owned[0]
    assert OUT.reconstruct_index(4, len(owned) - 1, arity=3, n_v=24, grid=g) == owned[-1]
    with pytest.raises(IndexError):
        OUT.reconstruct_index(4, len(owned), arity=3, n_v=24, grid=g)
    with pytest.raises(IndexError):
        OUT.reconstruct_index(0, -1, arity=2, n_v=24, grid=g)
    from paper_1705_08210_b200.domain import MetricRecord

    spec = OUT.MetricOutputSpec(str(tmp_path), "full")
    recs = [MetricRecord(t, 0.25 * (n % 4)) for n, t in enumerate(owned)]
    OUT.write_metrics(list(reversed(recs)), spec, 4)
    back = OUT.read_metrics(spec, 4, arity=3, n_v=24, grid=g)
    assert [(r.id, float(r.value)) for r in back] == [(r.id, r.value) for r in recs]
    Path(spec.rank_path(4)).write_bytes(b"\0" * 3)
    with pytest.raises(DataError):
        OUT.read_metrics(spec, 4, arity=3, n_v=24, grid=g)
    assert TupleId((0, 1)) == OUT.reconstruct_index(0, 0, arity=2, n_v=24, grid=g)


@pytest.mark.parametrize("case", golden()["owners"], ids=lambda c: f"{c['arity']}w-{c['grid']}")
def test_planner_owners_match_reference(case):
    """The planner-walking scalar owns_pair / owns_triple (plan.py) agree with
    the reference's owners on a sample of tuples."""
    from paper_1705_08210_b200.domain import pair_unindex, triple_unindex
    from paper_1705_08210_b200.plan import owns_pair, owns_triple

    grid = DecompGrid(**case["grid"])
    n_v = case["n_v"]
    for c in range(0, len(case["rank"]), 41):
        if case["arity"] == 2:
            assert owns_pair(*pair_unindex(c, n_v), n_v, grid)[0] == case["rank"][c]
        else:
            r, st, _ = owns_triple(*triple_unindex(c, n_v), n_v, grid)
            assert (r, st) == (case["rank"][c], case["stage"][c])
