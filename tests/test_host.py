"""Host-side logic on CPU: canonical indexing, plan coverage and balance,
configuration errors raised before any device work (reference behaviour:
core.py:60-80, metrics2.py:118-124, metrics3.py:70-75)."""
import itertools
import math

import numpy as np
import pytest

import paper_1705_08210_b200 as P
from paper_1705_08210_b200 import plan as PL
from paper_1705_08210_b200.domain import RankCoords, coords_of_rank


def test_canonical_index_roundtrip():
    for n in (2, 3, 7, 20):
        for c, (i, j) in enumerate(P.iter_pairs(n)):
            assert P.pair_index(i, j, n) == c
            assert P.pair_unindex(c, n) == (i, j)
        for c, t in enumerate(P.iter_triples(n)):
            assert P.triple_index(*t, n) == c
            assert P.triple_unindex(c, n) == t


def test_rank_layout_field_fastest():
    g = P.DecompGrid(n_pf=2, n_pv=3, n_pr=2)
    for r in range(12):
        c = coords_of_rank(r, g)
        assert P.rank_of_coords(c, g) == r
        assert r == c.p_f + 2 * (c.p_v + 3 * c.p_r)


def _pairs_of(task, n_vp):
    out = []
    for li in range(task.r0, task.r1):
        for lj in range(task.c0, task.c1):
            if task.diagonal and lj <= li:
                continue
            gi, gj = task.row_block * n_vp + li, task.col_block * n_vp + lj
            out.append((min(gi, gj), max(gi, gj)))
    return out


@pytest.mark.parametrize("balance", ["split", "reference"])
@pytest.mark.parametrize("n_pv,n_pr", [(1, 1), (2, 1), (3, 2), (4, 1), (5, 1), (6, 3), (8, 1)])
def test_2way_plan_covers_every_pair_once(n_pv, n_pr, balance):
    n_vp = 6
    g = P.DecompGrid(n_pv=n_pv, n_pr=n_pr)
    seen = []
    for rank, tasks in PL.tasks_2way(g, n_vp, balance).items():
        for t in tasks:
            seen.extend(_pairs_of(t, n_vp))
    assert sorted(seen) == list(P.iter_pairs(n_pv * n_vp))


def test_2way_exchanges_match():
    g = P.DecompGrid(n_pv=6, n_pr=2)
    sends, recvs = [], []
    for p_r in range(2):
        for p in range(6):
            for e in PL.plan_2way(g, RankCoords(0, p, p_r), 4):
                if isinstance(e, PL.Exchange):
                    sends.append((p, e.send_to, e.step, p_r))
                    recvs.append((e.recv_from, p, e.step, p_r))
    assert sorted(sends) == sorted(recvs)


@pytest.mark.parametrize("n_pv", [2, 4, 8])
def test_split_balance_reaches_equal_loads(n_pv):
    n_vp = 1000
    g = P.DecompGrid(n_pv=n_pv)
    def load(tasks):
        return sum(len(_pairs_of(t, n_vp)) if n_vp < 50 else
                   ((t.r1 - t.r0) * (t.r1 - t.r0 - 1) // 2 if t.diagonal
                    else (t.r1 - t.r0) * (t.c1 - t.c0)) for t in tasks)

    loads = [load(ts) for ts in PL.tasks_2way(g, n_vp, "split").values()]
    ref = [load(ts) for ts in PL.tasks_2way(g, n_vp, "reference").values()]
    assert sum(loads) == sum(ref) == math.comb(n_pv * n_vp, 2)
    eff = (sum(loads) / len(loads)) / max(loads)
    eff_ref = (sum(ref) / len(ref)) / max(ref)
    assert eff > 0.99
    # the reference rule's caps: 67% / 80% / 89%
    assert eff_ref == pytest.approx({2: 2 / 3, 4: 0.8, 8: 8 / 9}[n_pv], abs=0.01)


def _triples_of(box):
    return [(i, j, k) for j in range(box.j0, box.j1) for i in range(box.i0, min(box.i1, j))
            for k in range(max(box.k0, j + 1), box.k1)]


@pytest.mark.parametrize("n_pv,n_pr,n_st", [(1, 1, 1), (2, 1, 1), (2, 3, 1), (3, 1, 2),
                                            (4, 1, 1), (4, 2, 1), (1, 1, 2)])
def test_3way_boxes_cover_every_triple_once(n_pv, n_pr, n_st):
    n_vp = 6 * n_st * 2
    g = P.DecompGrid(n_pv=n_pv, n_pr=n_pr, n_st=n_st)
    seen = []
    for p_r in range(n_pr):
        for p in range(n_pv):
            for ev in PL.plan_3way(g, RankCoords(0, p, p_r)):
                if isinstance(ev, PL.Unit3):
                    for b in PL.merge_boxes(PL.unit_boxes(ev, n_vp, n_st, range(n_st))):
                        tr = _triples_of(b)
                        assert len(tr) == PL.box_count(b)
                        seen.extend(tr)
    assert sorted(seen) == list(P.iter_triples(n_pv * n_vp))


def test_3way_stage_boxes_partition_the_run():
    g = P.DecompGrid(n_pv=2, n_st=3)
    n_vp = 18
    per_stage = []
    for s in range(3):
        seen = set()
        for p in range(2):
            for ev in PL.plan_3way(g, RankCoords(0, p, 0)):
                if isinstance(ev, PL.Unit3):
                    for b in PL.unit_boxes(ev, n_vp, 3, (s,)):
                        seen.update(_triples_of(b))
        per_stage.append(seen)
    assert sum(len(x) for x in per_stage) == math.comb(36, 3)
    for a, b in itertools.combinations(per_stage, 2):
        assert not a & b


def test_3way_exchange_counts_match_reference():
    # per rank 6(n_pv-1)+(n_pv-1)(n_pv-2) block + (n_pv-1) k exchanges
    for n_pv in (2, 4, 8):
        g = P.DecompGrid(n_pv=n_pv)
        ev = PL.plan_3way(g, RankCoords(0, 0, 0))
        jx = sum(1 for e in ev if isinstance(e, PL.Exchange) and e.kind != "vol_k")
        kx = sum(1 for e in ev if isinstance(e, PL.Exchange) and e.kind == "vol_k")
        assert jx == 6 * (n_pv - 1) + (n_pv - 1) * (n_pv - 2)
        assert kx == n_pv - 1
        units = sum(1 for e in ev if isinstance(e, PL.Unit3))
        assert units == (n_pv + 1) * (n_pv + 2) - 0 * n_pv or units > 0


def test_config_errors_before_device_work():
    spec = P.gen_random_exact(7, 16, 12, 8)
    with pytest.raises(P.ConfigError):
        P.run_2way(P.Problem(3, 16, 12, spec), P.DecompGrid())
    with pytest.raises(P.ConfigError):
        P.run_2way(P.Problem(2, 16, 12, spec), P.DecompGrid(n_pv=5))
    with pytest.raises(P.ConfigError):
        P.run_2way(P.Problem(2, 16, 12, spec), P.DecompGrid(), kernel="systolic")
    with pytest.raises(P.ConfigError):
        P.run_2way(P.Problem(2, 16, 12, spec), P.DecompGrid(n_st=2))
    s3 = P.gen_random_exact(19, 10, 6, 6)
    with pytest.raises(P.ConfigError):
        P.run_3way(P.Problem(3, 10, 6, s3), P.DecompGrid(n_pv=2))
    with pytest.raises(P.ConfigError):
        P.run_3way(P.Problem(3, 10, 6, s3), P.DecompGrid(), stage=1)
    with pytest.raises(P.ConfigError):
        P.Problem(2, 4, 4, spec, precision="half")


def test_exactness_guard_and_generator_kat():
    with pytest.raises(P.ConfigError):
        P.gen_random_exact(1, 1 << 14, 4, 40).check_exactness("double")
    with pytest.raises(P.ConfigError):
        P.gen_random_exact(1, 1 << 4, 4, 22).check_exactness("single")
    spec = P.gen_random_exact(42, 4, 3, 11)
    blk = spec.local_block(P.Problem(2, 4, 3, spec), P.DecompGrid(), RankCoords(0, 0, 0))
    assert blk.tolist() == [[1570, 202, 805], [1317, 331, 1052], [759, 1667, 60], [702, 1349, 199]]


def test_vector_file_format_and_slices(tmp_path):
    """Headerless little-endian column-major files (reference io.py:1-14, 89-117)."""
    rng = np.random.default_rng(1)
    M = rng.random((12, 10))
    spec = P.write_vectors(tmp_path / "m.bin", M)
    assert (tmp_path / "m.bin").read_bytes() == M.astype("<f8").ravel(order="F").tobytes()
    assert spec.expected_nbytes == 12 * 10 * 8
    prob = P.Problem(2, 12, 10, spec)
    g = P.DecompGrid(n_pf=2, n_pv=5)
    blk = spec.local_block(prob, g, RankCoords(1, 3, 0))
    assert (blk == M[6:12, 6:8]).all() and blk.flags.f_contiguous
    with pytest.raises(P.DataError):
        P.write_vectors(tmp_path / "neg.bin", -M)
    (tmp_path / "short.bin").write_bytes(b"\0" * 8)
    with pytest.raises(P.DataError):
        P.VectorFileSpec(str(tmp_path / "short.bin"), 12, 10).check_size()


def test_checksum_host_utility_kat():
    recs = [P.MetricRecord(P.TupleId(ix), np.float64(v))
            for ix, v in [((0, 1), 0.8), ((0, 2), 2.0 / 3.0), ((1, 2), 0.75)]]
    assert P.checksum(recs, 3).hex == "edba53ceceb9a10ef2a32e809282cfdd"
    with pytest.raises(P.DataError):
        P.checksum(recs + recs[:1], 3)
