"""The kernel plug-point drop-in (paper_1705_08210_b200.mingemm) against the
reference's own outputs (tests/golden/mingemm.json, written by running
propsim.mingemm: make_golden_mingemm.py).

CPU: operand checks (the reference's ValueError / DataError, raised before
any device work), the oracle pinned to the same vectors, the pivot-major ->
canonical reorder. GPU: every function bitwise against the golden vectors."""
import json
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

from conftest import cuda_available
from oracle import propsim_np as O

GOLD = Path(__file__).resolve().parent / "golden" / "mingemm.json"


@lru_cache(maxsize=1)
def gold():
    return json.loads(GOLD.read_text())


def _arr(hexes, shape, precision):
    ut, ft = (np.uint64, np.float64) if precision == "double" else (np.uint32, np.float32)
    a = np.array([int(h, 16) for h in hexes], dtype=ut).view(ft)
    return a.reshape(shape, order="F") if shape else a


def _bits(a):
    a = np.asfortranarray(np.asarray(a)).ravel(order="F")
    return [format(int(x), "x") for x in a.view(np.uint64 if a.dtype.itemsize == 8 else np.uint32)]


def _inputs(c):
    W = _arr(c["W"], (c["n_f"], c["m"]), c["precision"])
    V = _arr(c["V"], (c["n_f"], c["n"]), c["precision"])
    vj = _arr(c["vj"], None, c["precision"])
    return W, V, vj


def test_operand_checks_match_reference():
    from paper_1705_08210_b200 import mingemm as G
    from paper_1705_08210_b200.domain import DataError

    a = np.zeros((4, 3))
    with pytest.raises(ValueError, match="2-d"):
        G.mgemm_blocked(np.zeros(4), a)
    with pytest.raises(ValueError, match="field extents"):
        G.mgemm_blocked(a, np.zeros((5, 3)))
    with pytest.raises(ValueError, match="dtypes differ"):
        G.mgemm_blocked(a, a.astype(np.float32))
    with pytest.raises(ValueError, match="tile sides"):
        G.mgemm_blocked(a, a, tile=(0, 4))
    with pytest.raises(ValueError, match="float32 / float64"):
        G.mgemm_blocked(a.astype(np.int64), a.astype(np.int64))
    with pytest.raises(ValueError, match="2-d"):
        G.column_sums(np.zeros(3))
    with pytest.raises(ValueError, match="pivot column"):
        G.xj_columns(a, np.zeros(5))
    with pytest.raises(DataError):
        G.pack_bits(np.array([[0, 2], [1, 1]]))
    with pytest.raises(ValueError, match="row counts"):
        G.mgemm_bitpacked(G.BitMatrix(np.zeros((1, 2), np.uint64), 10),
                          G.BitMatrix(np.zeros((1, 2), np.uint64), 11))


def test_empty_operands_need_no_device():
    from paper_1705_08210_b200 import mingemm as G

    assert G.mgemm_blocked(np.zeros((5, 0)), np.zeros((5, 3))).shape == (0, 3)
    assert G.pair_numerators(np.zeros((5, 1))).shape == (0,)
    assert G.triple_min_numerators(np.zeros((5, 2))).shape == (0,)
    assert G.mgemm_bitpacked(G.BitMatrix(np.zeros((0, 2), np.uint64), 0),
                             G.BitMatrix(np.zeros((0, 3), np.uint64), 0)).tolist() == [[0] * 3] * 2


def test_oracle_matches_reference_mingemm():
    for c in gold()["dense"]:
        W, V, vj = _inputs(c)
        assert c["naive_equals_blocked"]
        assert _bits(O.mgemm(W, V)) == c["mgemm"]
        assert _bits(O.column_sums(V)) == c["column_sums"]
        assert _bits(np.minimum(vj[:, None], V)) == c["xj_columns"]
        n = V.shape[1]
        if n >= 3:
            T = O.triple_min(V)
            ids = O.triple_ids(n)
            assert _bits(T[ids]) == c["triple_min_numerators"]


def test_pivot_major_to_canonical_order():
    from paper_1705_08210_b200 import mingemm as G
    from paper_1705_08210_b200.domain import triple_index

    for n in (3, 4, 9, 17):
        order = G._canonical_order_of_box(n)
        want = [triple_index(i, j, k, n) for j in range(n) for i in range(j)
                for k in range(j + 1, n)]
        assert order.tolist() == want
        assert sorted(want) == list(range(n * (n - 1) * (n - 2) // 6))


gpu = pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")


@pytest.mark.gpu
@gpu
def test_dense_functions_bitwise_vs_reference():
    from paper_1705_08210_b200 import mingemm as G

    for c in gold()["dense"]:
        W, V, vj = _inputs(c)
        W0, V0 = W.copy(), V.copy()
        M = G.mgemm_blocked(W, V)
        assert M.flags.f_contiguous and M.shape == (c["m"], c["n"])
        assert _bits(M) == c["mgemm"]
        assert _bits(G.mgemm_naive(W, V)) == c["mgemm"]
        assert _bits(G.column_sums(V)) == c["column_sums"]
        assert _bits(G.xj_columns(V, vj)) == c["xj_columns"]
        assert _bits(G.pair_numerators(V)) == c["pair_numerators"]
        assert _bits(G.triple_min_numerators(V)) == c["triple_min_numerators"]
        assert _bits(W) == _bits(W0) and _bits(V) == _bits(V0)  # inputs not mutated


@pytest.mark.gpu
@gpu
def test_bitpacked_functions_vs_reference():
    from paper_1705_08210_b200 import mingemm as G

    for c in gold()["bits"]:
        A = np.asfortranarray(np.array(c["A"], dtype=np.float64).T)
        B = np.asfortranarray(np.array(c["B"], dtype=np.float64).T)
        pa, pb = G.pack_bits(A), G.pack_bits(B)
        assert [[format(int(x), "x") for x in col] for col in pa.words.T] == c["words_A"]
        assert pa.n_rows == c["n_f"] and pa.n_cols == c["m"]
        M = G.mgemm_bitpacked(pa, pb)
        assert M.dtype == np.int64 and M.flags.f_contiguous
        assert M.T.tolist() == c["counts"]
        # counts == the dense min-plus on 0/1 data (test_acceptance.py:240-257)
        assert (G.mgemm_blocked(A, B) == M).all()
    from paper_1705_08210_b200.domain import DataError

    with pytest.raises(DataError):
        G.pack_bits(np.array([[0.0, 0.5], [1.0, 1.0]]))


@pytest.mark.gpu
@gpu
def test_mgemm_larger_than_one_tile_vs_oracle():
    from paper_1705_08210_b200 import mingemm as G

    rng = np.random.default_rng(3)
    for dt in (np.float64, np.float32):
        W = np.asfortranarray(rng.random((333, 300)).astype(dt))
        V = np.asfortranarray(rng.random((333, 141)).astype(dt))
        assert _bits(G.mgemm_blocked(W, V)) == _bits(O.mgemm(W, V))
