"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
runs and the CPU oracle. Bit-exact everywhere: the kernels keep the
reference's per-element ascending-q summation order, so even general FP
data matches bitwise."""
import json
import math
from pathlib import Path

import numpy as np
import pytest

from conftest import cuda_available, golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _api():
    import paper_1705_08210_b200 as P

    return P


class ArraySource:
    """Reference tests/conftest.py:17-26 shape, over one global matrix."""

    def __init__(self, matrix):
        self.matrix = np.asarray(matrix)

    def local_block(self, problem, grid, coords):
        P = _api()
        from paper_1705_08210_b200.domain import field_range, vector_range

        f0, f1 = field_range(grid, coords.p_f, problem.n_f)
        v0, v1 = vector_range(grid, coords.p_v, problem.n_v)
        return self.matrix[f0:f1, v0:v1]


def _source(case):
    P = _api()
    if case["kind"] == "random-exact":
        return P.gen_random_exact(case["seed"], case["n_f"], case["n_v"], case["bits"])
    if case["kind"] == "analytic":
        return P.gen_analytic(0, case["n_f"], case["n_v"])
    if case["kind"] == "uniform":
        return P.gen_uniform(case["seed"], case["n_f"], case["n_v"])
    return ArraySource(np.asfortranarray(np.asarray(case["matrix"], dtype=np.float64)))


def _run(case, stage=None):
    P = _api()
    prob = P.Problem(case["arity"], case["n_f"], case["n_v"], _source(case), case["precision"],
                     case.get("metric", "czekanowski"))
    grid = P.DecompGrid(**case["grid"])
    if case["arity"] == 2:
        return P.run_2way(prob, grid)
    return P.run_3way(prob, grid, stage=stage)


CASES = golden()["cases"]


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_golden_case(idx):
    case = CASES[idx]
    res = _run(case, case.get("stage"))
    assert len(res.records) == case["records"]
    assert res.checksum.hex == case["checksum"]
    assert res.degenerate_count == case["degenerate"]
    if "value_bits" in case:
        from oracle import propsim_np as O

        got = [format(int(b), "x") for b in O.value_bits(res.records.values)]
        assert got == case["value_bits"]
        assert [r.degenerate for r in res.records] == case["degenerate_flags"]
    if "ids" in case:
        assert [list(r.id.indices) for r in res.records] == case["ids"]
        assert res.stages == (case["stage"],)
    if case.get("metric") == "sorenson":
        assert res.kernel == case["kernel"] == "bitpacked"


def test_sorenson_bitpacked_equals_dense_and_rejects_non_binary():
    """f3: the AND+POPC kernel gives the dense kernel's bits on 0/1 data, for
    n_f around word boundaries; non-0/1 input raises DataError (pack_bits)."""
    P = _api()
    for n_f in (1, 31, 32, 33, 1023, 1025, 4096):
        spec = P.gen_random_exact(5, n_f, 150, 1)
        for prec in ("double", "single"):
            a = P.run_2way(P.Problem(2, n_f, 150, spec, prec, "sorenson"), P.DecompGrid(n_pv=2))
            b = P.run_2way(P.Problem(2, n_f, 150, spec, prec), P.DecompGrid(), kernel="blocked")
            assert a.kernel == "bitpacked" and a.checksum == b.checksum, (n_f, prec)
            assert (a.records.values.view(np.uint8) == b.records.values.view(np.uint8)).all()
    with pytest.raises(P.DataError):
        P.run_2way(P.Problem(2, 16, 12, P.gen_random_exact(7, 16, 12, 3), metric="sorenson"),
                   P.DecompGrid())


def test_records_canonical_order_and_types():
    P = _api()
    spec = P.gen_random_exact(7, 16, 12, 8)
    res = P.run_2way(P.Problem(2, 16, 12, spec), P.DecompGrid(n_pv=3))
    assert [r.id.indices for r in res.records] == list(P.iter_pairs(12))
    assert isinstance(res.records[0].value, np.float64)
    r3 = P.run_3way(P.Problem(3, 8, 12, P.gen_random_exact(4, 8, 12, 5)), P.DecompGrid(n_pv=2))
    assert [r.id.indices for r in r3.records] == list(P.iter_triples(12))


def _rand(rng, n_f, n, dt):
    return np.asfortranarray(rng.random((n_f, n)).astype(dt))


@pytest.mark.parametrize("precision", ["double", "single"])
def test_mgemm_raw_fuzz_vs_oracle(precision):
    """psim_mgemm (col-major, rectangular and symmetric) == sequential-q oracle, bitwise,
    over ragged shapes (n_f not a multiple of the 128-B chunk, partial tiles)."""
    import torch

    from oracle import propsim_np as O
    from paper_1705_08210_b200 import device as D

    rng = np.random.default_rng(11)
    dt = np.float64 if precision == "double" else np.float32
    code = D.code_of(precision)
    for trial in range(12):
        n_f = int(rng.integers(1, 300))
        m = int(rng.integers(1, 300))
        n = int(rng.integers(1, 300))
        W = _rand(rng, n_f, m, dt)
        V = _rand(rng, n_f, n, dt)
        bw = D.block_from_host(torch.from_numpy(np.ascontiguousarray(W.T)), n_f, 0, precision, "cuda")
        bv = D.block_from_host(torch.from_numpy(np.ascontiguousarray(V.T)), n_f, 0, precision, "cuda")
        out = torch.zeros((n, m), dtype=D.torch_dtype(precision), device="cuda")
        D.mgemm_square(code, bw, bv, out, symmetric=False)
        got = np.ascontiguousarray(out.cpu().numpy().T)
        want = np.ascontiguousarray(O.mgemm(W, V))
        assert (got.view(np.uint8) == want.view(np.uint8)).all(), trial
        outs = torch.zeros((m, m), dtype=D.torch_dtype(precision), device="cuda")
        D.mgemm_square(code, bw, bw, outs, symmetric=True)
        assert (outs.cpu().numpy().T == O.mgemm(W, W)).all()


@pytest.mark.parametrize("precision", ["double", "single"])
def test_column_sums_equal_mgemm_diagonal(precision):
    import torch

    from paper_1705_08210_b200 import device as D

    rng = np.random.default_rng(4)
    dt = np.float64 if precision == "double" else np.float32
    V = _rand(rng, 333, 77, dt)
    b = D.block_from_host(torch.from_numpy(np.ascontiguousarray(V.T)), 333, 0, precision, "cuda")
    s = D.column_sums(b).cpu().numpy()
    out = torch.zeros((77, 77), dtype=D.torch_dtype(precision), device="cuda")
    D.mgemm_square(D.code_of(precision), b, b, out, symmetric=True)
    assert (np.diag(out.cpu().numpy()) == s).all()


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("grid", [dict(), dict(n_pv=2), dict(n_pv=4, n_pr=2), dict(n_pf=2, n_pv=3)])
def test_uniform_2way_bitwise_vs_oracle(precision, grid):
    """General FP data, several grids: identical bits to the sequential oracle
    (the n_pf=2 grid folds per-slab partials in ascending p_f, which the
    oracle reproduces by folding its own per-slab numerators)."""
    from oracle import propsim_np as O

    P = _api()
    n_f, n_v = 1002, 372
    spec = P.gen_uniform(99, n_f, n_v)
    res = P.run_2way(P.Problem(2, n_f, n_v, spec, precision), P.DecompGrid(**grid))
    dt = np.float64 if precision == "double" else np.float32
    V = O.uniform(99, n_f, n_v, dt)
    n_pf = grid.get("n_pf", 1)
    if n_pf == 1:
        want, _ = O.values_2way(V)
    else:
        w = n_f // n_pf
        Ns = [O.mgemm(V[p * w:(p + 1) * w], V[p * w:(p + 1) * w]) for p in range(n_pf)]
        Ss = [O.column_sums(V[p * w:(p + 1) * w]) for p in range(n_pf)]
        N, s = Ns[0], Ss[0]
        for a, b in zip(Ns[1:], Ss[1:]):
            N, s = N + a, s + b
        iu, ju = np.triu_indices(n_v, 1)
        d = s[iu] + s[ju]
        want = (dt(2) * N[iu, ju]) / d
    assert (res.records.values.view(np.uint8) == want.view(np.uint8)).all()
    assert res.checksum.hex == O.checksum_hex(np.arange(len(want)), want)


@pytest.mark.parametrize("precision", ["double", "single"])
def test_uniform_3way_bitwise_vs_oracle(precision):
    from oracle import propsim_np as O

    P = _api()
    n_f, n_v = 301, 48
    dt = np.float64 if precision == "double" else np.float32
    want, _ = O.values_3way(O.uniform(8, n_f, n_v, dt))
    for grid in (P.DecompGrid(), P.DecompGrid(n_pv=2), P.DecompGrid(n_pv=4, n_pr=2),
                 P.DecompGrid(n_pv=2, n_st=2)):
        res = P.run_3way(P.Problem(3, n_f, n_v, P.gen_uniform(8, n_f, n_v), precision), grid)
        assert (res.records.values.view(np.uint8) == want.view(np.uint8)).all(), grid


def test_large_2way_sampled_parity_and_properties():
    """Full-width field axis (cfg2's n_f = 20000) on 8192 vectors: checksum of
    the device run equals the checksum of its own values (host recompute),
    values lie in [0, 1], and 4000 random pairs recomputed from their
    columns alone (SURVEY 8d recipe) match bitwise."""
    from oracle import propsim_np as O

    P = _api()
    n_f, n_v = 20000, 8192
    spec = P.gen_random_exact(2026, n_f, n_v, 20)
    res = P.run_2way(P.Problem(2, n_f, n_v, spec), P.DecompGrid())
    vals = res.records.values
    assert len(vals) == math.comb(n_v, 2)
    assert res.checksum.hex == O.checksum_hex(np.arange(len(vals)), vals)
    assert float(vals.min()) >= 0.0 and float(vals.max()) <= 1.0
    rng = np.random.default_rng(1)
    pairs = set()
    while len(pairs) < 1000:
        i, j = sorted(int(x) for x in rng.integers(0, n_v, size=2))
        if i != j:
            pairs.add((i, j))
    pairs = sorted(pairs)
    cols = sorted({c for p in pairs for c in p})
    pos = {c: t for t, c in enumerate(cols)}
    V = O.random_exact_cols(2026, n_f, n_v, 20, cols)
    got = O.pair_values_sampled(V, [(pos[i], pos[j]) for i, j in pairs])
    idx = [P.pair_index(i, j, n_v) for i, j in pairs]
    assert (vals[idx].view(np.uint64) == got.view(np.uint64)).all()


def _sample(rng, n_v, count, arity):
    out = set()
    while len(out) < count:
        t = tuple(sorted(int(x) for x in rng.choice(n_v, size=arity, replace=False)))
        out.add(t)
    return sorted(out)


def _recompute(P, O, kind, seed, n_f, n_v, tuples, precision, n_pf=1, bits=20):
    dt = np.float64 if precision == "double" else np.float32
    cols = sorted({c for t in tuples for c in t})
    pos = {c: p for p, c in enumerate(cols)}
    if kind == "uniform":
        V = O.uniform_cols(seed, n_f, n_v, cols, dt)
    else:
        V = O.random_exact_cols(seed, n_f, n_v, bits, cols, dt)
    local = [tuple(pos[c] for c in t) for t in tuples]
    if len(tuples[0]) == 2:
        return O.pair_values_sampled_slabs(V, local, n_pf)
    return O.triple_values_sampled(V, local, n_pf)


def test_large_fp32_2way_sampled_uniform():
    """cfg3's field width (n_f = 50000, FP32) on general FP data: sampled pairs
    bitwise equal to the column-only sequential recompute; checksum equals the
    checksum of the returned values."""
    from oracle import propsim_np as O

    P = _api()
    n_f, n_v = 50000, 2048
    res = P.run_2way(P.Problem(2, n_f, n_v, P.gen_uniform(3, n_f, n_v), "single"), P.DecompGrid())
    vals = res.records.values
    assert res.checksum.hex == O.checksum_hex(np.arange(len(vals)), vals)
    pairs = _sample(np.random.default_rng(2), n_v, 300, 2)
    got = _recompute(P, O, "uniform", 3, n_f, n_v, pairs, "single")
    idx = [P.pair_index(i, j, n_v) for i, j in pairs]
    assert (vals[idx].view(np.uint32) == got.view(np.uint32)).all()


def test_large_3way_sampled_and_stage_tiling():
    """cfg4's field width (n_f = 10000, FP64), n_v = 600 (3.6e7 triples):
    sampled triples bitwise vs the column-only recompute; the two stages of
    n_st = 2 partition the run and their checksums add up to the full one."""
    from oracle import propsim_np as O

    P = _api()
    n_f, n_v = 10000, 600
    prob = P.Problem(3, n_f, n_v, P.gen_uniform(21, n_f, n_v), "double")
    full = P.run_3way(prob, P.DecompGrid())
    vals = full.records.values
    assert len(vals) == math.comb(n_v, 3)
    assert full.checksum.hex == O.checksum_hex(np.arange(len(vals)), vals)
    triples = _sample(np.random.default_rng(5), n_v, 200, 3)
    got = _recompute(P, O, "uniform", 21, n_f, n_v, triples, "double")
    idx = [P.triple_index(*t, n_v) for t in triples]
    assert (vals[idx].view(np.uint64) == got.view(np.uint64)).all()
    parts = [P.run_3way(prob, P.DecompGrid(n_st=2), stage=s, keep_values=False) for s in (0, 1)]
    assert P.combine_checksums([p.checksum for p in parts]) == full.checksum
    assert parts[0].records.__len__() + parts[1].records.__len__() == len(vals)


def test_3way_packed_pair_tiles_sampled():
    """FP64 boxes pair pivot j with its mate (box3_plan.cuh): the ragged rows
    [128R, j) and leading columns (j, 128R + 128) of two pivots share one
    tile. Triples inside one 128-block are exactly those cells; they, plus
    random ones, must equal the column-only recompute bit for bit, and the
    checksum must equal the checksum of all returned values."""
    from oracle import propsim_np as O

    P = _api()
    n_f, n_v = 700, 384
    prob = P.Problem(3, n_f, n_v, P.gen_uniform(8, n_f, n_v), "double")
    res = P.run_3way(prob, P.DecompGrid())
    vals = res.records.values
    assert res.checksum.hex == O.checksum_hex(np.arange(len(vals)), vals)
    rng = np.random.default_rng(17)
    triples = set(_sample(rng, n_v, 150, 3))
    while len(triples) < 450:  # i < j < k all inside one 128-block
        blk = int(rng.integers(0, n_v // 128))
        t = tuple(sorted(int(x) for x in rng.choice(128, size=3, replace=False) + 128 * blk))
        triples.add(t)
    triples = sorted(triples)
    got = _recompute(P, O, "uniform", 8, n_f, n_v, triples, "double")
    idx = [P.triple_index(*t, n_v) for t in triples]
    assert (vals[idx].view(np.uint64) == got.view(np.uint64)).all()
    # the same triples from a run whose boxes cannot pair (k range not aligned
    # with i): per-pivot tiling only
    part = P.run_3way(prob, P.DecompGrid(n_pv=2, n_st=2), stage=1)
    pv = dict(zip(part.records.canonical_indices.tolist(), part.records.values.tolist()))
    for t, v in zip(idx, vals[idx]):
        if t in pv:
            assert np.float64(pv[t]).view(np.uint64) == np.float64(v).view(np.uint64)


def test_large_field_split_sampled():
    """A cfg5-like deep field axis (n_f = 1,000,000 FP64) split over n_pf = 4
    slabs (ordered fold): sampled pairs bitwise vs the per-slab recompute."""
    from oracle import propsim_np as O

    P = _api()
    n_f, n_v = 1_000_000, 256
    res = P.run_2way(P.Problem(2, n_f, n_v, P.gen_uniform(7, n_f, n_v), "double"),
                     P.DecompGrid(n_pf=4))
    vals = res.records.values
    pairs = _sample(np.random.default_rng(9), n_v, 60, 2)
    got = _recompute(P, O, "uniform", 7, n_f, n_v, pairs, "double", n_pf=4)
    idx = [P.pair_index(i, j, n_v) for i, j in pairs]
    assert (vals[idx].view(np.uint64) == got.view(np.uint64)).all()
    assert res.checksum.hex == O.checksum_hex(np.arange(len(vals)), vals)


@pytest.mark.parametrize("mode", ["direct", "bands"])
def test_band_launches_equal_single_launch(mode, monkeypatch):
    """host_values=True: zero-copy ("direct": the kernel stores into pinned
    host memory) or row bands with overlapped D2H copies ("bands"); values
    and checksum must equal the device-resident run, for a single slab, a
    circulant grid and a field split."""
    monkeypatch.setenv("PSIM_HOST_OUTPUT", mode)
    P = _api()
    spec = P.gen_uniform(4, 3000, 3000)
    prob = P.Problem(2, 3000, 3000, spec, "double")
    for grid in (P.DecompGrid(), P.DecompGrid(n_pv=3, n_pr=2), P.DecompGrid(n_pf=2, n_pv=2)):
        a = P.run_2way(prob, grid)
        b = P.run_2way(prob, grid, host_values=True)
        assert a.checksum == b.checksum
        assert (a.records.values.view(np.uint64) == b.records.values.view(np.uint64)).all()


@pytest.mark.parametrize("mode", ["direct", "bands"])
def test_3way_streamed_host_values_equal_device_run(mode, monkeypatch):
    """run_3way(host_values=True) writes each box's values to pinned host
    memory (zero-copy, or pivot-range chunks copied while the next computes);
    results must equal the plain run."""
    monkeypatch.setenv("PSIM_HOST_OUTPUT", mode)
    P = _api()
    prob = P.Problem(3, 500, 96, P.gen_uniform(12, 500, 96), "single")
    for grid in (P.DecompGrid(), P.DecompGrid(n_pv=2, n_st=2)):
        a = P.run_3way(prob, grid)
        b = P.run_3way(prob, grid, host_values=True)
        assert a.checksum == b.checksum
        assert (a.records.values.view(np.uint32) == b.records.values.view(np.uint32)).all()


def test_vector_file_input_streams_to_device(tmp_path):
    """f4: runs fed from a raw vector file (streamed through pinned chunks into
    HBM) equal runs on the same data generated in HBM, for vector and field
    slabs; bad files raise DataError like the reference (io.py:78-117)."""
    from oracle import propsim_np as O
    from paper_1705_08210_b200 import vectorfile

    P = _api()
    n_f, n_v = 640, 96
    for precision, dt in (("double", np.float64), ("single", np.float32)):
        V = O.uniform(17, n_f, n_v, dt)
        spec = P.write_vectors(tmp_path / f"v_{precision}.bin", V, precision)
        old = vectorfile.CHUNK_BYTES
        vectorfile.CHUNK_BYTES = n_f * 8 * 7  # several chunks per slab
        try:
            for grid in (P.DecompGrid(), P.DecompGrid(n_pv=3), P.DecompGrid(n_pf=2, n_pv=2)):
                a = P.run_2way(P.Problem(2, n_f, n_v, spec, precision), grid)
                b = P.run_2way(P.Problem(2, n_f, n_v, P.gen_uniform(17, n_f, n_v), precision),
                               grid)
                assert a.checksum == b.checksum, (precision, grid)
            r3 = P.run_3way(P.Problem(3, n_f, n_v, spec, precision), P.DecompGrid(n_pv=2))
            w3 = P.run_3way(P.Problem(3, n_f, n_v, P.gen_uniform(17, n_f, n_v), precision),
                            P.DecompGrid(n_pv=2))
            assert r3.checksum == w3.checksum
        finally:
            vectorfile.CHUNK_BYTES = old
    bad = tmp_path / "short.bin"
    bad.write_bytes(b"\0" * 100)
    with pytest.raises(P.DataError):
        P.run_2way(P.Problem(2, n_f, n_v, P.VectorFileSpec(str(bad), n_f, n_v)), P.DecompGrid())
    nan = np.ones((n_f, n_v))
    nan[5, 7] = np.nan
    nan.ravel(order="F").tofile(tmp_path / "nan.bin")
    with pytest.raises(P.DataError):
        P.run_2way(P.Problem(2, n_f, n_v, P.VectorFileSpec(str(tmp_path / "nan.bin"), n_f, n_v)),
                   P.DecompGrid())


def test_data_errors_on_device():
    P = _api()
    m = np.ones((4, 4))
    m[1, 2] = -1.0
    with pytest.raises(P.DataError):
        P.run_2way(P.Problem(2, 4, 4, ArraySource(m)), P.DecompGrid())
    m[1, 2] = np.nan
    with pytest.raises(P.DataError):
        P.run_2way(P.Problem(2, 4, 4, ArraySource(m)), P.DecompGrid())


def _pinned_matrix(V):
    """V (n_f, n_v) copied into page-locked host memory, returned as a Fortran
    view of it (what a caller staging its data in pinned buffers hands over)."""
    import torch

    t = torch.empty((V.shape[1], V.shape[0]), dtype=torch.from_numpy(V[:1, :1].copy()).dtype,
                    pin_memory=True)
    t.numpy()[:] = V.T
    return t, t.numpy().T


@pytest.mark.parametrize("precision,n_f,n_v", [("double", 777, 1000), ("single", 300, 2500),
                                               ("double", 33, 5), ("double", 1, 300)])
def test_streamed_pinned_input_equals_plain_run(precision, n_f, n_v):
    """A pinned host source takes psim_czek2_streamed (chunked upload overlapped
    with the kernel, sums folded in the mainloop): values, checksum and
    degenerate flags equal the oracle's, with device or zero-copy host output."""
    from oracle import propsim_np as O

    P = _api()
    dt = np.float64 if precision == "double" else np.float32
    V = O.uniform(3, n_f, n_v, dt)
    V[:, 7 % n_v] = 0  # a zero vector: degenerate pairs with itself only if two zero vectors
    V[:, 11 % n_v] = 0
    keep, M = _pinned_matrix(V)
    prob = P.Problem(2, n_f, n_v, ArraySource(M), precision)
    vals, zero = O.values_2way(V)
    for host_values in (False, True):
        res = P.run_2way(prob, P.DecompGrid(), host_values=host_values)
        got = res.records.values
        assert (got.view(np.uint64 if dt == np.float64 else np.uint32)
                == vals.view(np.uint64 if dt == np.float64 else np.uint32)).all()
        assert res.checksum.hex == O.checksum_hex(np.arange(len(vals)), vals)
        assert res.degenerate_count == int(zero.sum())
    del keep


def test_streamed_pinned_input_rejects_bad_data():
    P = _api()
    V = np.asfortranarray(np.random.default_rng(0).random((64, 300)))
    V[5, 200] = np.nan
    keep, M = _pinned_matrix(V)
    with pytest.raises(P.DataError):
        P.run_2way(P.Problem(2, 64, 300, ArraySource(M), "double"), P.DecompGrid())
    M[5, 200] = -1.0
    with pytest.raises(P.DataError):
        P.run_2way(P.Problem(2, 64, 300, ArraySource(M), "double"), P.DecompGrid())
    del keep


def test_streamed_capi_validation():
    import ctypes as C

    import torch

    from paper_1705_08210_b200 import _native as N

    lib = N.lib()
    dev = torch.empty((10, 32), dtype=torch.float64, device="cuda")
    acc = torch.zeros(3, dtype=torch.int64, device="cuda")
    ready = torch.zeros(4, dtype=torch.int32, device="cuda")
    pageable = np.zeros((10, 32))
    sums = torch.empty(10, dtype=torch.float64, device="cuda")
    t = N.Block2(W=dev.data_ptr(), ldw=32, V=dev.data_ptr(), ldv=32, n_f=20, m=10, n=10,
                 diagonal=1, n_v=10, acc=acc.data_ptr(), s_row=sums.data_ptr())
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    # pageable host memory is staged through the pinned ring (accepted);
    # a device pointer passed as the host block is rejected
    rc = lib.psim_czek2_streamed(N.F64, C.byref(t), pageable.ctypes.data, 20, 4,
                                 ready.data_ptr(), s1.cuda_stream, s2.cuda_stream)
    assert rc == 0, lib.psim_last_error()
    torch.cuda.synchronize()
    rc = lib.psim_czek2_streamed(N.F64, C.byref(t), dev.data_ptr(), 32, 4,
                                 ready.data_ptr(), s1.cuda_stream, s2.cuda_stream)
    assert rc == 1 and b"device memory" in lib.psim_last_error()
    t.diagonal = 0
    rc = lib.psim_czek2_streamed(N.F64, C.byref(t), pageable.ctypes.data, 20, 4,
                                 ready.data_ptr(), s1.cuda_stream, s2.cuda_stream)
    assert rc == 1


@pytest.mark.parametrize("loader", ["tma", "cp.async"])
@pytest.mark.parametrize("precision", ["double", "single"])
def test_flattened_offdiagonal_tasks_bitwise_vs_oracle(precision, loader, monkeypatch):
    """Blocks wider than a column tile: a rank's off-diagonal circulant tasks
    run as one kCzek2Flat task (columns end to end, tiles straddling two
    blocks; czek2.cu flatten_tasks). n_vp = 500 / 375 / 300 / 250 covers full
    tasks, split half-blocks wider (187) and narrower (125) than BN, which stay
    separate. Identical bits and checksum to the sequential oracle, with and
    without kept values. With TMA staging (default) only blocks that lie back
    to back in memory are flattened (one V operand); PSIM_NO_TMA=1 runs the
    cp.async loader, whose two-pointer tiles flatten any consecutive blocks."""
    from oracle import propsim_np as O

    if loader == "cp.async":
        monkeypatch.setenv("PSIM_NO_TMA", "1")

    P = _api()
    n_f, n_v = 257, 1500
    dt = np.float64 if precision == "double" else np.float32
    want, _ = O.values_2way(O.uniform(5, n_f, n_v, dt))
    cks = O.checksum_hex(np.arange(len(want)), want)
    for n_pv in (3, 4, 5, 6):
        prob = P.Problem(2, n_f, n_v, P.gen_uniform(5, n_f, n_v), precision)
        res = P.run_2way(prob, P.DecompGrid(n_pv=n_pv))
        assert (res.records.values.view(np.uint8) == want.view(np.uint8)).all(), n_pv
        assert res.checksum.hex == cks, n_pv
        res = P.run_2way(prob, P.DecompGrid(n_pv=n_pv), keep_values=False)
        assert res.checksum.hex == cks, n_pv
    res = P.run_2way(prob, P.DecompGrid(n_pv=5), host_values=True)
    assert (res.records.values.view(np.uint8) == want.view(np.uint8)).all()
    assert res.checksum.hex == cks


CONFIG_CASES = json.loads((Path(__file__).resolve().parent / "golden" / "configs.json")
                          .read_text())["cases"]


@pytest.mark.parametrize("idx", range(len(CONFIG_CASES)),
                         ids=[f"{c['config']}-{c['kind']}-pf{c['grid']['n_pf']}"
                              f"pv{c['grid']['n_pv']}" for c in CONFIG_CASES])
def test_config_shaped_golden(idx):
    """The benchmarked configurations' shapes (n_f, dtype, bits and
    decomposition of cfg2..cfg5, n_v reduced) against the reference's own
    run_2way / run_3way (tests/golden/make_golden_configs.py): checksum,
    record count, degenerate count and a spread of individual value bits,
    all bitwise -- including the ascending-p_f fold of cfg5's field split
    on general FP data."""
    c = CONFIG_CASES[idx]
    P = _api()
    src = (P.gen_uniform(c["seed"], c["n_f"], c["n_v"]) if c["kind"] == "uniform"
           else P.gen_random_exact(c["seed"], c["n_f"], c["n_v"], c["bits"]))
    prob = P.Problem(c["arity"], c["n_f"], c["n_v"], src, c["precision"])
    grid = P.DecompGrid(**c["grid"])
    res = P.run_2way(prob, grid) if c["arity"] == 2 else P.run_3way(prob, grid)
    assert res.checksum.hex == c["checksum"]
    assert len(res.records) == c["records"]
    assert res.degenerate_count == c["degenerate"]
    from oracle import propsim_np as O

    vals = res.records.values
    for pos, bits in c["sample"].items():
        assert format(int(O.value_bits(vals[int(pos):int(pos) + 1])[0]), "x") == bits, pos


def test_full_cfg2_sampled_parity():
    """cfg2 at full size (2-way FP64, 20000 x 40000, bits 20) through the
    benchmark's own harness: >= 10^4 pairs (a grid of sampled rows x sampled
    columns of the canonical triangle, plus its first / last rows and
    columns) recomputed from their columns alone by the oracle, bitwise
    (SURVEY 8d), and the checksum equals the checksum every N of the round-1
    scaling runs produced."""
    import bench
    from paper_1705_08210_b200 import engine2

    P = _api()
    prob = P.Problem(2, 20000, 40000, P.gen_random_exact(2026, 20000, 40000, 20))
    r = engine2.Resident2(prob, P.DecompGrid())
    r.setup()
    r.step()
    par = bench.sampled_parity(r, prob, 20, 1, None)
    assert par["sampled"] >= 10000, par
    assert par["mismatches"] == 0, par
    assert r.checksum_hex() == "73cac6d75612b5f4372130e4fd66716c"
    r.teardown()


def test_pageable_source_streams_through_pinned_ring():
    """A plain numpy source (pageable memory, the reference's ArraySource) on
    the single-slab path: chunks are staged through the pinned ring while the
    streamed kernel runs (12 chunks through 4 slots); values and checksum
    equal the run on the device-generated block, and invalid data still
    raises DataError."""
    from oracle import propsim_np as O

    P = _api()
    n_f, n_v = 777, 3000
    m = O.uniform(6, n_f, n_v, np.float64)
    want = P.run_2way(P.Problem(2, n_f, n_v, P.gen_uniform(6, n_f, n_v)), P.DecompGrid())
    got = P.run_2way(P.Problem(2, n_f, n_v, ArraySource(np.asfortranarray(m))), P.DecompGrid())
    assert got.checksum == want.checksum
    assert (got.records.values.view(np.uint64) == want.records.values.view(np.uint64)).all()
    bad = np.asfortranarray(m.copy())
    bad[10, 2999] = -1.0
    with pytest.raises(P.DataError):
        P.run_2way(P.Problem(2, n_f, n_v, ArraySource(bad)), P.DecompGrid())
