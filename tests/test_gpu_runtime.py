"""The run-level runtime (psim_ctx / psim_run2 / psim_run3 / psim_checksum,
csrc/runtime.cu) driven through ctypes alone: torch only allocates device
memory, no torch.distributed anywhere. One rank on one GPU against the
reference's golden runs; and, on a box with >= 2 GPUs, two processes that
pass rank 0's NCCL id over a pipe and run circulant / tetrahedral / field
split grids whose checksums the reference computed
(tests/golden/configs.json)."""
import ctypes as C
import json
import math
import multiprocessing as mp
from pathlib import Path

import numpy as np
import pytest

from conftest import cuda_available, golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

CONF = json.loads((Path(__file__).resolve().parent / "golden" / "configs.json").read_text())


def _gold(arity, precision, n_f, n_v, bits, seed=2026):
    for c in golden()["cases"] + CONF["cases"]:
        if (c["arity"], c["precision"], c["n_f"], c["n_v"], c.get("bits"), c["seed"]) == \
                (arity, precision, n_f, n_v, bits, seed) and c["kind"] == "random-exact" \
                and c["grid"]["n_pf"] == 1 and "stage" not in c:
            return c
    raise KeyError


def _run(ctx, arity, dtype, n_f, n_v, grid, inp, seed=2026, bits=20, block=None, ld=0,
         stage=-1, keep=True):
    """One psim_run2 / psim_run3 call through ctypes; returns (out, vals, pieces)."""
    import torch

    from paper_1705_08210_b200 import _native as N

    prob = N.Problem(arity=arity, dtype=dtype, n_f=n_f, n_v=n_v, input=inp, bits=bits,
                     seed=seed, block=block, ld=ld)
    g = N.Grid(n_pf=grid[0], n_pv=grid[1], n_pr=grid[2], n_st=grid[3])
    plan = N.Plan()
    N.call("psim_run_plan", ctx, C.byref(prob), C.byref(g), stage, 0, C.byref(plan))
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
    tdt = torch.float64 if dtype == N.F64 else torch.float32
    vals = torch.empty(max(1, plan.n_vals), dtype=tdt, device="cuda") if keep else None
    pieces = (N.Piece * max(1, plan.n_pieces))()
    world = grid[0] * grid[1] * grid[2]
    rt = (N.Traffic * world)()
    sums = torch.empty(n_v, dtype=tdt, device="cuda")
    out = N.Out(vals=None if vals is None else vals.data_ptr(), pieces=pieces,
                sums=sums.data_ptr(), rank_traffic=rt)
    args = (ctx, C.byref(prob), C.byref(g)) + ((stage,) if arity == 3 else ())
    st = torch.cuda.current_stream().cuda_stream
    N.call("psim_run2" if arity == 2 else "psim_run3", *args, 0, ws.data_ptr(), ws.numel(),
           C.byref(out), st)
    return out, vals, pieces, sums, rt


def _ctx(device=0, rank=0, world=1, nid=None):
    from paper_1705_08210_b200 import _native as N

    h = C.c_void_p()
    N.call("psim_ctx_create", device, rank, world, nid, C.byref(h))
    return h


def _hex(out):
    return format((out.checksum[1] << 64) | out.checksum[0], "032x")


def test_ctypes_only_run2_cfg1_golden():
    """cfg1 (2-way FP64, 1000 x 500, bits 20): the reference's checksum, record
    count and degenerate count from one psim_run2 call; the values re-checksum
    to the same words through psim_checksum; column sums equal psim_column_sums."""
    import torch

    from paper_1705_08210_b200 import _native as N

    c = _gold(2, "double", 1000, 500, 20)
    ctx = _ctx()
    try:
        out, vals, pieces, sums, rt = _run(ctx, 2, N.F64, 1000, 500, (1, 1, 1, 1),
                                           N.INPUT_RANDOM_EXACT)
        assert _hex(out) == c["checksum"] == "ea23ebab734aeaaefdc87babae741b72"
        assert out.count == c["records"] == math.comb(500, 2) == out.local_count == out.n_vals
        assert out.degenerate == c["degenerate"]
        assert out.n_pieces == 1 and pieces[0].kind == 2 and list(pieces[0].v)[:5] == \
            [0, 0, 500, 500, 1]
        assert out.elapsed > 0 and out.kernel_grids >= 1 and out.kernel_seconds > 0
        assert sum(rt[0].messages) == 0  # one rank: no traffic
        acc = torch.zeros(3, dtype=torch.int64, device="cuda")
        N.call("psim_checksum", N.F64, vals.data_ptr(), None, 0, out.n_vals, acc.data_ptr(),
               torch.cuda.current_stream().cuda_stream)
        lo, hi, _ = [int(x) & ((1 << 64) - 1) for x in acc.cpu().tolist()]
        assert format((hi << 64) | lo, "032x") == c["checksum"]
        blk = torch.empty((500, 1024), dtype=torch.float64, device="cuda")
        N.call("psim_gen_random_exact", N.F64, 2026, 20, 500, 0, 0, 1000, 500, blk.data_ptr(),
               1024, torch.cuda.current_stream().cuda_stream)
        s2 = torch.empty(500, dtype=torch.float64, device="cuda")
        N.call("psim_column_sums", N.F64, blk.data_ptr(), 1000, 500, 1024, s2.data_ptr(),
               torch.cuda.current_stream().cuda_stream)
        assert torch.equal(sums, s2)
        # the same block as caller input: device (in place), pinned host (streamed
        # upload), pageable host (plain upload) -- one checksum
        out_d, *_ = _run(ctx, 2, N.F64, 1000, 500, (1, 1, 1, 1), N.INPUT_DEVICE,
                         block=blk.data_ptr(), ld=1024)
        host = blk.cpu().pin_memory()
        out_p, *_ = _run(ctx, 2, N.F64, 1000, 500, (1, 1, 1, 1), N.INPUT_HOST,
                         block=host.data_ptr(), ld=1024)
        pageable = blk.cpu().numpy().copy()
        out_h, *_ = _run(ctx, 2, N.F64, 1000, 500, (1, 1, 1, 1), N.INPUT_HOST,
                         block=pageable.ctypes.data, ld=1024)
        assert _hex(out_d) == _hex(out_p) == _hex(out_h) == c["checksum"]
        # invalid caller data: DataError (status 2) like VectorBlock (core.py:239-242)
        pageable[3, 7] = -1.0
        prob = N.Problem(arity=2, dtype=N.F64, n_f=1000, n_v=500, input=N.INPUT_HOST,
                         block=pageable.ctypes.data, ld=1024)
        g = N.Grid(1, 1, 1, 1)
        plan = N.Plan()
        N.call("psim_run_plan", ctx, C.byref(prob), C.byref(g), -1, 0, C.byref(plan))
        ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
        o = N.Out()
        assert N.lib().psim_run2(ctx, C.byref(prob), C.byref(g), 0, ws.data_ptr(), ws.numel(),
                                 C.byref(o), None) == 2
        assert b"nonnegative" in N.lib().psim_last_error()
    finally:
        N.lib().psim_ctx_destroy(ctx)


@pytest.mark.parametrize("precision,n_f,n_v,bits", [("double", 1000, 60, 20),
                                                    ("single", 1000, 60, 8),
                                                    ("double", 10000, 96, 20)])
def test_ctypes_only_run3_golden(precision, n_f, n_v, bits):
    from paper_1705_08210_b200 import _native as N

    c = _gold(3, precision, n_f, n_v, bits)
    ctx = _ctx()
    try:
        dt = N.F64 if precision == "double" else N.F32
        out, vals, pieces, _, _ = _run(ctx, 3, dt, n_f, n_v, (1, 1, 1, 1), N.INPUT_RANDOM_EXACT,
                                       bits=bits)
        assert _hex(out) == c["checksum"]
        assert out.count == c["records"] == math.comb(n_v, 3)
        # staged: the stages of n_st = 2 add up to the whole run
        parts = [_run(ctx, 3, dt, n_f, n_v, (1, 1, 1, 2), N.INPUT_RANDOM_EXACT, bits=bits,
                      stage=s)[0] for s in (0, 1)]
        tot = sum((p.checksum[1] << 64) | p.checksum[0] for p in parts) % (1 << 128)
        assert format(tot, "032x") == c["checksum"]
        assert sum(p.count for p in parts) == c["records"]
    finally:
        N.lib().psim_ctx_destroy(ctx)


def _worker(rank, world, conn, cases):
    """One rank: the NCCL id comes over a pipe (no torch.distributed)."""
    import torch

    from paper_1705_08210_b200 import _native as N

    torch.cuda.set_device(rank)
    if rank == 0:
        buf = C.create_string_buffer(128)
        N.call("psim_nccl_unique_id", buf)
        for c in conn:
            c.send(buf.raw)
        nid = buf.raw
    else:
        nid = conn.recv()
    ctx = _ctx(rank, rank, world, C.create_string_buffer(nid, 128))
    res = []
    try:
        for arity, prec, n_f, n_v, grid, kind, seed, bits in cases:
            dt = N.F64 if prec == "double" else N.F32
            inp = N.INPUT_UNIFORM if kind == "uniform" else N.INPUT_RANDOM_EXACT
            out, _, _, _, rt = _run(ctx, arity, dt, n_f, n_v, grid, inp, seed=seed, bits=bits)
            res.append((_hex(out), out.count, [sum(rt[r].nbytes) for r in range(world)]))
    finally:
        N.lib().psim_ctx_destroy(ctx)
    return res


def _proc(rank, world, conn, cases, q):
    try:
        q.put((rank, _worker(rank, world, conn, cases)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_two_processes_nccl_without_torch_distributed():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    picks = [c for c in CONF["cases"] if c["grid"]["n_pf"] * c["grid"]["n_pv"] == 2]
    cases = [(c["arity"], c["precision"], c["n_f"], c["n_v"],
              (c["grid"]["n_pf"], c["grid"]["n_pv"], c["grid"]["n_pr"], c["grid"]["n_st"]),
              c["kind"], c["seed"], c["bits"]) for c in picks]
    assert {c[0] for c in cases} == {2, 3} and any(c[4][0] == 2 for c in cases)
    ctxm = mp.get_context("spawn")
    a, b = ctxm.Pipe()
    q = ctxm.Queue()
    ps = [ctxm.Process(target=_proc, args=(0, 2, [a], cases, q)),
          ctxm.Process(target=_proc, args=(1, 2, b, cases, q))]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=900) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in (0, 1):
        assert not isinstance(got[r], str), got[r]
    for k, c in enumerate(picks):
        assert got[0][k][0] == got[1][k][0] == c["checksum"], c
        assert got[0][k][1] == c["records"]
        assert got[0][k][2] == got[1][k][2]  # every rank sees every rank's traffic
        assert sum(got[0][k][2]) > 0
