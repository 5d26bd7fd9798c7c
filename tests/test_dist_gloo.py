"""Multi-rank host logic on CPU (world_size 2, gloo): the ordered field-axis
reduce-scatter and the global checksum gather of dist.py. The device folds
are replaced by the same in-order elementwise add on CPU tensors."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1705_08210_b200 import dist as PD

        out = {}
        rng = np.random.default_rng(0)
        for m, n, diagonal in ((37, 37, True), (11, 23, False), (2, 2, True)):
            count = m * (m - 1) // 2 if diagonal else m * n
            parts = [rng.random(count).astype(np.float32) for _ in range(world)]
            mine = torch.from_numpy(parts[rank].copy())
            total, r0, r1 = PD.reduce_scatter_rows(
                mine, m, n, diagonal, rank, world, None, lambda d, s: d.add_(s))
            a = PD.packed_offset(r0, m, n, diagonal)
            b = PD.packed_offset(r1, m, n, diagonal)
            want = parts[0][a:b].copy()
            for p in parts[1:]:
                want = want + p[a:b]  # ascending p_f fold
            out[(m, n, diagonal)] = (bool((total.numpy() == want).all()), r0, r1)
        # int64 words carry u64 bits (as the device accumulator does); the two
        # low words sum past 2^64 so the carry into the high word is exercised
        lo = -((1 << 63) - rank) if rank else -(1 << 63)
        acc = torch.tensor([lo, rank, 2 + rank], dtype=torch.int64)
        lo, hi, deg, cnt = PD.gather_totals(acc, 10 + rank, world, "cpu")
        out["totals"] = (lo, hi, deg, cnt)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_field_reduce_scatter_and_totals_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    results = dict(q.get(timeout=10) for _ in range(world))
    for key in ((37, 37, True), (11, 23, False), (2, 2, True)):
        spans = []
        for r in range(world):
            ok, r0, r1 = results[r][key]
            assert ok, (key, r)
            spans.append((r0, r1))
        m = key[0]
        assert spans[0][0] == 0 and spans[-1][1] == m
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    # both ranks see the same global totals; lo words wrap with carry into hi
    t0, t1 = results[0]["totals"], results[1]["totals"]
    assert t0 == t1
    M64 = (1 << 64) - 1
    lo0 = (-(1 << 63)) & M64
    lo1 = (-((1 << 63) - 1)) & M64
    total = (lo0 + (0 << 64)) + (lo1 + (1 << 64))
    assert (t0[0], t0[1]) == (total & M64, (total >> 64) & M64)
    assert t0[2] == 2 + 3 and t0[3] == 21


def _writer_worker(rank, world, port, directory, q):
    """Each process holds an arbitrary half of the records (not the owned
    set); write_run_output routes them to their owners and every process
    writes its own metrics_<rank>.bin (output.py _write_distributed)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import dataclasses

        from conftest import golden
        from paper_1705_08210_b200 import output as OUT
        from test_output import _Records, oracle_result

        case = next(c for c in golden()["outputs"]
                    if c["arity"] == 3 and c["stage"] == 1 and c["mode"] == "byte")
        full = oracle_result(case)
        idx, vals = full.records.canonical_indices, full.records.values
        mine = (idx // 7) % world == rank
        res = dataclasses.replace(full, transport="nccl",
                                  records=_Records(idx[mine], vals[mine]))
        OUT.write_run_output(res, OUT.MetricOutputSpec(directory, "byte"),
                             source={"kind": case["kind"]})
        q.put((rank, case))
    finally:
        dist.destroy_process_group()


def test_distributed_output_writer_gloo(tmp_path):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_writer_worker, args=(r, world, port, str(tmp_path), q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    case = dict(q.get(timeout=10) for _ in range(world))[0]
    from test_output import check_directory

    check_directory(tmp_path, case)


def _exchange_worker(rank, world, port, q):
    """2-way circulant steps (every Exchange of plan_2way, posted all at once as
    the fused NCCL runner does, then one at a time) and the 3-way all-gather,
    through the runners' own op builders, on CPU tensors."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1705_08210_b200 import DecompGrid
        from paper_1705_08210_b200 import dist as PD
        from paper_1705_08210_b200.domain import coords_of_rank, rank_of_coords
        from paper_1705_08210_b200.plan import Exchange, plan_2way

        grid = DecompGrid(n_pv=world)
        c = coords_of_rank(rank, grid)
        me = c.p_v
        peer = lambda slab: rank_of_coords(type(c)(c.p_f, slab % world, c.p_r), grid)  # noqa: E731
        own = torch.full((3, 4), float(me))
        s_own = torch.full((3,), 10.0 + me)
        exs = [e for e in plan_2way(grid, c, 12, "split") if isinstance(e, Exchange)]
        ok = []
        for fused in (True, False):
            bufs = [(torch.empty(3, 4), torch.empty(3)) for _ in exs]
            works = []
            for e, (b, s) in zip(exs, bufs):
                w = dist.batch_isend_irecv(PD.exchange_ops(own, s_own, b, s, peer(e.send_to),
                                                           peer(e.recv_from)))
                if fused:
                    works.extend(w)
                else:
                    for x in w:
                        x.wait()
            for x in works:
                x.wait()
            for e, (b, s) in zip(exs, bufs):
                src = (me + e.step) % world
                ok.append(bool((b == src).all()) and bool((s == 10.0 + src).all()))
        blocks = {sl: (own if sl == me else torch.empty(3, 4)) for sl in range(world)}
        sums = {sl: (s_own if sl == me else torch.empty(3)) for sl in range(world)}
        for x in dist.batch_isend_irecv(PD.allgather_ops(me, world, blocks, sums, peer)):
            x.wait()
        ok.append(all(bool((blocks[sl] == sl).all()) and bool((sums[sl] == 10.0 + sl).all())
                      for sl in range(world)))
        q.put((rank, len(exs), ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [8])
def test_circulant_exchanges_and_allgather_gloo(world):
    """n_pv = 8 (the size no GPU run here covers): every block arrives from the
    slab the plan names, in fused and stepwise posting, and the 3-way
    all-gather delivers every slab to every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    results = dict((r, (n, ok)) for r, n, ok in (q.get(timeout=10) for _ in range(world)))
    for r in range(world):
        n, ok = results[r]
        assert n == world // 2  # steps 1 .. n_pv/2 (the last one split, schedule.py:128-136)
        assert all(ok), (r, ok)
