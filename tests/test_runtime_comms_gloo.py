"""The run-level runtime's NCCL schedule, replayed over gloo on CPU.

psim_run_comms returns, for each rank, the exact sequence of NCCL groups of
send / recv that psim_run2 / psim_run3 would issue (planning-only context,
no GPU). Here every rank of a grid -- up to world 8, the size the GPU service
never hands out -- replays its groups in order with torch.distributed
batch_isend_irecv over gloo, byte for byte: every receive must be matched by
the right peer's send of the same size, in the same order (as NCCL requires),
and carry what the plan says -- the block / sums of the slab the circulant
(schedule.py:116-142) or tetrahedral (schedule.py:184-214) plan expects, the
task / table / box chunk of the field reduce-scatter (engine.py:197-216)."""
import ctypes as C
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1705_08210_b200 as P
from paper_1705_08210_b200 import _native as N
from paper_1705_08210_b200.domain import coords_of_rank


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _msgs(arity, n_f, n_v, grid, rank, stage=-1, dtype=N.F64):
    ctx = C.c_void_p()
    world = grid.n_pf * grid.n_pv * grid.n_pr
    N.call("psim_ctx_create", -1, rank, world, None, C.byref(ctx))
    try:
        prob = N.Problem(arity=arity, dtype=dtype, n_f=n_f, n_v=n_v,
                         input=N.INPUT_RANDOM_EXACT, bits=8, seed=1)
        g = N.Grid(n_pf=grid.n_pf, n_pv=grid.n_pv, n_pr=grid.n_pr, n_st=grid.n_st)
        n = C.c_int64()
        N.call("psim_run_comms", ctx, C.byref(prob), C.byref(g), stage, 0, None, 0, C.byref(n))
        arr = (N.Msg * max(1, n.value))()
        N.call("psim_run_comms", ctx, C.byref(prob), C.byref(g), stage, 0, arr, n.value,
               C.byref(n))
        return [(m.group, m.op, m.peer, m.what, m.bytes, m.slot) for m in arr[:n.value]]
    finally:
        N.lib().psim_ctx_destroy(ctx)


def _pattern(src, what, slot, nbytes):
    x = torch.arange(nbytes, dtype=torch.int64)
    return ((x * 31 + src * 7 + what * 13 + slot * 17) % 251).to(torch.uint8)


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        arity, n_f, n_v, g, stage, dtype = case
        grid = P.DecompGrid(**g)
        msgs = _msgs(arity, n_f, n_v, grid, rank, stage, dtype)
        me = coords_of_rank(rank, grid)
        errors, checked = [], 0
        for gid in sorted({m[0] for m in msgs}):
            ops, recvs = [], []
            for _, op, peer, what, nbytes, slot in (m for m in msgs if m[0] == gid):
                if op == 0:
                    tag_slot = me.p_v if what in (N.MSG_BLOCK, N.MSG_SUMS) else slot
                    ops.append(dist.P2POp(dist.isend, _pattern(rank, what, tag_slot, nbytes),
                                          peer))
                else:
                    buf = torch.zeros(nbytes, dtype=torch.uint8)
                    ops.append(dist.P2POp(dist.irecv, buf, peer))
                    recvs.append((buf, peer, what, slot, nbytes))
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            for buf, peer, what, slot, nbytes in recvs:
                if what in (N.MSG_BLOCK, N.MSG_SUMS):  # the block of the slab the plan names
                    if coords_of_rank(peer, grid).p_v != slot:
                        errors.append(("wrong slab", gid, peer, slot))
                if not torch.equal(buf, _pattern(peer, what, slot, nbytes)):
                    errors.append(("payload", gid, peer, what, slot, nbytes))
                checked += 1
        q.put((rank, errors, checked, len(msgs)))
    finally:
        dist.destroy_process_group()


CASES = [
    # 2-way circulant (cfg2 / cfg3 at 8 GPUs), with replicas, with a field split
    (2, 8, 8 * 24, dict(n_pv=8), -1, N.F64),
    (2, 8, 5 * 12, dict(n_pv=5), -1, N.F32),
    (2, 8, 4 * 12, dict(n_pv=4, n_pr=2), -1, N.F64),
    (2, 16, 4 * 12, dict(n_pv=4, n_pf=2), -1, N.F64),
    # cfg5: the field split over 8 ranks (ordered reduce-scatter of every task)
    (2, 64, 40, dict(n_pf=8), -1, N.F64),
    # 3-way tetrahedral (cfg4 at 8 GPUs), staged, with replicas / a field split
    (3, 8, 8 * 6, dict(n_pv=8), -1, N.F64),
    (3, 8, 4 * 6, dict(n_pv=4, n_st=2), 1, N.F32),
    (3, 8, 3 * 6, dict(n_pv=3, n_pr=2), -1, N.F64),
    (3, 16, 4 * 6, dict(n_pv=4, n_pf=2), -1, N.F64),
    (3, 32, 12, dict(n_pf=8), -1, N.F64),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}way-" + "-".join(
    f"{k}{v}" for k, v in c[3].items()))
def test_runtime_comm_schedule_replays_over_gloo(case):
    g = P.DecompGrid(**case[3])
    world = g.n_pf * g.n_pv * g.n_pr
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [q.get(timeout=10) for _ in range(world)]
    for rank, errors, checked, n in res:
        assert not errors, (rank, errors[:5])
    assert sum(r[2] for r in res) > 0
