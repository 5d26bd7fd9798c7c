"""Multi-rank host logic on CPU (gloo): the collective output writer
(write_run_output under transport "nccl", io.py:310-346), whose all-to-all
routing of records to their owning ranks runs on torch.distributed. The
run's own NCCL schedule (psim_run2 / psim_run3) is replayed over gloo in
tests/test_runtime_comms_gloo.py."""
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
