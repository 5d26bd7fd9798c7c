"""End-to-end breakdown of the NCCL 2-way path from pinned host slabs (experiment).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 tools/exp_e2e_nccl.py

Per rank and repetition: wall time of run_2way(transport="nccl",
host_values=True), the device-timed pipeline (res.elapsed, max over ranks)
and the streamed kernel's chunk-wait statistics (psim_stream_stats).
"""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1705_08210_b200 as P  # noqa: E402
from paper_1705_08210_b200 import _native as N  # noqa: E402
from paper_1705_08210_b200 import device as D  # noqa: E402
from paper_1705_08210_b200.domain import coords_of_rank  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    n_f, n_v = 20000, 40000
    grid = P.DecompGrid(n_pv=world)
    gen = P.Problem(2, n_f, n_v, P.gen_random_exact(2026, n_f, n_v, 20), "double")
    coords = coords_of_rank(rank, grid)
    blk = D.load_block(gen, grid, coords, torch.device("cuda"))
    host = torch.empty((blk.n_vp, blk.n_fp), dtype=blk.data.dtype, pin_memory=True)
    host.copy_(blk.data[:, :blk.n_fp])
    del blk
    torch.cuda.synchronize()

    class Slab:
        def local_block(self, problem, grid_, coords_):
            return host.numpy().T

    prob = P.Problem(2, n_f, n_v, Slab(), "double")
    os.environ["PSIM_TRACE"] = "1"
    from paper_1705_08210_b200 import dist as PD
    for rep in range(int(os.environ.get("REPS", "6"))):
        dist.barrier()
        torch.cuda.synchronize()
        st = (C.c_uint64 * 4)()
        N.call("psim_stream_stats", st, 1)
        t0 = time.perf_counter()
        res = P.run_2way(prob, grid, transport="nccl", host_values=True)
        wall = time.perf_counter() - t0
        lead = (PD.LAST_TRACE[0][1] - t0) * 1e3 if PD.LAST_TRACE else None
        N.call("psim_stream_stats", st, 1)
        print(json.dumps({"rank": rank, "rep": rep, "wall_s": round(wall, 4), "lead_ms": lead,
                          "device_s": round(res.elapsed, 4),
                          "chunk_wait_sm_ms": st[0] / 1e6, "max_wait_ms": st[3] / 1e6,
                          "trace_ms": {b[0]: round((b[1] - a[1]) * 1e3, 2) for a, b in
                                       zip(PD.LAST_TRACE, PD.LAST_TRACE[1:])},
                          "tail_ms": round((time.perf_counter() - PD.LAST_TRACE[-1][1]) * 1e3, 2)
                          if PD.LAST_TRACE else None,
                          "checksum": res.checksum.hex}), flush=True)
        del res
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
