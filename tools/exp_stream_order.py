"""Streamed 2-way kernel: its own speed vs the upload overlap (experiment).

    python tools/exp_stream_order.py [n_f n_v]

run_2way from a pinned host slab (the e2e path) with the upload cut into the
default 64 chunks, into 1 chunk (the kernel waits for the whole block, then
runs without waits: its intrinsic speed in the streamed tile order), and into
256 chunks; each reported as device seconds per call (RunResult.elapsed) with
the streamed-wait statistics. Compare with bench.py's device-resident value.
"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1705_08210_b200 as P  # noqa: E402
from paper_1705_08210_b200 import _native as N  # noqa: E402
from paper_1705_08210_b200 import device as D  # noqa: E402
from paper_1705_08210_b200 import engine2  # noqa: E402
from paper_1705_08210_b200.domain import RankCoords  # noqa: E402


class Slab:
    def __init__(self, m):
        self.m = m

    def local_block(self, problem, grid, coords):
        return self.m


def main():
    n_f = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    n_v = int(sys.argv[2]) if len(sys.argv) > 2 else 40000
    gen = P.Problem(2, n_f, n_v, P.gen_random_exact(2026, n_f, n_v, 20), "double")
    blk = D.load_block(gen, P.DecompGrid(), RankCoords(0, 0, 0), torch.device("cuda"))
    host = torch.empty((n_v, n_f), dtype=torch.float64, pin_memory=True)
    host.copy_(blk.data[:, :n_f])
    del blk
    torch.cuda.synchronize()
    prob = P.Problem(2, n_f, n_v, Slab(host.numpy().T), "double")
    cmp = n_f * n_v * (n_v - 1) // 2
    default = engine2.stream_chunk
    for name, chunk in (("64 chunks (product)", default), ("1 chunk", lambda n: n),
                        ("256 chunks", lambda n: max(64, -(-n // 256)))):
        engine2.stream_chunk = chunk
        P.run_2way(prob, P.DecompGrid(), host_values=True)  # warm-up
        for rep in range(3):
            N.call("psim_stream_stats", (C.c_uint64 * 4)(), 1)
            res = P.run_2way(prob, P.DecompGrid(), host_values=True)
            st = (C.c_uint64 * 4)()
            N.call("psim_stream_stats", st, 1)
            print(json.dumps({"upload": name, "rep": rep, "device_s": round(res.elapsed, 4),
                              "cmp_per_s": cmp / res.elapsed, "checksum": res.checksum.hex,
                              "chunk_wait_sm_ms": st[0] / 1e6, "max_wait_ms": st[3] / 1e6}),
                  flush=True)
    engine2.stream_chunk = default


if __name__ == "__main__":
    main()
