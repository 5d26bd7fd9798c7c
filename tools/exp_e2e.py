"""End-to-end (host-resident input) breakdown for the cfg2 2-way run (experiment).

    python tools/exp_e2e.py [n_f n_v]

Wall time of run_2way from a pinned host slab under each input / output
path, and the device time of the same run's CUDA work, to locate what the
e2e number pays beyond the device-resident kernel.
"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import ctypes as C  # noqa: E402

import torch  # noqa: E402

import paper_1705_08210_b200 as P  # noqa: E402
from paper_1705_08210_b200 import _native as N  # noqa: E402
from paper_1705_08210_b200 import device as D  # noqa: E402
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
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from bench import ClockSampler

    reps = int(os.environ.get("REPS", "4"))
    modes = os.environ.get("MODES", "1,0").split(",")
    os.environ["PSIM_TRACE"] = "1"
    from paper_1705_08210_b200 import engine2

    for streamed in modes:
        for host_values in ((True, False) if os.environ.get("HV") is None
                            else (os.environ["HV"] == "1",)):
            os.environ["PSIM_STREAMED"] = streamed
            P.run_2way(prob, P.DecompGrid(), host_values=host_values)  # warm-up
            for _ in range(reps):
                torch.cuda.synchronize()
                m0 = torch.cuda.memory_stats()
                if os.environ.get("NOGC") == "1":
                    import gc

                    gc.collect()
                    gc.disable()
                with (ClockSampler(0, 0.02) if os.environ.get("NOCLK") != "1"
                      else ClockSampler(0, 3600.0)) as clk:
                    t0 = time.perf_counter()
                    res = P.run_2way(prob, P.DecompGrid(), host_values=host_values)
                    el_dev = time.perf_counter() - t0
                    _ = res.records.values
                    el = time.perf_counter() - t0
                mhz = sorted(m for m, _ in clk.samples) or [0]
                st = (C.c_uint64 * 4)()
                N.call("psim_stream_stats", st, 1)
                print(json.dumps({"streamed": streamed, "host_values": host_values,
                                  "wall_s": round(el, 4), "device_s": round(res.elapsed, 4),
                                  "cmp_per_s": cmp / el, "chunk_wait_sm_ms": st[0] / 1e6,
                                  "sum_wait_sm_ms": st[1] / 1e6, "sum_waits": st[2],
                                  "max_wait_ms": st[3] / 1e6, "call_s": round(el_dev, 4),
                                  "mhz_min": mhz[0], "mhz_med": mhz[len(mhz) // 2],
                                  "reasons": sorted({r for _, r in clk.samples}),
                                  "dev_segments_new": torch.cuda.memory_stats().get(
                                      "segment.all.allocated", 0) - m0.get("segment.all.allocated", 0),
                                  "trace_ms": {b[0]: round(a[1].elapsed_time(b[1]), 3) for a, b in
                                               zip(engine2.LAST_TRACE, engine2.LAST_TRACE[1:])},
                                  "host_trace_ms": {b[0]: round((b[2] - a[2]) * 1e3, 3) for a, b in
                                                    zip(engine2.LAST_TRACE,
                                                        engine2.LAST_TRACE[1:])},
                                  "alloc_retries": torch.cuda.memory_stats().get(
                                      "num_alloc_retries", 0) - m0.get("num_alloc_retries", 0),
                                  "host_segments": torch.cuda.host_memory_stats().get(
                                      "segment.allocated", torch.cuda.host_memory_stats().get(
                                          "num_host_alloc", -1))}), flush=True)
                del res
    # pinned allocation reuse
    for _ in range(3):
        t0 = time.perf_counter()
        b = torch.empty(n_v * (n_v - 1) // 2, dtype=torch.float64, pin_memory=True)
        el = time.perf_counter() - t0
        print(json.dumps({"pinned_alloc_s": el}), flush=True)
        del b
    # H2D alone
    dev = torch.empty((n_v, n_f), dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(host, non_blocking=True)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        print(json.dumps({"h2d_s": el, "GB_per_s": host.numel() * 8 / el / 1e9}), flush=True)


if __name__ == "__main__":
    main()
