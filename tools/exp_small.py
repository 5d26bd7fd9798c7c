"""Small-problem latency of the public API (experiment, not product).

    python tools/exp_small.py [n_f n_v]

cfg1 (2-way FP64, 1000 x 500) is the reference's own CPU-runnable case: the
GPU path is dominated by per-call overhead there, not by the kernel. This
times run_2way end to end (host wall clock, records materialised on the
host) for a synthetic source and for a plain numpy (pageable) source, first
call and steady state, next to the device pipeline time it reports
(RunResult.elapsed) and the kernel's own time, so each layer's share shows.
"""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_08210_b200 as P  # noqa: E402
from oracle import propsim_np as O  # noqa: E402


class ArraySource:  # the reference's test source (pkg/tests/conftest.py:17-26)
    def __init__(self, m):
        self.m = np.asfortranarray(m)

    def local_block(self, problem, grid, coords):
        return self.m


def main():
    n_f = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    n_v = int(sys.argv[2]) if len(sys.argv) > 2 else 500
    torch.cuda.set_device(0)
    V = O.random_exact(2026, n_f, n_v, 20)
    want = O.run_2way(V)[2] if n_v <= 2000 else None
    for name, src in (("synthetic", P.gen_random_exact(2026, n_f, n_v, 20)),
                      ("numpy", ArraySource(V))):
        prob = P.Problem(2, n_f, n_v, src, "double")
        walls, dev = [], []
        first = None
        for rep in range(30):
            t0 = time.perf_counter()
            res = P.run_2way(prob, P.DecompGrid())
            vals = res.records.values
            t1 = time.perf_counter()
            assert len(vals) == n_v * (n_v - 1) // 2
            if want is not None:
                assert res.checksum.hex == want, (res.checksum.hex, want)
            if rep == 0:
                first = (t1 - t0, res.elapsed)
            else:
                walls.append(t1 - t0)
                dev.append(res.elapsed)
        cmp = n_f * n_v * (n_v - 1) // 2
        print(json.dumps({
            "source": name, "n_f": n_f, "n_v": n_v,
            "first_call_wall_ms": first[0] * 1e3, "first_call_device_ms": first[1] * 1e3,
            "steady_wall_ms": statistics.median(walls) * 1e3,
            "steady_device_ms": statistics.median(dev) * 1e3,
            "steady_cmp_per_s": cmp / statistics.median(walls),
            "checksum_ok": want is not None}), flush=True)


if __name__ == "__main__":
    main()
