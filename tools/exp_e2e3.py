"""Where the run_3way API spends its wall time beyond the kernels (experiment).

    python tools/exp_e2e3.py [n_v] [n_f]
"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1705_08210_b200 as P  # noqa: E402
from paper_1705_08210_b200 import device as D  # noqa: E402
from paper_1705_08210_b200.domain import RankCoords  # noqa: E402
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import SlabSource  # noqa: E402


def main():
    n_v = int(sys.argv[1]) if len(sys.argv) > 1 else 1200
    n_f = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
    grid = P.DecompGrid()
    prob = P.Problem(3, n_f, n_v, P.gen_random_exact(2026, n_f, n_v, 20), "double")
    blk = D.load_block(prob, grid, RankCoords(0, 0, 0), torch.device("cuda"))
    host = torch.empty((blk.n_vp, blk.n_fp), dtype=blk.data.dtype, pin_memory=True)
    host.copy_(blk.data[:, :blk.n_fp])
    del blk
    e2e = P.Problem(3, n_f, n_v, SlabSource(host.numpy().T, (0, 0, 0)), "double")
    for keep in (False, True):
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = P.run_3way(e2e, grid, keep_values=keep)
            t1 = time.perf_counter()
            print(f"keep={keep} rep={rep} wall {t1 - t0:.4f} s elapsed {r.elapsed:.4f} s "
                  f"{r.checksum.hex}", flush=True)
            del r
    pr = cProfile.Profile()
    pr.enable()
    P.run_3way(e2e, grid, keep_values=False)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
