"""The same cfg2 problem on ONE GPU under the circulant plans of n_pv = 1, 2, 4, 8
(transport="local": every rank's tasks run in turn on this device), to separate
the cost of the multi-task grids from communication (experiment).

    python tools/exp_local_grids.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1705_08210_b200 as P  # noqa: E402


def main():
    n_f, n_v = 20000, 40000
    prob = P.Problem(2, n_f, n_v, P.gen_random_exact(2026, n_f, n_v, 20), "double")
    cmp = n_f * n_v * (n_v - 1) // 2
    for n_pv in (1, 2, 4, 8):
        for rep in range(2):
            res = P.run_2way(prob, P.DecompGrid(n_pv=n_pv), keep_values=False)
            print(json.dumps({"n_pv": n_pv, "rep": rep, "elapsed_s": round(res.elapsed, 4),
                              "cmp_per_s": cmp / res.elapsed, "checksum": res.checksum.hex}),
                  flush=True)


if __name__ == "__main__":
    main()
