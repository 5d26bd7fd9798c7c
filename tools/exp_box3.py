"""3-way box-kernel rate per padded tile (experiment, not product).

    python tools/exp_box3.py [n_f]

Times psim_czek3_box (and psim_czek3_box_numerators: the same tiles with
the raw n_ijk stored instead of the Eq. 1 epilogue) on boxes of one resident 6144-vector block and prints,
per box, useful and padded-tile cmp/clk/SM (clock 1965 MHz assumed; the bench
samples clocks), so the kernel's own overhead can be separated from tile
padding: a volume box (i < j < k ranges disjoint: every tile full) vs
diagonal pivot ranges like the cfg4 chunks.
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
from paper_1705_08210_b200.domain import RankCoords  # noqa: E402
from paper_1705_08210_b200.engine3 import Tables, box_plan, box_struct  # noqa: E402
from paper_1705_08210_b200.plan import Box  # noqa: E402


def main():
    n_f = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    only = sys.argv[2] if len(sys.argv) > 2 else None
    n = 6144
    prob = P.Problem(3, n_f, n, P.gen_random_exact(2026, n_f, n, 20), "double")
    dev = torch.device("cuda", 0)
    blk = D.load_block(prob, P.DecompGrid(), RankCoords(0, 0, 0), dev)
    blocks, sums = {0: blk}, {0: D.column_sums(blk)}
    tables = Tables(blocks, N.F64)
    tables(0, 0)
    acc = D.new_acc(dev)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    cases = {
        "volume 512^3 (all tiles full)": Box((0, 0, 0), 0, 512, 2048, 2560, 4096, 4608),
        "volume 1024^3 (all tiles full)": Box((0, 0, 0), 0, 1024, 2048, 3072, 4096, 5120),
        "volume 2048^3 (all tiles full)": Box((0, 0, 0), 0, 2048, 2048, 4096, 4096, 6144),
        "volume 2000^3 (ragged edges)": Box((0, 0, 0), 0, 2000, 2048, 4048, 4096, 6096),
        "diag pivots [2000,2600) full k": Box((0, 0, 0), 0, n, 2000, 2600, 0, n),
        "diag pivots [0,6144) k in [0,1024)": Box((0, 0, 0), 0, n, 0, n, 0, 1024),
        "face I<J=K 3000 rows (FLAT_COLS)": Box((0, 0, 0), 0, 3000, 3000, 6000, 3000, 6000),
        "face I=J<K 3000 cols (FLAT_ROWS)": Box((0, 0, 0), 0, 3000, 0, 3000, 3000, 6000),
        "face small 512 x 1024 (FLAT_COLS)": Box((0, 0, 0), 0, 512, 2048, 3072, 2048, 3072),
        "diag 3000 (PAIR)": Box((0, 0, 0), 0, 3000, 0, 3000, 0, 3000),
    }
    for name, box in cases.items():
        if only and only not in name:
            continue
        probe = box_struct(box, blocks, sums, tables, n_f, n, None, acc)
        n_out, n_tiles = box_plan(probe)
        vals = torch.empty(n_out, dtype=torch.float64, device=dev)
        b = box_struct(box, blocks, sums, tables, n_f, n, vals, acc)
        N.call("psim_czek3_box", N.F64, C.byref(b), D.stream_ptr())
        for fn in ("psim_czek3_box", "psim_czek3_box_numerators"):
            if fn != "psim_czek3_box":  # raw n_ijk (no epilogue) into the same buffer
                N.call(fn, N.F64, C.byref(b), D.stream_ptr())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            N.call(fn, N.F64, C.byref(b), D.stream_ptr())
            e1.record()
            torch.cuda.synchronize()
            s = e0.elapsed_time(e1) * 1e-3
            clk = sms * 1.965e9 * s
            print(json.dumps({"box": name, "fn": fn, "ms": s * 1e3, "tiles": n_tiles,
                              "fill": n_out / (n_tiles * 16384),
                              "useful_cmp_clk_sm": n_out * n_f / clk,
                              "padded_cmp_clk_sm": n_tiles * 16384 * n_f / clk}), flush=True)

if __name__ == "__main__":
    main()
