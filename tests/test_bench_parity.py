"""bench.py's full-size parity checker on CPU, with stand-in runners holding
oracle-computed values: the 2-way piece grid and the 3-way pivot-grid paths
find 0 mismatches on correct values and count a corrupted one, and a checker
that raises is reported in the line instead of ending the bench."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from oracle import propsim_np as O  # noqa: E402
from paper_1705_08210_b200 import Problem, gen_random_exact  # noqa: E402
from paper_1705_08210_b200.plan import Box  # noqa: E402
from paper_1705_08210_b200.records import PairPiece  # noqa: E402

N_F, BITS = 200, 20


def _V(n_v):
    return O.random_exact(bench.SEED, N_F, n_v, BITS)


class Runner2:
    def __init__(self, n_v):
        vals, _, _ = O.run_2way(_V(n_v))
        self.pieces = [PairPiece(0, 0, n_v, n_v, True, 0, n_v, torch.from_numpy(vals.copy()))]


class Runner3:
    """Resident3 stand-in: one pivot chunk [j0, j1) over all i, k, pivot-major."""

    def __init__(self, n_v, j0, j1):
        V = _V(n_v)
        box = Box((0, 0, 0), 0, n_v, j0, j1, 0, n_v)
        out = []
        for j in range(j0, j1):
            for i in range(0, j):
                ks = list(range(j + 1, n_v))
                if ks:
                    out.append(O.triple_values_sampled(V, [(i, j, k) for k in ks]))
        self.stage_boxes = [[box]]
        self.buf = torch.from_numpy(np.concatenate(out))


def test_two_way_checker_counts_mismatches():
    prob = Problem(2, N_F, 60, gen_random_exact(bench.SEED, N_F, 60, BITS), "double")
    r = Runner2(60)
    got = bench.sampled_parity(r, prob, BITS, 1, None)
    assert got["mismatches"] == 0 and got["sampled"] > 100 and "checker_errors" not in got
    r.pieces[0].values[5] += 1.0
    r.pieces[0].values[0] = -1.0
    got = bench.sampled_parity(r, prob, BITS, 1, None)
    # the first pair (0, 1) is always sampled (first row, first column)
    assert got["mismatches"] >= 1


def test_three_way_checker_counts_mismatches():
    n_v = 40
    prob = Problem(3, N_F, n_v, gen_random_exact(bench.SEED, N_F, n_v, BITS), "double")
    r = Runner3(n_v, 10, 30)
    got = bench.sampled_parity(r, prob, BITS, 1, None)
    assert got["mismatches"] == 0 and got["sampled"] > 300
    r.buf[:] = 0.5
    got = bench.sampled_parity(r, prob, BITS, 1, None)
    assert got["mismatches"] == got["sampled"]


def test_checker_failure_is_reported_not_raised():
    class Broken:
        @property
        def pieces(self):
            raise RuntimeError("no values")

    prob = Problem(2, N_F, 60, gen_random_exact(bench.SEED, N_F, 60, BITS), "double")
    got = bench.sampled_parity(Broken(), prob, BITS, 1, None)
    assert got["checker_errors"] == 1 and "no values" in got["how"]


def test_e2e_legs_skip_when_pinned_buffers_exceed_host_memory():
    """cfg5 at N = 4 would pin 4 x 80 GB of input (its ranks were killed by the
    host on the B200 box): the bench reports the e2e leg as skipped instead;
    cfg2 at N = 1 pins 12.8 GB and runs."""
    from paper_1705_08210_b200 import DecompGrid

    a, prec, nf, nv, bits, _ = bench.CONFIGS["cfg5"]
    p5 = Problem(a, nf, nv, gen_random_exact(bench.SEED, nf, nv, bits), prec)
    assert "pinned host buffers" in bench.e2e_host_shortfall(p5, DecompGrid(n_pf=4), 4)
    a, prec, nf, nv, bits, _ = bench.CONFIGS["cfg2"]
    p2 = Problem(a, nf, nv, gen_random_exact(bench.SEED, nf, nv, bits), prec)
    assert bench.e2e_host_shortfall(p2, DecompGrid(), 1) is None
