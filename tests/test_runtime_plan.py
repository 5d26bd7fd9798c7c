"""The run-level runtime's planner (csrc/runtime.cu), on CPU through a
planning-only context (device -1): for every grid, the value pieces the
ranks of a run will report (psim_run_pieces) cover every unique pair /
triple exactly once -- the reference's coverage contract (metrics2.py:177-181,
schedule.py:1-15) -- and the 3-way boxes are the Python planner's
(plan.plan_3way / unit_boxes / merge_boxes, schedule.py:184-263)."""
import ctypes as C
import itertools
import math

import numpy as np
import pytest

import paper_1705_08210_b200 as P
from paper_1705_08210_b200 import _native as N
from paper_1705_08210_b200 import plan as PL
from paper_1705_08210_b200.domain import coords_of_rank
from paper_1705_08210_b200.records import BoxPiece, PairPiece


def _pieces(arity, n_f, n_v, grid, rank, stage=-1, flags=0, dtype=N.F64):
    ctx = C.c_void_p()
    world = grid.n_pf * grid.n_pv * grid.n_pr
    N.call("psim_ctx_create", -1, rank, world, None, C.byref(ctx))
    try:
        prob = N.Problem(arity=arity, dtype=dtype, n_f=n_f, n_v=n_v,
                         input=N.INPUT_RANDOM_EXACT, bits=8, seed=1)
        g = N.Grid(n_pf=grid.n_pf, n_pv=grid.n_pv, n_pr=grid.n_pr, n_st=grid.n_st)
        plan = N.Plan()
        N.call("psim_run_plan", ctx, C.byref(prob), C.byref(g), stage, flags, C.byref(plan))
        arr = (N.Piece * max(1, plan.n_pieces))()
        N.call("psim_run_pieces", ctx, C.byref(prob), C.byref(g), stage, flags, C.byref(plan),
               arr, plan.n_pieces)
        assert plan.workspace_bytes > 0
        out, off = [], 0
        for k in range(plan.n_pieces):
            pc = arr[k]
            assert pc.offset == off  # values of a rank are packed in piece order
            off += pc.count
            v = list(pc.v)
            if pc.kind == 2:
                out.append(PairPiece(v[0], v[1], v[2], v[3], bool(v[4]), v[5], v[6], None))
            else:
                out.append(BoxPiece(v[0], v[1], v[2], v[3], v[4], v[5], None, v[6], v[7]))
            assert len(out[-1].canonical(n_v)) == pc.count
        assert off == plan.n_vals
        return out
    finally:
        N.lib().psim_ctx_destroy(ctx)


GRIDS2 = [P.DecompGrid(n_pv=v, n_pr=r, n_pf=f)
          for v, r, f in itertools.product((1, 2, 3, 4, 5, 8), (1, 2, 3), (1, 2, 4))
          if v * r * f <= 32]


@pytest.mark.parametrize("grid", GRIDS2, ids=lambda g: f"pf{g.n_pf}pv{g.n_pv}pr{g.n_pr}")
@pytest.mark.parametrize("balance", [0, N.RUN_BALANCE_REFERENCE])
def test_2way_pieces_cover_every_pair_once(grid, balance):
    n_v = 24 * grid.n_pv
    n_f = 8 * grid.n_pf
    idx = np.concatenate([pc.canonical(n_v) for r in range(grid.n_pf * grid.n_pv * grid.n_pr)
                          for pc in _pieces(2, n_f, n_v, grid, r, flags=balance)])
    assert len(idx) == math.comb(n_v, 2)
    assert (np.sort(idx) == np.arange(math.comb(n_v, 2))).all()


GRIDS3 = [P.DecompGrid(n_pv=v, n_pr=r, n_pf=f, n_st=s)
          for v, r, f, s in itertools.product((1, 2, 3, 4), (1, 2, 3), (1, 2), (1, 2))]


@pytest.mark.parametrize("grid", GRIDS3,
                         ids=lambda g: f"pf{g.n_pf}pv{g.n_pv}pr{g.n_pr}st{g.n_st}")
def test_3way_pieces_cover_every_triple_once(grid):
    n_v = 12 * grid.n_pv
    world = grid.n_pf * grid.n_pv * grid.n_pr
    for stages in ([-1], list(range(grid.n_st))):
        idx = np.concatenate([pc.canonical(n_v) for r in range(world) for s in stages
                              for pc in _pieces(3, 4 * grid.n_pf, n_v, grid, r, stage=s)])
        assert len(idx) == math.comb(n_v, 3)
        assert (np.sort(idx) == np.arange(math.comb(n_v, 3))).all()


@pytest.mark.parametrize("grid", [g for g in GRIDS3 if g.n_pf == 1],
                         ids=lambda g: f"pv{g.n_pv}pr{g.n_pr}st{g.n_st}")
def test_3way_boxes_match_python_planner(grid):
    n_vp = 12
    n_v = n_vp * grid.n_pv
    for rank in range(grid.n_pv * grid.n_pr):
        c = coords_of_rank(rank, grid)
        edge, rest = [], []
        for u in PL.plan_3way(grid, c):
            if isinstance(u, PL.Unit3):
                (edge if u.cls == "edge" else rest).extend(
                    PL.unit_boxes(u, n_vp, grid.n_st, range(grid.n_st)))
        want = [(b.i0, b.i1, b.j0, b.j1, b.k0, b.k1)
                for b in PL.merge_boxes(edge) + PL.merge_boxes(rest) if PL.box_count(b)]
        got = [(p.i0, p.i1, p.j0, p.j1, p.k0, p.k1) for p in _pieces(3, 4, n_v, grid, rank)]
        assert got == want


def test_runtime_rejects_bad_configs():
    ctx = C.c_void_p()
    N.call("psim_ctx_create", -1, 0, 2, None, C.byref(ctx))
    try:
        prob = N.Problem(arity=2, dtype=N.F64, n_f=10, n_v=10, input=N.INPUT_RANDOM_EXACT,
                         bits=8)
        plan = N.Plan()
        g = N.Grid(n_pf=1, n_pv=1, n_pr=1, n_st=1)  # world 2 != 1 rank
        assert N.lib().psim_run_plan(ctx, C.byref(prob), C.byref(g), -1, 0, C.byref(plan)) == 1
        assert b"world size" in N.lib().psim_last_error()
        g = N.Grid(n_pf=1, n_pv=2, n_pr=1, n_st=1)
        prob.n_v = 9  # n_pv must divide n_v
        assert N.lib().psim_run_plan(ctx, C.byref(prob), C.byref(g), -1, 0, C.byref(plan)) == 1
        out = N.Out()
        assert N.lib().psim_run2(ctx, C.byref(prob), C.byref(g), 0, None, 0, C.byref(out),
                                 None) == 1
    finally:
        N.lib().psim_ctx_destroy(ctx)
