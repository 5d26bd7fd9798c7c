"""Per-rank 3-way pipeline on the GPU (the body of run_3way's rank_fn).

Reference: metrics3.py:82-113 (rank_fn), 131-192 (_execute_slice).
The slab plan's units (plan.plan_3way, schedule.py:184-214) become interval
boxes (plan.unit_boxes); each box is one psim_czek3_box launch. The 2-way
numerator tables n_ij / n_ik / n_jk the boxes read are computed once per
block pair with the same min-plus kernel (psim_mgemm), replacing the
reference's per-unit P_bc and per-pivot column_sums(X) (metrics3.py:148-164),
which are bitwise the same numbers (SURVEY Appendix C rule 8).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from . import device as D
from .domain import RankCoords
from .engine2 import Outcome, fold_sums
from .plan import Box, Unit3, merge_boxes, plan_3way, unit_boxes
from .records import BoxPiece


def box_struct(box: Box, blocks: dict, sums: dict, tables, n_f: int, n_v: int,
               vals, acc) -> N.Box3:
    """psim_box3_t for `box`; tables / sums may be None (raw-numerator launches)."""
    A, B, Cb = box.blocks
    bA, bB, bC = blocks[A], blocks[B], blocks[Cb]
    b = N.Box3(
        n_f=n_f, n_v=n_v,
        VA=D.ptr(bA.data), ldA=bA.ld, a0=bA.v0,
        VB=D.ptr(bB.data), ldB=bB.ld, b0=bB.v0,
        VC=D.ptr(bC.data), ldC=bC.ld, c0=bC.v0,
        i0=box.i0, i1=box.i1, j0=box.j0, j1=box.j1, k0=box.k0, k1=box.k1,
        vals=D.ptr(vals), acc=D.ptr(acc),
    )
    if sums is not None:
        b.SA, b.SB, b.SC = D.ptr(sums[A]), D.ptr(sums[B]), D.ptr(sums[Cb])
    if tables is not None:
        NAB, NAC, NBC = tables(A, B), tables(A, Cb), tables(B, Cb)
        b.NAB, b.ldAB = D.ptr(NAB), NAB.shape[1]
        b.NAC, b.ldAC = D.ptr(NAC), NAC.shape[1]
        b.NBC, b.ldBC = D.ptr(NBC), NBC.shape[1]
    return b


def box_plan(b: N.Box3, code: int = N.F64) -> tuple[int, int]:
    n_out, n_tiles = C.c_int64(), C.c_int64()
    N.call("psim_box3_plan", code, C.byref(b), C.byref(n_out), C.byref(n_tiles))
    return n_out.value, n_tiles.value


class Tables:
    """Lazily computed 2-way numerator tables N_XY (column-major, X <= Y)."""

    def __init__(self, blocks: dict, code: int):
        self.blocks, self.code, self.cache = blocks, code, {}

    def __call__(self, X: int, Y: int) -> torch.Tensor:
        key = (X, Y)
        if key not in self.cache:
            bx, by = self.blocks[X], self.blocks[Y]
            out = torch.empty((by.n_vp, bx.n_vp), dtype=bx.data.dtype, device=bx.data.device)
            D.mgemm_square(self.code, bx, by, out, symmetric=(X == Y))
            self.cache[key] = out
        return self.cache[key]


class FoldedTables:
    """Numerator tables over a field split: each field slab's table, folded in
    ascending p_f order (the reference reduces P_bc and the per-pivot
    column sums the same way, metrics3.py:149, 163-164; engine.py:197-216)."""

    def __init__(self, slab_tables: list, code: int):
        self.slab_tables, self.code, self.cache = slab_tables, code, {}

    def __call__(self, X: int, Y: int) -> torch.Tensor:
        if (X, Y) not in self.cache:
            total = self.slab_tables[0](X, Y).clone()
            for t in self.slab_tables[1:]:
                D.fold_(total, t(X, Y), self.code)
            self.cache[X, Y] = total
        return self.cache[X, Y]


def run_boxes_field(code, problem, boxes, slab_blocks, sums, tables, acc, keep_values,
                    pieces) -> int:
    """Boxes over a field split on one device: per-slab raw n_ijk, ordered fold,
    then the epilogue from folded numerators."""
    count = 0
    tdt = D.torch_dtype(problem.precision)
    dev = acc.device
    for box in boxes:
        n_out, _ = box_plan(box_struct(box, slab_blocks[0], None, None, problem.n_f, problem.n_v,
                                       None, acc), code)
        if n_out == 0:
            continue
        total = torch.empty(n_out, dtype=tdt, device=dev)
        part = torch.empty_like(total) if len(slab_blocks) > 1 else None
        for f, blocks in enumerate(slab_blocks):
            dst = total if f == 0 else part
            b = box_struct(box, blocks, None, None, blocks[box.blocks[0]].n_fp, problem.n_v, dst,
                           acc)
            N.call("psim_czek3_box_numerators", code, C.byref(b), D.stream_ptr())
            if f:
                D.fold_(total, part, code)
        vals = torch.empty(n_out, dtype=tdt, device=dev) if keep_values else None
        b = box_struct(box, slab_blocks[0], sums, tables, problem.n_f, problem.n_v, None, acc)
        N.call("psim_czek3_from_numerators", code, C.byref(b), D.ptr(total), 0, n_out,
               D.ptr(vals), D.stream_ptr())
        pieces.append(BoxPiece(box.i0, box.i1, box.j0, box.j1, box.k0, box.k1, vals))
        count += n_out
    return count


def pivot_chunks(box: Box, parts: int) -> list[Box]:
    """Split a box along J into <= parts sub-boxes of about equal output."""
    counts = []
    for j in range(box.j0, box.j1):
        r = max(0, min(box.i1, j) - box.i0)
        c = max(0, box.k1 - max(box.k0, j + 1))
        counts.append(r * c)
    total = sum(counts)
    if total == 0 or parts <= 1:
        return [box]
    out, start, run, k = [], box.j0, 0, 1
    for jj, c in enumerate(counts):
        run += c
        if run >= total * k / parts and box.j0 + jj + 1 < box.j1:
            out.append(Box(box.blocks, box.i0, box.i1, start, box.j0 + jj + 1, box.k0, box.k1))
            start, k = box.j0 + jj + 1, k + 1
    out.append(Box(box.blocks, box.i0, box.i1, start, box.j1, box.k0, box.k1))
    return out


def run_boxes(code, problem, boxes, blocks, sums, tables, acc, keep_values, pieces,
              sink=None) -> int:
    count = 0
    tdt = D.torch_dtype(problem.precision)
    dev = acc.device
    banded = sink is not None and not sink.direct
    if banded:  # pivot-range sub-boxes so each D2H overlaps the next launch
        boxes = [sub for b in boxes for sub in pivot_chunks(b, sink.bands)]
    for box in boxes:
        probe = box_struct(box, blocks, sums, tables, problem.n_f, problem.n_v, None, acc)
        n_out, _ = box_plan(probe)
        if n_out == 0:
            continue
        if sink is not None and sink.direct:  # zero-copy: the kernel writes pinned host memory
            vals = sink.buffer(n_out, tdt)
        else:
            keep = keep_values or sink is not None
            vals = torch.empty(n_out, dtype=tdt, device=dev) if keep else None
        b = box_struct(box, blocks, sums, tables, problem.n_f, problem.n_v, vals, acc)
        N.call("psim_czek3_box", code, C.byref(b), D.stream_ptr())
        if banded:
            host = sink.buffer(n_out, tdt)
            sink.copy(host, vals, 0, n_out)
            vals = host
        pieces.append(BoxPiece(box.i0, box.i1, box.j0, box.j1, box.k0, box.k1, vals))
        count += n_out
    return count


def run_local(problem, grid, stages, keep_values: bool = True,
              host_values: bool = False) -> Outcome:
    from .engine2 import HostSink

    dev = torch.device("cuda", torch.cuda.current_device())
    sink = HostSink() if host_values and grid.n_pf == 1 else None
    code = D.code_of(problem.precision)
    n_vp = problem.n_v // grid.n_pv
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    slab_blocks = [{p: D.load_block(problem, grid, RankCoords(f, p, 0), dev)
                    for p in range(grid.n_pv)} for f in range(grid.n_pf)]
    blocks = slab_blocks[0]
    sums = {p: fold_sums([D.column_sums(sb[p]) for sb in slab_blocks], code)
            for p in range(grid.n_pv)}
    if grid.n_pf == 1:
        tables = Tables(blocks, code)
    else:
        tables = FoldedTables([Tables(sb, code) for sb in slab_blocks], code)
    acc = D.new_acc(dev)
    pieces: list = []
    count = 0
    for p_r in range(grid.n_pr):
        for p_v in range(grid.n_pv):
            boxes = []
            for ev in plan_3way(grid, RankCoords(0, p_v, p_r)):
                if isinstance(ev, Unit3):
                    boxes.extend(unit_boxes(ev, n_vp, grid.n_st, stages))
            if grid.n_pf == 1:
                count += run_boxes(code, problem, merge_boxes(boxes), blocks, sums, tables, acc,
                                   keep_values, pieces, sink)
            else:
                count += run_boxes_field(code, problem, merge_boxes(boxes), slab_blocks, sums,
                                         tables, acc, keep_values, pieces)
    end.record()
    D.spin_event(end)
    if sink is not None:
        sink.finish()
    lo, hi, deg = D.acc_words(acc)
    all_sums = D.to_host(torch.cat([sums[p] for p in range(grid.n_pv)]))
    return Outcome(pieces, lo, hi, deg, count, all_sums, start.elapsed_time(end) * 1e-3)


class Resident3:
    """Benchmark harness for one GPU: input, sums and the 2-way numerator table
    stay resident; each step runs the whole single-slab tetrahedron as boxes
    over consecutive pivot ranges J (each box's values fit ``out_budget``
    bytes), writing all values to a reused HBM buffer and accumulating the
    checksum. Pivot-range boxes keep the full k extent, so tiles are less
    ragged than the reference's k-sliced stages (plan.stage_range)."""

    kernel_name = "k_czek3<T> (psim_czek3_box)"

    def __init__(self, problem, grid, out_budget: float = 40e9):
        from .domain import DecompGrid, n_ranks

        if n_ranks(grid) != 1:
            raise ValueError("Resident3 runs a single-rank grid")
        self.problem = problem
        n, isz = problem.n_v, (8 if problem.precision == "double" else 4)
        cap = max(1, int(out_budget // isz))
        chunks, j0, cnt = [], 0, 0
        for j in range(n):
            c = j * (n - 1 - j)
            if cnt + c > cap and j > j0:
                chunks.append((j0, j))
                j0, cnt = j, 0
            cnt += c
        chunks.append((j0, n))
        self.chunks = chunks
        self.grid = DecompGrid()
        self.code = D.code_of(problem.precision)
        self.kernel_cmp_per_launch = None

    def setup(self) -> None:
        dev = torch.device("cuda", torch.cuda.current_device())
        p, g = self.problem, self.grid
        self.block = D.load_block(p, g, RankCoords(0, 0, 0), dev)
        self.blocks = {0: self.block}
        self.sums = {0: D.column_sums(self.block)}
        self.tables = Tables(self.blocks, self.code)
        self.tables(0, 0)
        self.acc = D.new_acc(dev)
        n = p.n_v
        self.stage_boxes = [[Box((0, 0, 0), 0, n, ja, jb, 0, n)] for ja, jb in self.chunks]
        sizes = []
        for boxes in self.stage_boxes:
            sizes.append(sum(box_plan(box_struct(b, self.blocks, self.sums, self.tables, p.n_f,
                                                 p.n_v, None, self.acc))[0] for b in boxes))
        self.buf = torch.empty(max(sizes), dtype=D.torch_dtype(p.precision), device=dev)
        nb = sum(len(b) for b in self.stage_boxes)
        self.kernel_cmp_per_launch = p.n_f * (p.n_v * (p.n_v - 1) * (p.n_v - 2) // 6) / nb

    def step(self, timed: bool = False) -> list:
        p = self.problem
        self.sums[0] = D.column_sums(self.block)
        D.mgemm_square(self.code, self.block, self.block, self.tables.cache[0, 0], symmetric=True)
        self.acc.zero_()
        events = []
        for boxes in self.stage_boxes:
            off = 0
            for box in boxes:
                probe = box_struct(box, self.blocks, self.sums, self.tables, p.n_f, p.n_v, None,
                                   self.acc)
                n_out, _ = box_plan(probe)
                vals = self.buf[off:off + n_out]
                b = box_struct(box, self.blocks, self.sums, self.tables, p.n_f, p.n_v, vals,
                               self.acc)
                if timed:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                N.call("psim_czek3_box", self.code, C.byref(b), D.stream_ptr())
                if timed:
                    e1.record()
                    events.append((e0, e1))
                off += n_out
        return events

    def checksum_hex(self) -> str:
        from .synthetic import Checksum128

        lo, hi, _ = D.acc_words(self.acc)
        return Checksum128.from_words(lo, hi).hex

    def teardown(self) -> None:
        del self.block, self.blocks, self.sums, self.tables, self.buf, self.acc
        torch.cuda.empty_cache()
