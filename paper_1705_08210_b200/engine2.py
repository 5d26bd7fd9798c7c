"""Per-rank 2-way pipeline on the GPU (the body of run_2way's rank_fn).

Reference: metrics2.py:131-159 (rank_fn), 174-203 (_gather).
For each Task2 of the slab plan (plan.py) one fused kernel computes the
numerators, values, compaction and checksum terms (psim_czek2_block). With a
field split (n_pf > 1) each field slab's partial packed numerators are
folded in ascending p_f order -- the reference's reduce_field_axis
(engine.py:197-216) -- and psim_czek2_from_numerators finishes the task.

Transports:
  "local"  every rank of the grid runs on this process's current GPU, one
           after another; "exchanges" are reads of blocks already in HBM.
           (The reference's "thread" / "process" transports map here.)
  "nccl"   one process per GPU: libpsim's run-level runtime (psim_run2,
           csrc/runtime.cu; runtime.py), world_size == grid.n_p.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import device as D
from .domain import RankCoords, n_ranks
from .plan import Task2, plan_2way
from .records import PairPiece


@dataclass
class Outcome:
    pieces: list
    lo: int = 0
    hi: int = 0
    degenerate: int = 0
    count: int = 0
    sums: np.ndarray | None = None
    elapsed: float = 0.0
    traffic: object = None  # TrafficStats of this process (nccl runtime), else None
    local_count: int | None = None  # records held by this process (nccl: its share)
    rank_traffic: dict = field(default_factory=dict)  # rank -> TrafficStats


def fold_sums(parts: list[torch.Tensor], code: int) -> torch.Tensor:
    """((P0 + P1) + P2) + ... in ascending p_f (engine.py:197-216)."""
    total = parts[0].clone()
    for p in parts[1:]:
        D.fold_(total, p, code)
    return total


class HostSink:
    """Delivers a run's values into pinned host memory.

    ``direct`` (default): the fused kernels store each value straight into
    the pinned buffer (zero-copy: a device store to a UVA host address goes
    over PCIe as the epilogue runs), so a task is ONE launch and nothing is
    left to copy when it ends. ``bands`` (PSIM_HOST_OUTPUT=bands): values go
    to HBM and finished row bands are copied D2H on a side stream while the
    next band's kernel runs. Pinned buffers come from torch's caching host
    allocator (reused once the previous result is released)."""

    def __init__(self, bands: int = 8, direct: bool | None = None):
        import os

        self.bands = bands
        if direct is None:
            direct = os.environ.get("PSIM_HOST_OUTPUT", "direct") != "bands"
        self.direct = direct
        self.stream = torch.cuda.Stream()

    def buffer(self, count: int, dtype) -> torch.Tensor:
        return torch.empty(count, dtype=dtype, pin_memory=True)

    def copy(self, host: torch.Tensor, dev: torch.Tensor, a: int, b: int) -> None:
        ev = torch.cuda.Event()
        ev.record()
        self.stream.wait_event(ev)
        with torch.cuda.stream(self.stream):
            host[a:b].copy_(dev[a:b], non_blocking=True)
        dev.record_stream(self.stream)

    def finish(self) -> None:
        ev = torch.cuda.Event()
        ev.record(self.stream)
        D.spin_event(ev)


def run_task(code: int, problem, grid, task: Task2, row_blocks: list, col_blocks: list,
             s_row: torch.Tensor, s_col: torch.Tensor, acc: torch.Tensor,
             keep_values: bool, sink: HostSink | None = None) -> PairPiece:
    """One Task2 over field-slab lists row_blocks[p_f] / col_blocks[p_f]."""
    m, n = task.r1 - task.r0, task.c1 - task.c0
    count = D.pair_count(m, n, task.diagonal)
    dev = acc.device
    tdt = D.torch_dtype(problem.precision)
    W0, V0 = row_blocks[0], col_blocks[0]
    if len(row_blocks) == 1 and sink is not None and sink.direct:
        host = sink.buffer(count, tdt)  # the kernel stores the values into it
        D.czek2_block(code, W0, task.r0, task.r1, V0, task.c0, task.c1, s_row, s_col,
                      task.diagonal, problem.n_v, host, acc)
        return PairPiece(W0.v0 + task.r0, V0.v0 + task.c0, m, n, task.diagonal, 0, m, host)
    vals = torch.empty(count, dtype=tdt, device=dev) if keep_values or sink else None
    if len(row_blocks) == 1 and sink is not None:
        host = sink.buffer(count, tdt)
        bm, _ = N.tile_shape(code)
        for a, b in D.row_bands(m, n, task.diagonal, sink.bands, bm):
            D.czek2_block(code, W0, task.r0, task.r1, V0, task.c0, task.c1, s_row, s_col,
                          task.diagonal, problem.n_v, vals, acc, band=(a, b))
            sink.copy(host, vals, D.packed_offset(a, m, n, task.diagonal),
                      D.packed_offset(b, m, n, task.diagonal))
        return PairPiece(W0.v0 + task.r0, V0.v0 + task.c0, m, n, task.diagonal, 0, m, host)
    if len(row_blocks) == 1:
        D.czek2_block(code, W0, task.r0, task.r1, V0, task.c0, task.c1, s_row, s_col,
                      task.diagonal, problem.n_v, vals, acc)
    else:
        if sink is not None and sink.direct:  # zero-copy: the epilogue writes pinned host memory
            vals = sink.buffer(count, tdt)
        total = torch.empty(count, dtype=tdt, device=dev)
        D.mgemm_packed(code, W0, task.r0, task.r1, V0, task.c0, task.c1, task.diagonal, total)
        part = torch.empty_like(total)
        for Wp, Vp in zip(row_blocks[1:], col_blocks[1:]):
            D.mgemm_packed(code, Wp, task.r0, task.r1, Vp, task.c0, task.c1, task.diagonal, part)
            D.fold_(total, part, code)
        finish_numerators(code, total, 0, m, m, n, task.diagonal,
                          s_row[task.r0:], s_col[task.c0:], W0.v0 + task.r0, V0.v0 + task.c0,
                          problem.n_v, vals, acc)
        if sink is not None and not sink.direct:
            host = sink.buffer(count, tdt)
            sink.copy(host, vals, 0, count)
            vals = host
    return PairPiece(W0.v0 + task.r0, V0.v0 + task.c0, m, n, task.diagonal, 0, m, vals)


def finish_numerators(code, N, r0, r1, m, n, diagonal, s_row, s_col, g_row, g_col, n_v, vals,
                      acc) -> None:
    from . import _native as Nat
    Nat.call("psim_czek2_from_numerators", code, D.ptr(N), r0, r1, m, n, 1 if diagonal else 0,
             D.ptr(s_row), D.ptr(s_col), g_row, g_col, n_v, D.ptr(vals), D.ptr(acc),
             D.stream_ptr())


_COPY_STREAM: dict = {}


def host_stream_block(problem, grid, coords=None):
    """A generic source's block (default: the single slab) as an (n_vp, n_fp)
    host tensor over the same bytes, for the streamed run: pinned memory is
    uploaded by the copy engine directly, pageable memory is staged through a
    pinned ring chunk by chunk (psim_czek2_streamed). None for synthetic and
    vector-file sources (generated / streamed to the device elsewhere)."""
    import os

    from .domain import host_block
    from .synthetic import synthetic_kind
    from .vectorfile import is_vector_file

    src = problem.source
    if os.environ.get("PSIM_STREAMED", "1") == "0":
        return None
    if synthetic_kind(src) is not None or is_vector_file(src):
        return None
    arr = host_block(problem, grid, coords or RankCoords(0, 0, 0))  # (n_fp, n_vp) Fortran
    return torch.from_numpy(np.ascontiguousarray(arr.T))  # (n_v, n_f), same bytes


# PSIM_TRACE=1: run_streamed records CUDA events (and host clocks) at its
# phase boundaries into LAST_TRACE [(name, event, perf_counter)]
# (diagnostics for tools/exp_e2e.py)
LAST_TRACE: list = []


def _mark(name: str) -> None:
    import os

    if os.environ.get("PSIM_TRACE") == "1":
        import time

        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        LAST_TRACE.append((name, ev, time.perf_counter()))


def copy_stream(dev) -> torch.cuda.Stream:
    """The per-device side stream the streamed inputs are uploaded on."""
    if dev.index not in _COPY_STREAM:
        _COPY_STREAM[dev.index] = torch.cuda.Stream(device=dev)
    return _COPY_STREAM[dev.index]


def stream_chunk(n: int) -> int:
    """Vectors per upload chunk of a streamed block (<= 256 chunks; measured
    on cfg2, tools/exp_stream_order.py: 256 chunks 2.4515 s vs 64 chunks
    2.4557 s per run, the first wave waits less for its rows)."""
    return max(64, -(-n // 256))


def run_streamed(problem, host: torch.Tensor, keep_values: bool, sink) -> Outcome:
    """Single-slab run whose input is still in host memory (pinned, or
    pageable staged through a pinned ring): the copy engine uploads the block
    in chunks (last vectors first) while the fused kernel starts on the bottom
    tiles (psim_czek2_streamed), so the H2D copy is hidden behind the compute
    instead of preceding it; the column sums come out of the kernel. The block is validated (finite, >= 0) once it has
    landed -- before the result is returned."""
    import ctypes as C

    dev = torch.device("cuda", torch.cuda.current_device())
    code = D.code_of(problem.precision)
    n_f, n = problem.n_f, problem.n_v
    tdt = D.torch_dtype(problem.precision)
    copy = copy_stream(dev)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    LAST_TRACE.clear()
    start.record()
    _mark("start")
    data = D.alloc_block(n_f, n, problem.precision, dev)
    ld = data.shape[1]
    chunk = stream_chunk(n)
    bm, _ = N.tile_shape(code)
    ready = torch.empty(-(-n // chunk) + -(-n // bm), dtype=torch.int32, device=dev)
    sums = torch.empty(n, dtype=tdt, device=dev)  # written by the kernel
    count = n * (n - 1) // 2
    if sink is not None:
        vals = sink.buffer(count, tdt)  # zero-copy host output
    else:
        vals = torch.empty(count, dtype=tdt, device=dev) if keep_values else None
    acc = D.new_acc(dev)
    t = N.Block2(W=data.data_ptr(), ldw=ld, V=data.data_ptr(), ldv=ld, n_f=n_f, m=n, n=n,
                 diagonal=1, g_row=0, g_col=0, n_v=n, vals=D.ptr(vals), acc=acc.data_ptr(),
                 s_row=sums.data_ptr())
    _mark("buffers")
    N.call("psim_czek2_streamed", code, C.byref(t), host.data_ptr(), n_f, chunk,
           ready.data_ptr(), D.stream_ptr(), copy.cuda_stream)
    _mark("kernel")
    torch.cuda.current_stream().wait_stream(copy)
    _mark("copies")
    flags = D.check_values_async(data, n_f, n, ld, code)
    _mark("check")
    D.raise_on_flags(flags)  # DataError like VectorBlock (core.py:239-242)
    _mark("checked")
    end.record()
    D.spin_event(end)
    D.raise_on_stream_abort()
    lo, hi, deg = D.acc_words(acc)
    piece = PairPiece(0, 0, n, n, True, 0, n, vals)
    return Outcome([piece], lo, hi, deg, count, D.to_host(sums),
                   start.elapsed_time(end) * 1e-3)


def run_local(problem, grid, balance: str = "split", keep_values: bool = True,
              host_values: bool = False, bitpacked: bool = False) -> Outcome:
    dev = torch.device("cuda", torch.cuda.current_device())
    sink = HostSink() if host_values else None
    bitpacked = bitpacked and grid.n_pf == 1
    code = D.code_of(problem.precision)
    if n_ranks(grid) == 1 and not bitpacked and (sink is None or sink.direct):
        host = host_stream_block(problem, grid)
        if host is not None:
            return run_streamed(problem, host, keep_values, sink)
    n_vp = problem.n_v // grid.n_pv
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    blocks = {}
    for p_f in range(grid.n_pf):
        # the slabs of one field range back to back in one allocation: a rank's
        # consecutive off-diagonal tasks then read one contiguous V operand
        n_fp = problem.n_f // grid.n_pf
        slab = D.alloc_block(n_fp, n_vp * grid.n_pv, problem.precision, dev)
        for p_v in range(grid.n_pv):
            blocks[p_f, p_v] = D.load_block(problem, grid, RankCoords(p_f, p_v, 0), dev,
                                            into=slab[p_v * n_vp:(p_v + 1) * n_vp])
    sums = {p_v: fold_sums([D.column_sums(blocks[p_f, p_v]) for p_f in range(grid.n_pf)], code)
            for p_v in range(grid.n_pv)}
    acc = D.new_acc(dev)
    pieces = []
    count = 0
    specs = []  # single-slab tasks (device or zero-copy host values): batched into shared grids
    tdt = D.torch_dtype(problem.precision)
    bits = {p_v: D.pack_bits(blocks[0, p_v]) for p_v in range(grid.n_pv)} if bitpacked else None
    for p_r in range(grid.n_pr):
        for p_v in range(grid.n_pv):
            for ev in plan_2way(grid, RankCoords(0, p_v, p_r), n_vp, balance):
                if not isinstance(ev, Task2):
                    continue
                rows = [blocks[p_f, ev.row_block] for p_f in range(grid.n_pf)]
                cols = [blocks[p_f, ev.col_block] for p_f in range(grid.n_pf)]
                m, n = ev.r1 - ev.r0, ev.c1 - ev.c0
                if bitpacked:  # Sorenson on 0/1 data: AND + POPC mainloop
                    cnt = D.pair_count(m, n, ev.diagonal)
                    if sink is not None and sink.direct:
                        vals = sink.buffer(cnt, tdt)  # zero-copy host output
                    else:
                        vals = torch.empty(cnt, dtype=tdt, device=dev)
                    Wb, Vb = bits[ev.row_block], bits[ev.col_block]
                    D.sorenson2_block(code, Wb, ev.r0, ev.r1, Vb, ev.c0, ev.c1,
                                      sums[ev.row_block], sums[ev.col_block], ev.diagonal,
                                      problem.n_v, vals, acc)
                    if sink is not None and not sink.direct:
                        host = sink.buffer(vals.numel(), tdt)
                        sink.copy(host, vals, 0, vals.numel())
                        vals = host
                    elif not keep_values:
                        vals = None
                    piece = PairPiece(Wb.v0 + ev.r0, Vb.v0 + ev.c0, m, n, ev.diagonal, 0, m, vals)
                elif grid.n_pf == 1 and (sink is None or sink.direct):
                    cnt = D.pair_count(m, n, ev.diagonal)
                    if sink is not None:  # zero-copy: the kernel writes pinned host memory
                        vals = sink.buffer(cnt, tdt)
                    else:
                        vals = torch.empty(cnt, dtype=tdt, device=dev) if keep_values else None
                    W, V = rows[0], cols[0]
                    specs.append((W, ev.r0, ev.r1, V, ev.c0, ev.c1, sums[ev.row_block],
                                  sums[ev.col_block], ev.diagonal, vals))
                    piece = PairPiece(W.v0 + ev.r0, V.v0 + ev.c0, m, n, ev.diagonal, 0, m, vals)
                else:
                    piece = run_task(code, problem, grid, ev, rows, cols, sums[ev.row_block],
                                     sums[ev.col_block], acc, keep_values, sink)
                pieces.append(piece)
                count += D.pair_count(piece.m, piece.n, piece.diagonal)
    for k in range(0, len(specs), 16):
        D.czek2_tasks(code, specs[k:k + 16], problem.n_v, acc)
    end.record()
    D.spin_event(end)
    if sink is not None:
        sink.finish()
    lo, hi, deg = D.acc_words(acc)
    all_sums = D.to_host(torch.cat([sums[p] for p in range(grid.n_pv)]))
    return Outcome(pieces, lo, hi, deg, count, all_sums, start.elapsed_time(end) * 1e-3)


def ranks(grid) -> int:
    return n_ranks(grid)


class Resident2:
    """Benchmark harness for one GPU: the input block stays resident in HBM and
    each step re-runs the hot path (column sums + the fused 2-way kernel, all
    values written to HBM, checksum accumulated)."""

    kernel_name = "k_minplus2<T, kCzek2> (psim_czek2_block)"

    def __init__(self, problem, grid):
        if n_ranks(grid) != 1:
            raise ValueError("Resident2 runs a single-rank grid")
        self.problem, self.grid = problem, grid
        self.code = D.code_of(problem.precision)
        n = problem.n_v
        self.kernel_cmp_per_launch = problem.n_f * (n * (n - 1) // 2)

    def setup(self) -> None:
        dev = torch.device("cuda", torch.cuda.current_device())
        self.block = D.load_block(self.problem, self.grid, RankCoords(0, 0, 0), dev)
        n = self.problem.n_v
        self.vals = torch.empty(n * (n - 1) // 2, dtype=D.torch_dtype(self.problem.precision),
                                device=dev)
        self.acc = D.new_acc(dev)

    def step(self, timed: bool = False) -> list:
        b = self.block
        s = D.column_sums(b)
        self.acc.zero_()
        sor = self.problem.metric == "sorenson"
        if sor:  # f3: pack 0/1 fields into words, then the AND+POPC kernel
            self.kernel_name = "k_sorenson2<T> (psim_sorenson2_block)"
            bits = D.pack_bits(b)
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        if sor:
            D.sorenson2_block(self.code, bits, 0, b.n_vp, bits, 0, b.n_vp, s, s, True,
                              self.problem.n_v, self.vals, self.acc)
        else:
            D.czek2_block(self.code, b, 0, b.n_vp, b, 0, b.n_vp, s, s, True, self.problem.n_v,
                          self.vals, self.acc)
        if timed:
            e1.record()
            return [(e0, e1)]
        return []

    def checksum_hex(self) -> str:
        from .synthetic import Checksum128

        lo, hi, _ = D.acc_words(self.acc)
        return Checksum128.from_words(lo, hi).hex

    def teardown(self) -> None:
        del self.block, self.vals, self.acc
        torch.cuda.empty_cache()
