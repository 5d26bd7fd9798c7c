"""Multi-GPU runtime: one process per GPU, torch.distributed over NCCL.

Replaces the reference's in-session transports (engine.py:158-216, 230-384):

* block circulation (RankContext.send/receive, metrics2.py:140-147 and
  metrics3.py:93-109) -> grouped NCCL send/recv (``batch_isend_irecv``),
  issued one step ahead so the exchange of step d+1 overlaps the min-plus
  kernel of step d;
* the ordered field-axis fold (reduce_field_axis, engine.py:197-216) ->
  an NCCL all-to-all of row chunks inside each field group, then every
  rank folds its chunk's partials in ascending p_f order on the device
  (bitwise the reference's ((P0 + P1) + P2) + ...)
  and finishes the metric epilogue for those rows, so the reduction is a
  reduce-scatter, not a broadcast;
* result gathering (_gather, metrics2.py:174-203) -> an all-gather of each
  rank's 128-bit checksum words, degenerate and record counts.

The device work per rank is exactly the local engine's (engine2/engine3).
``transport="nccl"`` requires world_size == grid.n_p; rank r takes the
reference's coordinates coords_of_rank(r) (field-fastest, core.py:83-97).
"""
from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from . import device as D
from .domain import ConfigError, RankCoords, coords_of_rank, n_ranks, rank_of_coords
from .engine2 import HostSink, Outcome, finish_numerators, run_task
from .plan import Exchange, Task2, plan_2way
from .records import PairPiece


def ensure_initialized(grid) -> tuple[int, int]:
    """Initialise the default NCCL group from the torchrun environment if needed."""
    if not dist.is_initialized():
        if "RANK" not in os.environ:
            raise ConfigError("transport='nccl' needs a torch.distributed launch (torchrun)")
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    if world != n_ranks(grid):
        raise ConfigError(f"transport='nccl' needs world_size == grid.n_p "
                          f"({world} != {n_ranks(grid)})")
    return world, rank


_GROUPS: dict = {}


def field_group(grid, coords):
    """Process group of the ranks sharing (p_v, p_r) (one slab's field axis)."""
    if grid.n_pf == 1:
        return None
    key = (grid.n_pf, grid.n_pv, grid.n_pr)
    if key not in _GROUPS:
        groups = {}
        for p_r in range(grid.n_pr):
            for p_v in range(grid.n_pv):
                ranks = [rank_of_coords(RankCoords(f, p_v, p_r), grid) for f in range(grid.n_pf)]
                groups[p_v, p_r] = dist.new_group(ranks)  # every rank creates every group
        _GROUPS[key] = groups
    return _GROUPS[key][coords.p_v, coords.p_r]


def row_chunks(m: int, n: int, diagonal: bool, parts: int) -> list[tuple[int, int]]:
    """Split rows [0, m) of a packed task into `parts` contiguous ranges of
    about equal element count (triangle rows hold m-1-i entries)."""
    if diagonal:
        w = np.maximum(m - 1 - np.arange(m, dtype=np.int64), 0)
    else:
        w = np.full(m, n, dtype=np.int64)
    cum = np.concatenate([[0], np.cumsum(w)])
    total = int(cum[-1])
    bounds = [0]
    for p in range(1, parts):
        bounds.append(int(np.searchsorted(cum, total * p / parts, side="left")))
    bounds.append(m)
    bounds = [min(max(b, 0), m) for b in bounds]
    for i in range(1, len(bounds)):
        bounds[i] = max(bounds[i], bounds[i - 1])
    return [(bounds[i], bounds[i + 1]) for i in range(parts)]


def packed_offset(row: int, m: int, n: int, diagonal: bool) -> int:
    return row * (2 * m - row - 1) // 2 if diagonal else row * n


def piece_count(pc) -> int:
    if isinstance(pc, PairPiece):
        return (packed_offset(pc.r1, pc.m, pc.n, pc.diagonal)
                - packed_offset(pc.r0, pc.m, pc.n, pc.diagonal))
    from .plan import Box, box_count

    full = box_count(Box((0, 0, 0), pc.i0, pc.i1, pc.j0, pc.j1, pc.k0, pc.k1))
    return (full if pc.e1 is None else pc.e1) - pc.e0


def gather_totals(acc: torch.Tensor, count: int, world: int, dev) -> tuple[int, int, int, int]:
    """All-gather every rank's (checksum lo, hi, degenerate, count); sum mod 2^128."""
    mine = D.to_device([*D.to_host(acc).tolist(), count], torch.int64, dev)
    allv = torch.empty(world * 4, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allv, mine)
    allv = allv.view(world, 4)
    M64 = (1 << 64) - 1
    total = deg = cnt = 0
    for lo, hi, d, c in D.to_host(allv).tolist():
        total += ((hi & M64) << 64) | (lo & M64)
        deg += d
        cnt += c
    total &= (1 << 128) - 1
    return total & M64, total >> 64, deg, cnt


def reduce_scatter_rows(part: torch.Tensor, m: int, n: int, diagonal: bool, p_f: int, n_pf: int,
                        group, fold) -> tuple[torch.Tensor, int, int]:
    """Ordered field-axis reduction of one task's packed partial numerators.

    Rows are cut into n_pf chunks of ~equal size; field rank f receives
    chunk f from every field rank (one NCCL all-to-all) and folds the
    partials as ((P0 + P1) + P2) + ... with ``fold(dst, src)`` -- the
    reference's ascending-p_f fold (engine.py:197-216), bit for bit.
    Returns (folded chunk, r0, r1)."""
    chunks = row_chunks(m, n, diagonal, n_pf)
    sizes = [packed_offset(b, m, n, diagonal) - packed_offset(a, m, n, diagonal)
             for a, b in chunks]
    mine = sizes[p_f]
    recv = torch.empty(mine * n_pf, dtype=part.dtype, device=part.device)
    dist.all_to_all_single(recv, part, output_split_sizes=[mine] * n_pf,
                           input_split_sizes=sizes, group=group)
    total = recv[:mine].clone()
    for f in range(1, n_pf):
        fold(total, recv[f * mine:(f + 1) * mine])
    r0, r1 = chunks[p_f]
    return total, r0, r1


def reduce_scatter_flat(part: torch.Tensor, p_f: int, n_pf: int, group,
                        fold) -> tuple[torch.Tensor, int, int]:
    """Ordered field-axis reduction of a flat partial array (3-way boxes):
    element range f of n_pf equal ranges goes to field rank f, folded in
    ascending p_f. Returns (folded chunk, e0, e1)."""
    count = part.numel()
    bounds = [count * f // n_pf for f in range(n_pf + 1)]
    sizes = [bounds[f + 1] - bounds[f] for f in range(n_pf)]
    mine = sizes[p_f]
    recv = torch.empty(mine * n_pf, dtype=part.dtype, device=part.device)
    dist.all_to_all_single(recv, part, output_split_sizes=[mine] * n_pf,
                           input_split_sizes=sizes, group=group)
    total = recv[:mine].clone()
    for f in range(1, n_pf):
        fold(total, recv[f * mine:(f + 1) * mine])
    return total, bounds[p_f], bounds[p_f + 1]


def fold_over_field(local_parts: torch.Tensor, code: int, group, n_pf: int) -> torch.Tensor:
    """All-gather a small vector over the field group and fold in p_f order."""
    out = torch.empty(n_pf * local_parts.numel(), dtype=local_parts.dtype,
                      device=local_parts.device)
    dist.all_gather_into_tensor(out, local_parts.contiguous(), group=group)
    out = out.view((n_pf,) + tuple(local_parts.shape))
    total = out[0].clone()
    for p in range(1, n_pf):
        D.fold_(total, out[p], code)
    return total


def exchange_ops(own, own_sums, recv, recv_sums, send_rank: int, recv_rank: int) -> list:
    """One circulant step (metrics2.py:140-147, RankContext.send/receive
    engine.py:177-184): ship the own block and its sums to ``send_rank``,
    receive the peer block and sums from ``recv_rank`` -- one grouped
    send/recv (batch_isend_irecv)."""
    return [
        dist.P2POp(dist.isend, own, send_rank),
        dist.P2POp(dist.isend, own_sums, send_rank),
        dist.P2POp(dist.irecv, recv, recv_rank),
        dist.P2POp(dist.irecv, recv_sums, recv_rank),
    ]


def allgather_ops(me: int, n_pv: int, blocks: dict, sums: dict, peer) -> list:
    """The 3-way block circulation (face_j / vol_k / vol_j exchanges,
    metrics3.py:93-109) as one circulant all-gather: slab ``me`` sends its
    block and sums to me - d and receives slab me + d's, d = 1 .. n_pv - 1
    (blocks / sums: slab -> buffer; peer: slab -> rank)."""
    ops = []
    for d in range(1, n_pv):
        ops.extend(exchange_ops(blocks[me], sums[me], blocks[(me + d) % n_pv],
                                sums[(me + d) % n_pv], peer((me - d) % n_pv),
                                peer((me + d) % n_pv)))
    return ops



class Runner2:
    """One rank's 2-way pipeline over NCCL (also the multi-GPU bench harness)."""

    kernel_name = "k_minplus2<T, kCzek2> (psim_czek2_block)"

    def __init__(self, problem, grid, balance: str = "split", keep_values: bool = True,
                 host_values: bool = False):
        self.world, self.rank = ensure_initialized(grid)
        self.problem, self.grid, self.balance, self.keep = problem, grid, balance, keep_values
        self.sink = HostSink() if host_values else None
        # fused: the diagonal task runs while every block exchange is in flight,
        # then all remaining tasks of the slab share one grid (no per-task tail);
        # host values go zero-copy into pinned buffers (banded copies need the
        # per-task path)
        self.fused = grid.n_pf == 1 and (self.sink is None or self.sink.direct)
        self.coords = coords_of_rank(self.rank, grid)
        self.code = D.code_of(problem.precision)
        self.n_vp = problem.n_v // grid.n_pv
        self.events = plan_2way(grid, self.coords, self.n_vp, balance)
        self.group = field_group(grid, self.coords)
        tasks = [e for e in self.events if isinstance(e, Task2)]
        self.my_cmp = sum(problem.n_f // grid.n_pf * D.pair_count(t.r1 - t.r0, t.c1 - t.c0,
                                                                   t.diagonal) for t in tasks)
        # min-plus grids per step (for the per-launch roofline figure): fused
        # mode runs one group for the diagonal task and one for all others; a
        # field split runs one per task. Launch totals come from libpsim's own
        # counter (psim_launch_count), not from a model of its launch rules.
        if self.fused:
            grids = int(any(t.diagonal for t in tasks)) + int(any(not t.diagonal for t in tasks))
        else:
            grids = len(tasks)
        self.kernel_cmp_per_launch = self.my_cmp / max(1, grids)

    def peer(self, slab: int) -> int:
        c = self.coords
        return rank_of_coords(RankCoords(c.p_f, slab, c.p_r), self.grid)

    def setup(self) -> None:
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        # a pinned host slab (end-to-end use) is uploaded in chunks during the
        # step, overlapped with the diagonal task (_step_streamed)
        self.host, self.flags = None, None
        if self.fused and os.environ.get("PSIM_STREAMED", "1") != "0":
            from .engine2 import pinned_host_block

            self.host = pinned_host_block(self.problem, self.grid, self.coords)
        if self.host is not None:
            n_fp = self.problem.n_f // self.grid.n_pf
            data = D.alloc_block(n_fp, self.n_vp, self.problem.precision, dev)
            self.own = D.Block(data, n_fp, self.n_vp, data.shape[1], self.coords.p_v * self.n_vp,
                               self.problem.precision)
        else:
            self.own = D.load_block(self.problem, self.grid, self.coords, dev)
        # receive buffers: fused mode keeps every received block (all exchanges
        # in flight at once, one multi-task grid after them); otherwise one per
        # in-flight exchange (double buffering). None without a vector split.
        n_ex = sum(1 for e in self.events if isinstance(e, Exchange))
        n_buf = n_ex if self.fused else min(2, n_ex)
        self.remote = [D.Block(torch.empty_like(self.own.data), self.own.n_fp, self.own.n_vp,
                               self.own.ld, 0, self.problem.precision) for _ in range(n_buf)]
        self.remote_sums = [torch.empty(self.n_vp, dtype=self.own.data.dtype, device=dev)
                            for _ in range(n_buf)]
        self.acc = D.new_acc(dev)

    def _sums(self) -> torch.Tensor:
        s = D.column_sums(self.own)
        if self.grid.n_pf > 1:
            s = fold_over_field(s, self.code, self.group, self.grid.n_pf)
        return s

    def _post_exchange(self, ev: Exchange, slot: int, s_own: torch.Tensor):
        return dist.batch_isend_irecv(exchange_ops(
            self.own.data, s_own, self.remote[slot].data, self.remote_sums[slot],
            self.peer(ev.send_to), self.peer(ev.recv_from)))

    def _step_fused(self, s_own, timed: bool) -> list:
        p = self.problem
        tdt = D.torch_dtype(p.precision)
        exchanges = [e for e in self.events if isinstance(e, Exchange)]
        works = []
        slot_of = {}
        for k, ev in enumerate(exchanges):
            slot_of[ev.step] = k
            self.remote[k].v0 = ((self.coords.p_v + ev.step) % self.grid.n_pv) * self.n_vp
            works.extend(self._post_exchange(ev, k, s_own))
        tasks = [e for e in self.events if isinstance(e, Task2)]
        diag = [t for t in tasks if t.diagonal]
        rest = [t for t in tasks if not t.diagonal]
        events, pieces = [], []

        def grid_of(ts, blocks):
            specs = []
            for t, (V, s_col) in zip(ts, blocks):
                m, n = t.r1 - t.r0, t.c1 - t.c0
                cnt = D.pair_count(m, n, t.diagonal)
                if self.sink is not None:  # zero-copy: the epilogue writes pinned host memory
                    vals = self.sink.buffer(cnt, tdt)
                else:
                    vals = torch.empty(cnt, dtype=tdt, device=self.dev) if self.keep else None
                specs.append((self.own, t.r0, t.r1, V, t.c0, t.c1, s_own, s_col, t.diagonal,
                              vals))
                pieces.append(PairPiece(self.own.v0 + t.r0, V.v0 + t.c0, m, n, t.diagonal, 0, m,
                                        vals))
            if not specs:
                return
            if timed:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            D.czek2_tasks(self.code, specs, p.n_v, self.acc)
            if timed:
                e1.record()
                events.append((e0, e1))

        grid_of(diag, [(self.own, s_own)] * len(diag))  # overlaps the exchanges
        for w in works:
            w.wait()
        grid_of(rest, [(self.remote[slot_of[t.step]], self.remote_sums[slot_of[t.step]])
                       for t in rest])
        self.pieces = pieces
        self.s_own = s_own
        return events

    def _step_streamed(self, timed: bool) -> list:
        """Fused step with the own block still in pinned host memory: the
        diagonal task is the streamed kernel (psim_czek2_streamed: the copy
        engine uploads the block in chunks while the kernel starts on the
        tiles whose vectors have landed); the column sums, the device-side
        validation and every block exchange are queued on the copy stream
        behind the upload, so NCCL ships the block as soon as it is in HBM
        while the diagonal task computes; the remaining tasks form one grid."""
        import ctypes as C

        from .engine2 import copy_stream, stream_chunk

        p = self.problem
        tdt = D.torch_dtype(p.precision)
        own, n = self.own, self.n_vp
        copy = copy_stream(self.dev)
        copy.wait_stream(torch.cuda.current_stream())  # buffers of the previous step are free
        chunk = stream_chunk(n)
        bm, _ = N.tile_shape(self.code)
        ready = torch.empty(-(-n // chunk) + -(-n // bm), dtype=torch.int32, device=self.dev)
        s_kernel = torch.empty(n, dtype=tdt, device=self.dev)  # written by the streamed kernel
        cnt = D.pair_count(n, n, True)
        if self.sink is not None:
            vals = self.sink.buffer(cnt, tdt)  # zero-copy host output
        else:
            vals = torch.empty(cnt, dtype=tdt, device=self.dev) if self.keep else None
        t = N.Block2(W=own.data.data_ptr(), ldw=own.ld, V=own.data.data_ptr(), ldv=own.ld,
                     n_f=own.n_fp, m=n, n=n, diagonal=1, g_row=own.v0, g_col=own.v0, n_v=p.n_v,
                     vals=D.ptr(vals), acc=self.acc.data_ptr(), s_row=s_kernel.data_ptr())
        events = []
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        N.call("psim_czek2_streamed", self.code, C.byref(t), self.host.data_ptr(), own.n_fp, chunk,
               ready.data_ptr(), D.stream_ptr(), copy.cuda_stream)
        if timed:
            e1.record()
            events.append((e0, e1))
        exchanges = [e for e in self.events if isinstance(e, Exchange)]
        slot_of, works = {}, []
        with torch.cuda.stream(copy):  # behind the upload
            s_own = D.column_sums(own)  # == the kernel's sums, bit for bit (k_colsum order)
            self.flags = D.check_values_async(own.data, own.n_fp, n, own.ld, self.code)
            for k, ev in enumerate(exchanges):
                slot_of[ev.step] = k
                self.remote[k].v0 = ((self.coords.p_v + ev.step) % self.grid.n_pv) * self.n_vp
                works.extend(self._post_exchange(ev, k, s_own))
        for w in works:
            w.wait()
        torch.cuda.current_stream().wait_stream(copy)
        pieces = [PairPiece(own.v0, own.v0, n, n, True, 0, n, vals)]
        rest = [e for e in self.events if isinstance(e, Task2) and not e.diagonal]
        specs = []
        for tk in rest:
            V, s_col = self.remote[slot_of[tk.step]], self.remote_sums[slot_of[tk.step]]
            m2, n2 = tk.r1 - tk.r0, tk.c1 - tk.c0
            c2 = D.pair_count(m2, n2, False)
            if self.sink is not None:
                v2 = self.sink.buffer(c2, tdt)
            else:
                v2 = torch.empty(c2, dtype=tdt, device=self.dev) if self.keep else None
            specs.append((own, tk.r0, tk.r1, V, tk.c0, tk.c1, s_own, s_col, False, v2))
            pieces.append(PairPiece(own.v0 + tk.r0, V.v0 + tk.c0, m2, n2, False, 0, m2, v2))
        if specs:
            if timed:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            D.czek2_tasks(self.code, specs, p.n_v, self.acc)
            if timed:
                e1.record()
                events.append((e0, e1))
        self.pieces = pieces
        self.s_own = s_own
        return events

    def step(self, timed: bool = False) -> list:
        """Run this rank's whole plan once; returns (start, end) kernel events."""
        p, g = self.problem, self.grid
        self.acc.zero_()
        if self.host is not None:
            return self._step_streamed(timed)
        s_own = self._sums()
        if self.fused:
            return self._step_fused(s_own, timed)
        pieces, events = [], []
        evs = list(self.events)
        exchanges = [e for e in evs if isinstance(e, Exchange)]
        pending = {}
        slot_of = {}
        # post the first exchange before any compute; later ones one step ahead
        if exchanges:
            slot_of[exchanges[0].step] = 0
            pending[exchanges[0].step] = self._post_exchange(exchanges[0], 0, s_own)
        nxt = 1
        for ev in evs:
            if isinstance(ev, Exchange):
                for w in pending.pop(ev.step):
                    w.wait()
                if nxt < len(exchanges):
                    e2 = exchanges[nxt]
                    slot_of[e2.step] = nxt % 2
                    pending[e2.step] = self._post_exchange(e2, nxt % 2, s_own)
                    nxt += 1
                continue
            if ev.diagonal:
                V, s_col = self.own, s_own
            else:
                slot = slot_of[ev.step]
                V, s_col = self.remote[slot], self.remote_sums[slot]
                V.v0 = ev.col_block * self.n_vp
            self.own.v0 = ev.row_block * self.n_vp
            if timed:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            pieces.extend(self._task(ev, V, s_own, s_col))
            if timed:
                e1.record()
                events.append((e0, e1))
        self.pieces = pieces
        self.s_own = s_own
        return events

    def _task(self, t: Task2, V, s_row, s_col) -> list:
        p, g = self.problem, self.grid
        m, n = t.r1 - t.r0, t.c1 - t.c0
        count = D.pair_count(m, n, t.diagonal)
        tdt = D.torch_dtype(p.precision)
        W = self.own
        if g.n_pf == 1:
            return [run_task(self.code, p, g, t, [W], [V], s_row, s_col, self.acc, self.keep,
                             self.sink)]
        # field split: partial packed numerators -> all-to-all row chunks -> ordered fold
        part = torch.empty(count, dtype=tdt, device=self.dev)
        D.mgemm_packed(self.code, W, t.r0, t.r1, V, t.c0, t.c1, t.diagonal, part)
        total, r0, r1 = reduce_scatter_rows(part, m, n, t.diagonal, self.coords.p_f, g.n_pf,
                                            self.group,
                                            lambda dst, src: D.fold_(dst, src, self.code))
        direct = self.sink is not None and self.sink.direct
        keep = self.keep or self.sink is not None
        if direct:  # zero-copy: the epilogue writes pinned host memory
            vals = self.sink.buffer(total.numel(), tdt)
        else:
            vals = torch.empty(total.numel(), dtype=tdt, device=self.dev) if keep else None
        if r1 > r0:
            finish_numerators(self.code, total, r0, r1, m, n, t.diagonal, s_row[t.r0:],
                              s_col[t.c0:], W.v0 + t.r0, V.v0 + t.c0, p.n_v, vals, self.acc)
        if self.sink is not None and not direct:
            host = self.sink.buffer(vals.numel(), tdt)
            self.sink.copy(host, vals, 0, vals.numel())
            vals = host
        return [PairPiece(W.v0 + t.r0, V.v0 + t.c0, m, n, t.diagonal, r0, r1, vals)]

    def checksum_hex(self) -> str:
        lo, hi, _, _ = self.totals()
        from .synthetic import Checksum128

        return Checksum128.from_words(lo, hi).hex

    def totals(self) -> tuple[int, int, int, int]:
        """Global (lo, hi, degenerate, count) over all ranks."""
        count = sum(piece_count(pc) for pc in self.pieces)
        return gather_totals(self.acc, count, self.world, self.dev)

    def global_sums(self) -> np.ndarray:
        out = torch.empty(self.world * self.n_vp, dtype=self.s_own.dtype, device=self.dev)
        dist.all_gather_into_tensor(out, self.s_own.contiguous())
        out = out.view(self.world, self.n_vp)
        host = D.to_host(out)
        sums = np.empty(self.problem.n_v, dtype=host.dtype)
        for r in range(self.world):
            c = coords_of_rank(r, self.grid)
            sums[c.p_v * self.n_vp:(c.p_v + 1) * self.n_vp] = host[r]
        return sums

    def teardown(self) -> None:
        for name in ("own", "remote", "remote_sums", "acc", "pieces"):
            if hasattr(self, name):
                delattr(self, name)
        torch.cuda.empty_cache()


# PSIM_TRACE=1: host perf_counter marks of run_2way_nccl (tools/exp_e2e_nccl.py)
LAST_TRACE: list = []


def _mark(name: str) -> None:
    if os.environ.get("PSIM_TRACE") == "1":
        import time

        LAST_TRACE.append((name, time.perf_counter()))


def run_2way_nccl(problem, grid, balance: str = "split", keep_values: bool = True,
                  host_values: bool = False) -> Outcome:
    LAST_TRACE.clear()
    _mark("enter")
    r = Runner2(problem, grid, balance, keep_values, host_values)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    r.setup()
    _mark("setup")
    r.step()
    _mark("step")
    end.record()
    D.spin_event(end)
    _mark("device")
    if r.sink is not None:
        r.sink.finish()
    if r.flags is not None:  # streamed input, validated on the device: every rank raises
        D.raise_on_stream_abort()
        dist.all_reduce(r.flags)
        D.raise_on_flags(r.flags)
    _mark("flags")
    el = D.to_device([start.elapsed_time(end) * 1e-3], torch.float64, r.dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    lo, hi, deg, cnt = r.totals()
    _mark("totals")
    sums = r.global_sums()
    _mark("sums")
    pieces = r.pieces
    return Outcome(pieces, lo, hi, deg, cnt, sums, float(D.to_host(el)[0]),
                   local_count=sum(piece_count(pc) for pc in pieces))


def run_3way_nccl(problem, grid, stages, keep_values: bool = True) -> Outcome:
    from .engine3 import Runner3Dist

    r = Runner3Dist(problem, grid, stages, keep_values)
    r.setup()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    r.step()
    end.record()
    D.spin_event(end)
    el = D.to_device([start.elapsed_time(end) * 1e-3], torch.float64, r.dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    lo, hi, deg, cnt = r.totals()
    return Outcome(r.pieces, lo, hi, deg, cnt, r.global_sums(), float(D.to_host(el)[0]),
                   local_count=r.count)


Runner3 = None  # set below (avoids an import cycle)


def _bind():
    global Runner3
    from .engine3 import Runner3Dist

    Runner3 = Runner3Dist


_bind()
