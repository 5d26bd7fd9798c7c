"""Binding of libpsim's run-level runtime (csrc/runtime.cu, include/psim.h).

``run_2way`` / ``run_3way`` with ``transport="nccl"`` come here: this
process's whole part of the run -- the reference's rank_fn
(metrics2.py:131-159, metrics3.py:82-113) with its send / receive /
reduce_field_axis (engine.py:158-216) and the _gather of metrics2.py:174-203
-- is ONE call into libpsim (psim_run2 / psim_run3), which drives the
kernels and its own NCCL communicator. Python only allocates the buffers
(torch), hands over pointers and wraps the result; torch.distributed is used
once, to pass rank 0's 128-byte NCCL id to the other ranks.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _native as N
from . import device as D
from .domain import ConfigError, coords_of_rank, host_block, n_ranks
from .engine2 import Outcome
from .records import BoxPiece, PairPiece

_CTX: dict = {}


class Context:
    """psim_ctx of this process (device, rank, world; NCCL comm for world > 1)."""

    def __init__(self, device: int, rank: int, world: int, nccl_id: bytes | None):
        h = C.c_void_p()
        buf = None if nccl_id is None else C.create_string_buffer(nccl_id, N_ID)
        N.call("psim_ctx_create", device, rank, world, buf, C.byref(h))
        self.handle, self.device, self.rank, self.world = h, device, rank, world

    def close(self) -> None:
        if self.handle:
            N.lib().psim_ctx_destroy(self.handle)
            self.handle = None


N_ID = 128


def unique_id() -> bytes:
    buf = C.create_string_buffer(N_ID)
    N.call("psim_nccl_unique_id", buf)
    return buf.raw


def context(world: int, rank: int) -> Context:
    """The process's context for this world (created once; collective)."""
    dev = torch.cuda.current_device()
    key = (dev, world, rank)
    if key not in _CTX:
        nid = None
        if world > 1:
            import torch.distributed as dist

            obj = [unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, 0)  # plumbing: 128 bytes, once per process
            nid = obj[0]
        _CTX[key] = Context(dev, rank, world, nid)
    return _CTX[key]


def problem_struct(problem, grid, coords, dev) -> tuple[N.Problem, object]:
    """psim_problem_t for this rank plus whatever must stay alive during the run."""
    from .synthetic import synthetic_kind
    from .vectorfile import is_vector_file

    p = N.Problem(arity=problem.arity, dtype=D.code_of(problem.precision), n_f=problem.n_f,
                  n_v=problem.n_v)
    src = problem.source
    kind = synthetic_kind(src)
    if kind is not None:
        if hasattr(src, "check_problem"):
            src.check_problem(problem)
        else:  # a reference propsim.verify.SyntheticSpec
            if (problem.n_f, problem.n_v) != (src.n_f, src.n_v):
                raise ConfigError("problem dims do not match synthetic dims")
            src.check_exactness(problem.precision)
        p.input = {"random-exact": N.INPUT_RANDOM_EXACT, "analytic": N.INPUT_ANALYTIC,
                   "uniform": N.INPUT_UNIFORM}[kind]
        p.seed = src.seed & ((1 << 64) - 1)
        p.bits = getattr(src, "bits", 0)
        return p, None
    if is_vector_file(src):  # file -> pinned chunks -> HBM, validated on the device
        blk = D.load_block(problem, grid, coords, dev)
        p.input, p.block, p.ld = N.INPUT_DEVICE, blk.data.data_ptr(), blk.ld
        return p, blk
    arr = host_block(problem, grid, coords)  # (n_fp, n_vp) Fortran, run dtype
    if arr.size and arr.strides[0] != arr.itemsize:
        arr = np.asfortranarray(arr)
    p.input, p.block = N.INPUT_HOST, arr.ctypes.data
    p.ld = arr.strides[1] // arr.itemsize if arr.shape[1] > 1 else arr.shape[0]
    return p, arr


def grid_struct(grid) -> N.Grid:
    return N.Grid(n_pf=grid.n_pf, n_pv=grid.n_pv, n_pr=grid.n_pr, n_st=grid.n_st)


def traffic_stats(t: N.Traffic):
    from .api import TrafficStats

    st = TrafficStats()
    for ph in range(N.PHASES):
        m, e, b = t.messages[ph], t.elements[ph], t.nbytes[ph]
        if m:
            st.by_phase[ph] = (m, e, b)
            st.messages += m
            st.elements += e
            st.nbytes += b
    return st


class Run:
    """One prepared psim_run2 / psim_run3 call: plan, workspace, outputs.

    ``step()`` runs it (again); the benchmark's multi-GPU harness re-runs the
    same prepared call with the input resident in HBM."""

    def __init__(self, problem, grid, stage: int | None = None, keep_values: bool = True,
                 host_values: bool = False, balance: str = "split", scratch_values: bool = False,
                 world: int | None = None, rank: int | None = None, device_block=None):
        if world is None:
            from .dist import ensure_initialized

            world, rank = ensure_initialized(grid)
        if world != n_ranks(grid):
            raise ConfigError(f"transport='nccl' needs world_size == grid.n_p "
                              f"({world} != {n_ranks(grid)})")
        self.problem, self.grid, self.world, self.rank = problem, grid, world, rank
        self.ctx = context(world, rank)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.coords = coords_of_rank(rank, grid)
        if device_block is not None:  # this rank's block, resident in HBM (D.Block)
            self.prob = N.Problem(arity=problem.arity, dtype=D.code_of(problem.precision),
                                  n_f=problem.n_f, n_v=problem.n_v, input=N.INPUT_DEVICE,
                                  block=device_block.data.data_ptr(), ld=device_block.ld)
            self._keep = device_block
        else:
            self.prob, self._keep = problem_struct(problem, grid, self.coords, self.dev)
        self.gr = grid_struct(grid)
        self.stage = -1 if stage is None else stage
        self.flags = (N.RUN_BALANCE_REFERENCE if balance == "reference" else 0) | \
            (N.RUN_VALUES_SCRATCH if scratch_values else 0)
        if balance not in ("split", "reference"):
            raise ConfigError(f"balance must be 'split' or 'reference', got {balance!r}")
        plan = N.Plan()
        N.call("psim_run_plan", self.ctx.handle, C.byref(self.prob), C.byref(self.gr),
               self.stage, self.flags, C.byref(plan))
        self.plan = plan
        self.ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=self.dev)
        tdt = D.torch_dtype(problem.precision)
        self.vals = None
        if keep_values and not scratch_values:
            if host_values:  # zero-copy: the kernels store into pinned host memory
                self.vals = torch.empty(plan.n_vals, dtype=tdt, pin_memory=True)
            else:
                self.vals = torch.empty(plan.n_vals, dtype=tdt, device=self.dev)
        self.pieces = (N.Piece * max(1, plan.n_pieces))()
        self.sums = torch.empty(problem.n_v, dtype=tdt, pin_memory=True)
        self.rank_traffic = (N.Traffic * world)()
        self.out = None

    def step(self) -> N.Out:
        out = N.Out(vals=D.ptr(self.vals), pieces=self.pieces, sums=self.sums.data_ptr(),
                    rank_traffic=self.rank_traffic)
        fn = "psim_run2" if self.problem.arity == 2 else "psim_run3"
        args = (self.ctx.handle, C.byref(self.prob), C.byref(self.gr))
        if self.problem.arity == 3:
            args = args + (self.stage,)
        N.call(fn, *args, self.flags, self.ws.data_ptr(), self.ws.numel(), C.byref(out),
               D.stream_ptr())
        self.out = out
        return out

    def outcome(self) -> Outcome:
        out = self.out
        pieces = []
        for k in range(out.n_pieces):
            pc = self.pieces[k]
            v = list(pc.v)
            vals = None if self.vals is None else self.vals[pc.offset:pc.offset + pc.count]
            if pc.kind == 2:
                pieces.append(PairPiece(v[0], v[1], v[2], v[3], bool(v[4]), v[5], v[6], vals))
            else:
                pieces.append(BoxPiece(v[0], v[1], v[2], v[3], v[4], v[5], vals, v[6], v[7]))
        res = Outcome(pieces, out.checksum[0], out.checksum[1], out.degenerate, out.count,
                      self.sums.numpy().copy(), out.elapsed, local_count=out.local_count)
        res.traffic = traffic_stats(out.traffic)
        res.rank_traffic = {r: traffic_stats(self.rank_traffic[r]) for r in range(self.world)}
        return res


def run(problem, grid, stage: int | None = None, keep_values: bool = True,
        host_values: bool = False, balance: str = "split") -> Outcome:
    """This rank's part of run_2way / run_3way (transport "nccl")."""
    r = Run(problem, grid, stage, keep_values, host_values, balance)
    r.step()
    return r.outcome()


def close_all() -> None:
    for c in _CTX.values():
        c.close()
    _CTX.clear()


if os.environ.get("PSIM_RUNTIME_ATEXIT", "1") == "1":
    import atexit

    atexit.register(close_all)
