"""propsim/b200.py -- the binding a propsim maintainer would add to the
reference package to run its metric path on libpsim (include/psim.h).

numpy + ctypes only: no torch, no torch.distributed, no code from this
repository's Python package. The reference's own objects go in unchanged
(duck-typed): ``propsim.Problem`` (core.py:260-293), ``propsim.DecompGrid``
(core.py:44-80), a ``SyntheticSpec`` (verify.py:131-147) or any source with
``local_block``. One call does this rank's whole part of run_2way /
run_3way (psim_run2 / psim_run3: input, column sums, plan, NCCL exchanges,
fused kernels, checksum, gather).

Wiring it into propsim (two lines in metrics2.py / metrics3.py):

    # metrics2.py, top of run_2way:
    if kernel == "b200":
        from . import b200
        return b200.run_2way(problem, grid).to_run_result(problem, grid)

Multi-GPU: one process per GPU; rank 0 calls ``nccl_unique_id()`` and hands
the 128 bytes to the other ranks (any channel: the reference's own socket
transport, a file, MPI); every rank then passes ``rank``, ``world`` and
``nccl_id``. tests/test_gpu_integration.py runs this file as written.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_LIB = None
_i64, _vp = C.c_int64, C.c_void_p


class _Problem(C.Structure):
    _fields_ = [("arity", C.c_int32), ("dtype", C.c_int32), ("n_f", _i64), ("n_v", _i64),
                ("input", C.c_int32), ("bits", C.c_int32), ("seed", C.c_uint64),
                ("block", _vp), ("ld", _i64)]


class _Grid(C.Structure):
    _fields_ = [("n_pf", C.c_int32), ("n_pv", C.c_int32), ("n_pr", C.c_int32),
                ("n_st", C.c_int32)]


class _Piece(C.Structure):
    _fields_ = [("kind", _i64), ("offset", _i64), ("count", _i64), ("v", _i64 * 8)]


class _Traffic(C.Structure):
    _fields_ = [("messages", _i64 * 6), ("elements", _i64 * 6), ("nbytes", _i64 * 6)]


class _Out(C.Structure):
    _fields_ = [("vals", _vp), ("pieces", C.POINTER(_Piece)), ("sums", _vp),
                ("rank_traffic", C.POINTER(_Traffic)), ("n_pieces", _i64), ("n_vals", _i64),
                ("checksum", C.c_uint64 * 2), ("count", _i64), ("degenerate", _i64),
                ("local_count", _i64), ("elapsed", C.c_double), ("traffic", _Traffic),
                ("kernel_seconds", C.c_double), ("kernel_grids", _i64),
                ("scratch_piece", _i64), ("scratch_vals", _vp)]


class _Plan(C.Structure):
    _fields_ = [("n_pieces", _i64), ("n_vals", _i64), ("workspace_bytes", _i64)]


def lib(path: str | None = None) -> C.CDLL:
    """libpsim.so: $PSIM_LIBRARY, else next to this file, else the loader path."""
    global _LIB
    if _LIB is None:
        here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpsim.so")
        path = path or os.environ.get("PSIM_LIBRARY") or (here if os.path.exists(here)
                                                            else "libpsim.so")
        h = C.CDLL(path)
        h.psim_last_error.restype = C.c_char_p
        for name, args in {
            "psim_nccl_unique_id": [_vp],
            "psim_ctx_create": [C.c_int, C.c_int, C.c_int, _vp, C.POINTER(_vp)],
            "psim_ctx_destroy": [_vp],
            "psim_run_plan": [_vp, C.POINTER(_Problem), C.POINTER(_Grid), C.c_int, C.c_int,
                              C.POINTER(_Plan)],
            "psim_run2": [_vp, C.POINTER(_Problem), C.POINTER(_Grid), C.c_int, _vp, _i64,
                          C.POINTER(_Out), _vp],
            "psim_run3": [_vp, C.POINTER(_Problem), C.POINTER(_Grid), C.c_int, C.c_int, _vp,
                          _i64, C.POINTER(_Out), _vp],
            "psim_malloc": [C.POINTER(_vp), _i64, C.c_int],
            "psim_free": [_vp, C.c_int],
            "psim_memcpy": [_vp, _vp, _i64],
        }.items():
            getattr(h, name).argtypes = args
            getattr(h, name).restype = C.c_int
        _LIB = h
    return _LIB


# status codes -> the reference's exception families (core.py:20-29)
def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib().psim_last_error().decode(errors="replace")
    try:  # the reference's own exception classes when propsim is importable
        from propsim.core import ConfigError, DataError, EngineError
    except ImportError:
        ConfigError, DataError, EngineError = ValueError, ValueError, RuntimeError
    raise (ConfigError if status == 1 else DataError if status == 2 else EngineError)(msg)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().psim_nccl_unique_id(buf))
    return buf.raw


_CTX: dict = {}


def _context(device: int, rank: int, world: int, nccl_id: bytes | None):
    key = (device, rank, world)
    if key not in _CTX:
        h = _vp()
        nid = None if nccl_id is None else C.create_string_buffer(nccl_id, 128)
        _check(lib().psim_ctx_create(device, rank, world, nid, C.byref(h)))
        _CTX[key] = h
    return _CTX[key]


class _Buffer:
    def __init__(self, nbytes: int, pinned: bool = False):
        self.ptr, self.pinned = _vp(), pinned
        _check(lib().psim_malloc(C.byref(self.ptr), int(nbytes), int(pinned)))

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value:
            lib().psim_free(self.ptr, int(self.pinned))


@dataclass
class B200Result:
    """What psim_run2 / psim_run3 returned for this rank (global totals,
    this rank's values). ``to_run_result`` builds propsim's RunResult."""

    arity: int
    n_v: int
    precision: str
    checksum: int
    count: int
    degenerate_count: int
    elapsed: float
    values: np.ndarray                 # this rank's values, piece by piece
    pieces: list = field(default_factory=list)  # (kind, v[8], offset, count)
    traffic: dict = field(default_factory=dict)  # phase -> (messages, elements, bytes)

    @property
    def checksum_hex(self) -> str:
        return format(self.checksum, "032x")

    def to_run_result(self, problem=None, grid=None):  # pragma: no cover - needs propsim
        from propsim.core import MetricRecord, TupleId
        from propsim.engine import TrafficStats
        from propsim.metrics2 import RunResult
        from propsim.verify import Checksum128

        recs = []
        for kind, v, off, cnt in self.pieces:
            vals = self.values[off:off + cnt]
            if kind == 2:
                g_row, g_col, m, n, diag, r0, r1, _ = v
                k = 0
                for li in range(r0, r1):
                    for lj in (range(li + 1, m) if diag else range(n)):
                        i, j = sorted((g_row + li, g_col + lj))
                        recs.append(MetricRecord(TupleId((i, j)), vals[k]))
                        k += 1
            else:
                raise NotImplementedError("3-way records: use .values and .pieces")
        recs.sort(key=lambda r: r.id.indices)
        t = TrafficStats()
        for ph, (m, e, b) in self.traffic.items():
            t.by_phase[ph] = (m, e, b)
            t.messages, t.elements, t.nbytes = t.messages + m, t.elements + e, t.nbytes + b
        return RunResult(arity=self.arity, n_f=problem.n_f, n_v=self.n_v,
                         precision=self.precision, metric="czekanowski", grid=grid,
                         transport="nccl", kernel="b200", records=tuple(recs),
                         checksum=Checksum128(self.checksum), traffic=t, rank_traffic={},
                         degenerate_count=self.degenerate_count, elapsed=self.elapsed,
                         stages=None)


_KINDS = {"random-exact": 0, "analytic": 1}


def _run(arity, problem, grid, stage, device, rank, world, nccl_id):
    dtype = 1 if problem.precision == "double" else 0
    p = _Problem(arity=arity, dtype=dtype, n_f=problem.n_f, n_v=problem.n_v)
    src = problem.source
    keep = None
    if getattr(src, "kind", None) in _KINDS and hasattr(src, "seed"):
        p.input, p.seed, p.bits = _KINDS[src.kind], src.seed, getattr(src, "bits", 0)
    else:  # any source: this rank's block, Fortran (n_f / n_pf, n_v / n_pv), on the host
        n_pf, n_pv = grid.n_pf, grid.n_pv
        rank_pf, rest = rank % n_pf, rank // n_pf
        coords = type("Coords", (), {"p_f": rank_pf, "p_v": rest % n_pv, "p_r": rest // n_pv})()
        keep = np.asfortranarray(src.local_block(problem, grid, coords),
                                 dtype=np.float64 if dtype else np.float32)
        p.input, p.block, p.ld = 4, keep.ctypes.data, keep.shape[0]
    g = _Grid(grid.n_pf, grid.n_pv, grid.n_pr, grid.n_st)
    ctx = _context(device, rank, world, nccl_id)
    plan = _Plan()
    st = -1 if stage is None else stage
    _check(lib().psim_run_plan(ctx, C.byref(p), C.byref(g), st, 0, C.byref(plan)))
    ws = _Buffer(plan.workspace_bytes)
    isz = 8 if dtype else 4
    vals = _Buffer(max(1, plan.n_vals) * isz, pinned=True)  # kernels store into host memory
    pieces = (_Piece * max(1, plan.n_pieces))()
    out = _Out(vals=vals.ptr, pieces=pieces)
    if arity == 2:
        _check(lib().psim_run2(ctx, C.byref(p), C.byref(g), 0, ws.ptr, plan.workspace_bytes,
                               C.byref(out), None))
    else:
        _check(lib().psim_run3(ctx, C.byref(p), C.byref(g), st, 0, ws.ptr,
                               plan.workspace_bytes, C.byref(out), None))
    host = np.ctypeslib.as_array(C.cast(vals.ptr, C.POINTER(C.c_double if dtype else C.c_float)),
                                 shape=(max(1, plan.n_vals),))[:out.n_vals].copy()
    traffic = {ph: (out.traffic.messages[ph], out.traffic.elements[ph], out.traffic.nbytes[ph])
               for ph in range(6) if out.traffic.messages[ph]}
    return B200Result(arity, problem.n_v, problem.precision,
                      (out.checksum[1] << 64) | out.checksum[0], out.count, out.degenerate,
                      out.elapsed, host,
                      [(pieces[k].kind, tuple(pieces[k].v), pieces[k].offset, pieces[k].count)
                       for k in range(out.n_pieces)], traffic)


def run_2way(problem, grid, *, device: int = 0, rank: int = 0, world: int = 1,
             nccl_id: bytes | None = None, **_ignored) -> B200Result:
    """run_2way (metrics2.py:108-171) for this rank on libpsim."""
    return _run(2, problem, grid, None, device, rank, world, nccl_id)


def run_3way(problem, grid, *, stage: int | None = None, device: int = 0, rank: int = 0,
             world: int = 1, nccl_id: bytes | None = None, **_ignored) -> B200Result:
    """run_3way (metrics3.py:59-128) for this rank on libpsim."""
    return _run(3, problem, grid, stage, device, rank, world, nccl_id)
