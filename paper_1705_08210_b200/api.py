"""Public entry points: drop-in ``run_2way`` / ``run_3way`` (metrics2.py:108-171,
metrics3.py:59-128) returning a ``RunResult`` with the reference's fields
(metrics2.py:52-70).

Differences a caller can see, all documented in INTEGRATION.md:
* ``kernel``: "b200" (default). The reference names "blocked" / "naive"
  are accepted and run the same GPU kernel (they are bitwise-identical
  definitions, mingemm.py:1-7); "bitpacked" selects the same dense GPU
  kernel after checking the input is 0/1 (metric "sorenson").
* ``transport``: "local" (all ranks of the grid on this process's GPU;
  the reference's "thread" / "process" map here) or "nccl" (one process
  per GPU under torch.distributed, world_size == grid.n_p).
* ``timeout`` / ``inject_delay`` / ``delay_seed`` are accepted and ignored:
  device work is stream-ordered and NCCL has its own timeouts.
* ``records`` is a lazy canonical ``Sequence[MetricRecord]``; under
  "nccl" it holds this rank's share; checksum / counts are global.
* ``elapsed`` is the device pipeline time (CUDA events), including input
  generation / upload, excluding the final record materialisation.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import engine2, engine3
from .domain import (
    ConfigError, DataError, EngineError, dtype_of, unique_tuple_count, validate_grid,
)
from .records import LazyRecords
from .synthetic import Checksum128

KERNELS = ("b200", "blocked", "naive", "bitpacked")
TRANSPORTS = ("local", "nccl", "thread", "process")
DEFAULT_TIMEOUT = 30.0


@dataclass
class TrafficStats:
    """Logical send-side traffic (engine.py:51-75 shape)."""

    messages: int = 0
    elements: int = 0
    nbytes: int = 0
    by_phase: dict = field(default_factory=dict)

    def merge(self, other: "TrafficStats") -> None:
        self.messages += other.messages
        self.elements += other.elements
        self.nbytes += other.nbytes
        for ph, (m, e, b) in other.by_phase.items():
            m0, e0, b0 = self.by_phase.get(ph, (0, 0, 0))
            self.by_phase[ph] = (m0 + m, e0 + e, b0 + b)


@dataclass(frozen=True)
class RunResult:
    arity: int
    n_f: int
    n_v: int
    precision: str
    metric: str
    grid: object
    transport: str
    kernel: str
    records: LazyRecords
    checksum: Checksum128
    traffic: TrafficStats
    rank_traffic: dict
    degenerate_count: int
    elapsed: float
    stages: tuple | None = None


def resolve_kernel(metric: str, kernel: str | None) -> str:
    """Mirror of metrics2.py:44-49: Sorenson defaults to the bit-packed path."""
    if kernel is None:
        return "bitpacked" if metric == "sorenson" else "b200"
    if kernel not in KERNELS:
        raise ConfigError(f"kernel must be one of {KERNELS}, got {kernel!r}")
    return "bitpacked" if kernel == "bitpacked" else "b200"


def resolve_transport(transport: str) -> str:
    if transport not in TRANSPORTS:
        raise ConfigError(f"transport must be one of {TRANSPORTS}, got {transport!r}")
    return "nccl" if transport == "nccl" else "local"


def _require_cuda() -> None:
    import torch

    if not torch.cuda.is_available():
        raise EngineError("no CUDA device visible: this engine has no CPU path")


def _check_sorenson(problem) -> None:
    """Sorenson runs need 0/1 input (mingemm.py:279-291, metrics3.py:84-85)."""
    if problem.metric != "sorenson":
        return
    from .synthetic import synthetic_kind

    src = problem.source
    kind = synthetic_kind(src)
    if kind == "random-exact" and src.bits <= 1:
        return
    if kind is not None:
        raise DataError("sorenson runs need strictly 0/1 input")
    arr = np.asarray(src.local_block(problem, _Whole(), _Origin()))
    if not bool(((arr == 0) | (arr == 1)).all()):
        raise DataError("sorenson runs need strictly 0/1 input")


class _Whole:
    n_pf = n_pv = n_pr = n_st = 1


class _Origin:
    p_f = p_v = p_r = 0


def _result(problem, grid, transport, out, stages, kern: str = "b200") -> RunResult:
    expected = unique_tuple_count(problem.n_v, problem.arity)
    if stages is None and out.count != expected:
        raise EngineError(f"schedule covered {out.count} tuples, expected {expected}")
    local = out.count if out.local_count is None else out.local_count
    recs = LazyRecords(problem.arity, problem.n_v, out.pieces, out.sums, local,
                       dtype_of(problem.precision))
    return RunResult(
        arity=problem.arity, n_f=problem.n_f, n_v=problem.n_v, precision=problem.precision,
        metric=problem.metric, grid=grid, transport=transport, kernel=kern, records=recs,
        checksum=Checksum128.from_words(out.lo, out.hi),
        traffic=out.traffic if out.traffic is not None else TrafficStats(),
        rank_traffic=dict(out.rank_traffic), degenerate_count=out.degenerate,
        elapsed=out.elapsed, stages=stages,
    )


def _nccl_runtime():
    """transport="nccl": libpsim's run-level runtime (psim_run2 / psim_run3
    drive the kernels and their own NCCL communicator, runtime.py)."""
    from . import runtime

    return runtime


def run_2way(problem, grid, *, transport: str = "local", kernel: str | None = None,
             timeout: float = DEFAULT_TIMEOUT, inject_delay: float = 0.0, delay_seed: int = 0,
             balance: str = "split", keep_values: bool = True,
             host_values: bool = False) -> RunResult:
    """All unique 2-way Czekanowski metrics of ``problem`` on the GPU(s).

    ``host_values=True`` streams the values into pinned host memory band by
    band while the kernel runs (local transport), so ``records`` are ready
    on the host when the call returns."""
    if problem.arity != 2:
        raise ConfigError(f"run_2way needs an arity-2 problem, got arity={problem.arity}")
    validate_grid(grid, problem.n_f, problem.n_v, 2)
    kern = resolve_kernel(problem.metric, kernel)
    mode = resolve_transport(transport)
    _require_cuda()
    # (like the reference, only the bit-packed path checks for 0/1 input --
    # on the device, while packing: metrics2.py:125-136, mingemm.py:287-288)
    if mode == "nccl":
        if kern == "bitpacked":  # NCCL ranks run the dense kernel: bitwise identical on 0/1
            _check_sorenson(problem)
        out = _nccl_runtime().run(problem, grid, None, keep_values=keep_values,
                                  host_values=host_values, balance=balance)
    else:
        if kern == "bitpacked" and grid.n_pf > 1:
            _check_sorenson(problem)  # field split: dense kernel, identical bits on 0/1
        out = engine2.run_local(problem, grid, balance=balance, keep_values=keep_values,
                                host_values=host_values, bitpacked=(kern == "bitpacked"))
    return _result(problem, grid, mode, out, None, kern)


def run_3way(problem, grid, *, stage: int | None = None, transport: str = "local",
             kernel: str | None = None, timeout: float = DEFAULT_TIMEOUT,
             inject_delay: float = 0.0, delay_seed: int = 0,
             keep_values: bool = True, host_values: bool = False) -> RunResult:
    """All unique 3-way Czekanowski metrics of ``problem`` (or one stage).

    ``host_values=True`` (local transport) streams each box's values to pinned
    host memory in pivot-range chunks while the next chunk computes -- the
    streaming form of the reference's result stages."""
    if problem.arity != 3:
        raise ConfigError(f"run_3way needs an arity-3 problem, got arity={problem.arity}")
    validate_grid(grid, problem.n_f, problem.n_v, 3)
    if stage is not None and not 0 <= stage < grid.n_st:
        raise ConfigError(f"stage must be in [0, {grid.n_st}), got {stage}")
    stages = tuple(range(grid.n_st)) if stage is None else (stage,)
    kern = resolve_kernel(problem.metric, kernel)
    mode = resolve_transport(transport)
    _check_sorenson(problem)  # 3-way always checks (metrics3.py:84-85); dense kernel
    _require_cuda()
    if mode == "nccl":
        out = _nccl_runtime().run(problem, grid, stage, keep_values=keep_values,
                                  host_values=host_values)
    else:
        out = engine3.run_local(problem, grid, stages, keep_values=keep_values,
                                host_values=host_values)
    return _result(problem, grid, mode, out, None if stage is None else stages, kern)
