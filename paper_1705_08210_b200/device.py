"""Device-memory plumbing: vector blocks in HBM and thin launch wrappers.

HBM layout of a vector block (the reference's, core.py:235-236): column
major, vector i's fields contiguous at V[i * ld + q]. ``ld`` is n_fp
rounded up to 32 elements (128 B FP32 / 256 B FP64) so every vector starts
on a 128-byte line and each 128-B field chunk the min-plus kernels stage is
one aligned line. Padding rows are never read (the kernels zero-fill past
n_fp). torch provides allocation and the current stream only; every
arithmetic step is a libpsim kernel.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .domain import DataError, dtype_of, field_range, host_block, vector_range
from .synthetic import synthetic_kind

LD_ALIGN = 32


def ld_for(n_fp: int) -> int:
    return max(LD_ALIGN, -(-n_fp // LD_ALIGN) * LD_ALIGN)


def code_of(precision: str) -> int:
    return N.F64 if precision == "double" else N.F32


def torch_dtype(precision: str):
    return torch.float64 if precision == "double" else torch.float32


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


class Block:
    """One (n_fp x n_vp) vector block in HBM plus its field-folded column sums."""

    __slots__ = ("data", "n_fp", "n_vp", "ld", "v0", "precision", "sums")

    def __init__(self, data, n_fp, n_vp, ld, v0, precision):
        self.data, self.n_fp, self.n_vp, self.ld = data, n_fp, n_vp, ld
        self.v0, self.precision = v0, precision
        self.sums = None

    @property
    def code(self) -> int:
        return code_of(self.precision)

    def col_ptr(self, local_col: int) -> int:
        return self.data.data_ptr() + local_col * self.ld * self.data.element_size()


def alloc_block(n_fp: int, n_vp: int, precision: str, device) -> torch.Tensor:
    return torch.empty((n_vp, ld_for(n_fp)), dtype=torch_dtype(precision), device=device)


def load_block(problem, grid, coords, device, pinned_cache: dict | None = None,
               into: torch.Tensor | None = None) -> Block:
    """The rank's block: generated in HBM for synthetic sources, else copied H2D.

    Generic sources are validated on the device (non-finite / negative ->
    DataError, core.py:239-242). ``into``: an (n_vp, ld) slice of a larger
    allocation to fill (blocks of one field slab back to back, so the
    kernels can stage consecutive blocks as one operand)."""
    n_fp, n_vp = problem.n_f // grid.n_pf, problem.n_v // grid.n_pv
    f0, _ = field_range(grid, coords.p_f, problem.n_f)
    v0, _ = vector_range(grid, coords.p_v, problem.n_v)
    data = alloc_block(n_fp, n_vp, problem.precision, device) if into is None else into
    ld = data.shape[1]
    code = code_of(problem.precision)
    src = problem.source
    kind = synthetic_kind(src)
    st = stream_ptr()
    if kind is not None:
        if hasattr(src, "check_problem"):
            src.check_problem(problem)
        else:  # a reference propsim.verify.SyntheticSpec
            if (problem.n_f, problem.n_v) != (src.n_f, src.n_v):
                from .domain import ConfigError
                raise ConfigError("problem dims do not match synthetic dims")
            src.check_exactness(problem.precision)
        if kind == "random-exact":
            N.call("psim_gen_random_exact", code, src.seed, src.bits, src.n_v, f0, v0, n_fp, n_vp,
                   ptr(data), ld, st)
        elif kind == "analytic":
            N.call("psim_gen_analytic", code, src.n_v, f0, v0, n_fp, n_vp, ptr(data), ld, st)
        else:
            N.call("psim_gen_uniform", code, src.seed, src.n_v, f0, v0, n_fp, n_vp, ptr(data),
                   ld, st)
        return Block(data, n_fp, n_vp, ld, v0, problem.precision)
    from .vectorfile import is_vector_file, stream_to_device

    if is_vector_file(src) and src.precision == problem.precision:
        stream_to_device(src, problem, grid, coords, data)  # file -> pinned chunks -> HBM
        check_values(data, n_fp, n_vp, ld, code)
        return Block(data, n_fp, n_vp, ld, v0, problem.precision)
    arr = host_block(problem, grid, coords)  # (n_fp, n_vp) Fortran
    host = torch.from_numpy(np.ascontiguousarray(arr.T))  # (n_vp, n_fp) == same bytes
    data[:, :n_fp].copy_(host, non_blocking=host.is_pinned())
    check_values(data, n_fp, n_vp, ld, code)
    return Block(data, n_fp, n_vp, ld, v0, problem.precision)


def block_from_host(host: torch.Tensor, n_fp: int, v0: int, precision: str, device) -> Block:
    """Block from a host tensor shaped (n_vp, n_fp) (= Fortran (n_fp, n_vp)).

    Pinned hosts are copied asynchronously on the current stream."""
    n_vp = host.shape[0]
    data = alloc_block(n_fp, n_vp, precision, device)
    data[:, :n_fp].copy_(host, non_blocking=host.is_pinned())
    return Block(data, n_fp, n_vp, data.shape[1], v0, precision)


def check_values_async(data, n_fp, n_vp, ld, code) -> torch.Tensor:
    """Enqueue the device validation; returns the flags for raise_on_flags."""
    flags = torch.zeros(2, dtype=torch.int64, device=data.device)
    N.call("psim_check_block", code, ptr(data), n_fp, n_vp, ld, ptr(flags), stream_ptr())
    return flags


def spin_event(ev) -> None:
    """Wait for a recorded CUDA event by spinning on cudaEventQuery.

    Measured on the B200 boxes (tools/exp_sync.cu, profiles/
    r01_host_sync_latency.jsonl): after a multi-second kernel a blocking wait
    (cudaEventSynchronize, with the default, spin or blocking-sync schedule)
    returned 1-650 ms late; a tight query loop returned within 0.1 ms. Every
    host wait of the run paths after their main kernels goes through here."""
    while not ev.query():
        pass


def spin_wait() -> None:
    """spin_event on an event recorded now on the current stream."""
    ev = torch.cuda.Event()
    ev.record()
    spin_event(ev)


def to_host(t: torch.Tensor) -> np.ndarray:
    """A small device tensor as numpy, through a pinned buffer and spin_wait
    (no blocking copy)."""
    if not t.is_cuda:
        return t.numpy()
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t, non_blocking=True)
    spin_wait()
    return host.numpy()


def to_device(values, dtype, dev) -> torch.Tensor:
    """A small host list as a device tensor without a blocking copy (pinned
    staging + an asynchronous upload; cf. spin_event). CPU devices (gloo
    tests) get a plain tensor."""
    if torch.device(dev).type != "cuda":
        return torch.tensor(values, dtype=dtype, device=dev)
    host = torch.tensor(values, dtype=dtype).pin_memory()
    return host.to(dev, non_blocking=True)


def raise_on_stream_abort() -> None:
    """EngineError when the last streamed kernel gave up waiting for an input
    chunk (psim_stream_error; the kernel exits instead of trapping, so the
    CUDA context stays usable)."""
    import ctypes as C

    from . import _native as N
    from .domain import EngineError

    flag = C.c_uint(0)
    N.call("psim_stream_error", C.byref(flag))
    if flag.value:
        raise EngineError("streamed input did not arrive within 20 s (upload stalled); "
                          "the run's results were discarded")


def raise_on_flags(flags: torch.Tensor) -> None:
    bad, neg = (int(x) for x in to_host(flags))
    if bad:
        raise DataError("non-finite element in vector block")
    if neg:
        raise DataError("negative element in vector block")


def check_values(data, n_fp, n_vp, ld, code) -> None:
    raise_on_flags(check_values_async(data, n_fp, n_vp, ld, code))


def column_sums(block: Block) -> torch.Tensor:
    out = torch.empty(block.n_vp, dtype=block.data.dtype, device=block.data.device)
    N.call("psim_column_sums", block.code, ptr(block.data), block.n_fp, block.n_vp, block.ld,
           ptr(out), stream_ptr())
    return out


def fold_(dst: torch.Tensor, src: torch.Tensor, code: int) -> None:
    """dst <- dst + src elementwise on the device (one ordered fold step)."""
    N.call("psim_fold_add", code, ptr(dst), ptr(src), dst.numel(), stream_ptr())


def new_acc(device) -> torch.Tensor:
    """Device accumulator: [checksum lo, checksum hi, degenerate count] (u64 bits)."""
    return torch.zeros(3, dtype=torch.int64, device=device)


def acc_words(acc: torch.Tensor) -> tuple[int, int, int]:
    lo, hi, deg = (int(x) & ((1 << 64) - 1) for x in to_host(acc).tolist())
    return lo, hi, deg


def czek2_block(code: int, W: Block, r0: int, r1: int, V: Block, c0: int, c1: int,
                s_row: torch.Tensor, s_col: torch.Tensor, diagonal: bool, n_v: int,
                vals: torch.Tensor | None, acc: torch.Tensor, band: tuple[int, int] = (0, 0)
                ) -> None:
    """One fused 2-way task; ``band`` = task-local rows [begin, end) of this launch."""
    t = N.Block2(
        W=W.col_ptr(r0), ldw=W.ld, V=V.col_ptr(c0), ldv=V.ld, n_f=W.n_fp,
        m=r1 - r0, n=c1 - c0, diagonal=1 if diagonal else 0,
        row_begin=band[0], row_end=band[1],
        s_row=s_row.data_ptr() + r0 * s_row.element_size(),
        s_col=s_col.data_ptr() + c0 * s_col.element_size(),
        g_row=W.v0 + r0, g_col=V.v0 + c0, n_v=n_v,
        vals=ptr(vals), acc=ptr(acc),
    )
    N.call("psim_czek2_block", code, C.byref(t), stream_ptr())


class Bits:
    """A bit-packed 0/1 block: 32 fields per uint32 word, vector i's words at
    row i of ``words`` (ld a multiple of 32 words = 128 B)."""

    __slots__ = ("words", "n_fp", "n_vp", "ld", "v0")

    def __init__(self, words, n_fp, n_vp, ld, v0):
        self.words, self.n_fp, self.n_vp, self.ld, self.v0 = words, n_fp, n_vp, ld, v0

    def col_ptr(self, local_col: int) -> int:
        return self.words.data_ptr() + local_col * self.ld * 4


def pack_bits(block: Block) -> Bits:
    """pack_bits (mingemm.py:279-291) on the device; non-0/1 entries -> DataError."""
    nw = -(-block.n_fp // 32)
    ld = max(32, -(-nw // 32) * 32)
    words = torch.empty((block.n_vp, ld), dtype=torch.int32, device=block.data.device)
    flags = torch.zeros(2, dtype=torch.int64, device=block.data.device)
    N.call("psim_pack_bits", block.code, ptr(block.data), block.n_fp, block.n_vp, block.ld,
           ptr(words), ld, ptr(flags), stream_ptr())
    if int(flags[0].item()):
        raise DataError("bit packing needs entries exactly in {0, 1}")
    return Bits(words, block.n_fp, block.n_vp, ld, block.v0)


def sorenson2_block(code: int, W: Bits, r0: int, r1: int, V: Bits, c0: int, c1: int,
                    s_row: torch.Tensor, s_col: torch.Tensor, diagonal: bool, n_v: int,
                    vals: torch.Tensor | None, acc: torch.Tensor) -> None:
    t = N.Block2(
        W=W.col_ptr(r0), ldw=W.ld, V=V.col_ptr(c0), ldv=V.ld, n_f=W.n_fp,
        m=r1 - r0, n=c1 - c0, diagonal=1 if diagonal else 0, row_begin=0, row_end=0,
        s_row=s_row.data_ptr() + r0 * s_row.element_size(),
        s_col=s_col.data_ptr() + c0 * s_col.element_size(),
        g_row=W.v0 + r0, g_col=V.v0 + c0, n_v=n_v, vals=ptr(vals), acc=ptr(acc),
    )
    N.call("psim_sorenson2_block", code, C.byref(t), stream_ptr())


def czek2_tasks(code: int, specs: list, n_v: int, acc: torch.Tensor) -> None:
    """Several fused 2-way tasks in one grid. specs: (W, r0, r1, V, c0, c1,
    s_row, s_col, diagonal, vals) tuples sharing n_f."""
    arr = (N.Block2 * len(specs))()
    for k, (W, r0, r1, V, c0, c1, s_row, s_col, diagonal, vals) in enumerate(specs):
        arr[k] = N.Block2(
            W=W.col_ptr(r0), ldw=W.ld, V=V.col_ptr(c0), ldv=V.ld, n_f=W.n_fp,
            m=r1 - r0, n=c1 - c0, diagonal=1 if diagonal else 0, row_begin=0, row_end=0,
            s_row=s_row.data_ptr() + r0 * s_row.element_size(),
            s_col=s_col.data_ptr() + c0 * s_col.element_size(),
            g_row=W.v0 + r0, g_col=V.v0 + c0, n_v=n_v, vals=ptr(vals), acc=ptr(acc),
        )
    N.call("psim_czek2_tasks", code, arr, len(specs), stream_ptr())


def mgemm_packed(code: int, W: Block, r0: int, r1: int, V: Block, c0: int, c1: int,
                 diagonal: bool, out: torch.Tensor) -> None:
    N.call("psim_mgemm", code, W.col_ptr(r0), W.ld, V.col_ptr(c0), V.ld, W.n_fp, r1 - r0, c1 - c0,
           1 if diagonal else 0, ptr(out), 0, 1, stream_ptr())


def mgemm_square(code: int, W: Block, V: Block, out: torch.Tensor, symmetric: bool) -> None:
    """Column-major numerator table out[x + y*ld] (ld = out.shape[1]) for all
    pairs of W's and V's vectors."""
    N.call("psim_mgemm", code, ptr(W.data), W.ld, ptr(V.data), V.ld, W.n_fp, W.n_vp, V.n_vp,
           1 if symmetric else 0, ptr(out), out.shape[1], 0, stream_ptr())


def pair_count(m: int, n: int, diagonal: bool) -> int:
    return m * (m - 1) // 2 if diagonal else m * n


def packed_offset(row: int, m: int, n: int, diagonal: bool) -> int:
    """Start of task-local row `row` in the packed layout (triangle / rectangle)."""
    return row * (2 * m - row - 1) // 2 if diagonal else row * n


def row_bands(m: int, n: int, diagonal: bool, parts: int, align: int) -> list[tuple[int, int]]:
    """Cut rows [0, m) into <= `parts` bands of about equal element count whose
    starts are multiples of `align` (the kernel's CTA tile height)."""
    total = pair_count(m, n, diagonal)
    bounds = [0]
    for p in range(1, parts):
        target = total * p / parts
        lo, hi = bounds[-1], m
        while lo < hi:  # first row whose packed start reaches the target
            mid = (lo + hi) // 2
            if packed_offset(mid, m, n, diagonal) < target:
                lo = mid + 1
            else:
                hi = mid
        b = (lo // align) * align
        if b > bounds[-1]:
            bounds.append(b)
    bounds.append(m)
    return [(bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1) if bounds[i + 1] > bounds[i]]


def dtype_np(precision: str):
    return dtype_of(precision)
