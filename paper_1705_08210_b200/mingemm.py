"""GPU drop-in for the reference's kernel plug-point module (``propsim.mingemm``).

The reference's ``_dense_kernel(name) -> dense(W, V) -> M`` plug-point
(metrics2.py:41-49, 73-74) and ``cli.bench_kernels`` (cli.py:349-379) call
these functions on host arrays. Here every function keeps the reference's
signature, operand checks (ValueError / DataError) and output contract --
a NEW Fortran-ordered array, inputs not mutated -- and computes on the GPU
through libpsim (include/psim.h); torch only moves the buffers. The values
are bitwise the reference's: each output is one sequential ascending-q sum
from +0 (mingemm.py:79-127), whatever the tile shape, exactly as the
reference's blocked kernel equals its naive one.

Only float32 / float64 operands are supported (the engine's precisions,
core.py:16); other dtypes raise ValueError. ``counter`` (the reference's
OpCounter) is honoured with the same algorithmic counts; the module-wide
op counting of the reference (mingemm.py:24-77) is not rebuilt -- ncu
replaces it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import device as D
from .domain import DataError, unique_tuple_count

DEFAULT_TILE = (64, 128)  # accepted for signature parity (mingemm.py:18); the GPU tile is fixed


def _precision(dt) -> str:
    if dt == np.float64:
        return "double"
    if dt == np.float32:
        return "single"
    raise ValueError(f"unsupported operand dtype {dt} (float32 / float64 only)")


def _check_operands(W: np.ndarray, V: np.ndarray) -> None:
    """mingemm.py:165-171."""
    if W.ndim != 2 or V.ndim != 2:
        raise ValueError("operands must be 2-d")
    if W.shape[0] != V.shape[0]:
        raise ValueError(f"field extents differ: {W.shape[0]} vs {V.shape[0]}")
    if W.dtype != V.dtype:
        raise ValueError(f"operand dtypes differ: {W.dtype} vs {V.dtype}")


def _device() -> torch.device:
    if not torch.cuda.is_available():
        from .domain import EngineError

        raise EngineError("no CUDA device visible: this engine has no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def _to_device(X: np.ndarray, precision: str, dev) -> D.Block:
    """Host (n_f, n) array -> padded column-major device block."""
    host = torch.from_numpy(np.ascontiguousarray(np.asarray(X).T))  # (n, n_f): Fortran bytes
    return D.block_from_host(host, X.shape[0], 0, precision, dev)


def _count(counter, **kw) -> None:
    if counter is not None:
        counter.count(**kw)


def mgemm_blocked(W: np.ndarray, V: np.ndarray, tile: tuple[int, int] = DEFAULT_TILE,
                  counter=None) -> np.ndarray:
    """M[i, j] = sum_q min(W[q, i], V[q, j]) (mgemm_blocked, mingemm.py:189-209)."""
    W, V = np.asarray(W), np.asarray(V)
    _check_operands(W, V)
    ti, tj = tile
    if ti < 1 or tj < 1:
        raise ValueError(f"tile sides must be >= 1, got {tile}")
    prec = _precision(W.dtype)
    nf, m = W.shape
    n = V.shape[1]
    out = np.zeros((m, n), dtype=W.dtype, order="F")
    if m and n:
        dev = _device()
        bw = _to_device(W, prec, dev)
        bv = bw if V is W else _to_device(V, prec, dev)
        M = torch.empty((n, m), dtype=D.torch_dtype(prec), device=dev)  # column-major (m, n)
        N.call("psim_mgemm", D.code_of(prec), D.ptr(bw.data), bw.ld, D.ptr(bv.data), bv.ld, nf,
               m, n, 0, D.ptr(M), m, 0, D.stream_ptr())
        out = np.asfortranarray(M.cpu().numpy().T)
    _count(counter, mins=m * n * nf, adds=m * n * max(nf - 1, 0))
    return out


def mgemm_naive(W: np.ndarray, V: np.ndarray, counter=None) -> np.ndarray:
    """mgemm_naive (mingemm.py:174-186): the same sums, so the same kernel."""
    return mgemm_blocked(W, V, counter=counter)


def column_sums(V: np.ndarray, counter=None) -> np.ndarray:
    """Per-column sums in ascending field order (mingemm.py:212-222)."""
    V = np.asarray(V)
    if V.ndim != 2:
        raise ValueError("operand must be 2-d")
    prec = _precision(V.dtype)
    out = np.zeros(V.shape[1], dtype=V.dtype)
    if V.shape[1]:
        b = _to_device(V, prec, _device())
        out = D.column_sums(b).cpu().numpy()
    _count(counter, adds=max(V.shape[0] - 1, 0) * V.shape[1])
    return out


def xj_columns(V: np.ndarray, vj: np.ndarray, counter=None) -> np.ndarray:
    """Columns np.minimum(v_j, v_k) for every column v_k of V (mingemm.py:225-234)."""
    V, vj = np.asarray(V), np.asarray(vj)
    if vj.shape != (V.shape[0],):
        raise ValueError(f"pivot column shape {vj.shape} does not match field extent {V.shape[0]}")
    prec = _precision(V.dtype)
    out = np.empty(V.shape, dtype=V.dtype, order="F")
    if V.size:
        dev = _device()
        b = _to_device(V, prec, dev)
        x = torch.from_numpy(np.ascontiguousarray(vj, dtype=V.dtype)).to(dev)
        res = torch.empty((V.shape[1], V.shape[0]), dtype=D.torch_dtype(prec), device=dev)
        N.call("psim_min_columns", D.code_of(prec), D.ptr(b.data), V.shape[0], V.shape[1], b.ld,
               D.ptr(x), D.ptr(res), V.shape[0], D.stream_ptr())
        out = np.asfortranarray(res.cpu().numpy().T)
    _count(counter, mins=V.shape[0] * V.shape[1])
    return out


def pair_numerators(V: np.ndarray, counter=None) -> np.ndarray:
    """2-way numerators of all unique column pairs, canonical order
    (mingemm.py:237-247): the symmetric min-plus triangle, packed."""
    V = np.asarray(V)
    prec = _precision(V.dtype)
    nf, n = V.shape
    out = np.zeros(unique_tuple_count(n, 2), dtype=V.dtype)
    if out.size:
        dev = _device()
        b = _to_device(V, prec, dev)
        res = torch.empty(out.size, dtype=D.torch_dtype(prec), device=dev)
        N.call("psim_mgemm", D.code_of(prec), D.ptr(b.data), b.ld, D.ptr(b.data), b.ld, nf, n, n,
               1, D.ptr(res), 0, 1, D.stream_ptr())
        out = res.cpu().numpy()
    _count(counter, mins=nf * out.size, adds=max(nf - 1, 0) * out.size)
    return out


def _canonical_order_of_box(n: int) -> np.ndarray:
    """Canonical triple index of every position of the pivot-major layout of
    the box [0, n)^3 (psim_box3_t: for j ascending, rows i < j, columns k > j)."""
    parts = []
    c3 = lambda x: x * (x - 1) * (x - 2) // 6  # noqa: E731
    for j in range(1, n - 1):
        i = np.arange(j, dtype=np.int64)[:, None]
        k = np.arange(j + 1, n, dtype=np.int64)[None, :]
        m = n - i - 1
        a, bb = j - i - 1, k - i - 1  # pair_index(a, b, m) inside the i-slice
        t = (c3(n) - c3(n - i)) + a * (2 * m - a - 1) // 2 + (bb - a - 1)
        parts.append(t.ravel())
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)


def triple_min_numerators(V: np.ndarray, counter=None) -> np.ndarray:
    """sum_q min(v_i, v_j, v_k) of all unique column triples, canonical order
    (mingemm.py:250-260): one raw 3-way box launch (psim_czek3_box_numerators),
    reordered from pivot-major to canonical on the host."""
    V = np.asarray(V)
    prec = _precision(V.dtype)
    nf, n = V.shape
    count = unique_tuple_count(n, 3)
    out = np.zeros(count, dtype=V.dtype)
    if count:
        dev = _device()
        b = _to_device(V, prec, dev)
        res = torch.empty(count, dtype=D.torch_dtype(prec), device=dev)
        box = N.Box3(n_f=nf, n_v=n, VA=D.ptr(b.data), ldA=b.ld, a0=0, VB=D.ptr(b.data), ldB=b.ld,
                     b0=0, VC=D.ptr(b.data), ldC=b.ld, c0=0, i0=0, i1=n, j0=0, j1=n, k0=0, k1=n,
                     vals=D.ptr(res))
        N.call("psim_czek3_box_numerators", D.code_of(prec), C.byref(box), D.stream_ptr())
        out[_canonical_order_of_box(n)] = res.cpu().numpy()
    _count(counter, mins=2 * nf * count, adds=max(nf - 1, 0) * count)
    return out


@dataclass(frozen=True)
class BitMatrix:
    """Column bit vectors packed 64 rows per word; padding bits are zero
    (mingemm.py:268-276)."""

    words: np.ndarray
    n_rows: int

    @property
    def n_cols(self) -> int:
        return self.words.shape[1]


def pack_bits(V: np.ndarray) -> BitMatrix:
    """Pack a 0/1-valued matrix column-wise (mingemm.py:279-291) on the device
    (psim_pack_bits: warp ballots, 32 rows per word, with the 0/1 check);
    two device words form one of the reference's 64-row uint64 words."""
    V = np.asarray(V)
    if V.ndim != 2:
        raise ValueError("operand must be 2-d")
    nf, n = V.shape
    n64 = (nf + 63) // 64 if nf else 0
    if V.dtype not in (np.float32, np.float64):  # integer / bool input: the same rule on host
        ones = V == 1
        if not (ones | (V == 0)).all():
            raise DataError("bit packing needs entries exactly in {0, 1}")
        V = V.astype(np.float64)
    prec = _precision(V.dtype)
    words = np.zeros((n64, n), dtype=np.uint64)
    if nf and n:
        dev = _device()
        b = _to_device(V, prec, dev)
        ldw = -(-2 * n64 // 4) * 4
        w = torch.zeros((n, ldw), dtype=torch.int32, device=dev)
        flags = torch.zeros(1, dtype=torch.int64, device=dev)
        N.call("psim_pack_bits", D.code_of(prec), D.ptr(b.data), nf, n, b.ld, D.ptr(w), ldw,
               D.ptr(flags), D.stream_ptr())
        if int(flags.item()):
            raise DataError("bit packing needs entries exactly in {0, 1}")
        w32 = np.ascontiguousarray(w.cpu().numpy()[:, :2 * n64]).view(np.uint32)
        words = np.ascontiguousarray(w32.view(np.uint64).T)  # little endian: rows 0-31 low
    return BitMatrix(words=words, n_rows=nf)


def mgemm_bitpacked(A: BitMatrix, B: BitMatrix, counter=None) -> np.ndarray:
    """popcount(a & b) counts as int64, Fortran (m, n) (mingemm.py:294-312)."""
    if A.n_rows != B.n_rows:
        raise ValueError(f"row counts differ: {A.n_rows} vs {B.n_rows}")
    m, n = A.n_cols, B.n_cols
    M = np.zeros((m, n), dtype=np.int64, order="F")
    if A.n_rows and m and n:
        dev = _device()

        def dev_words(X: BitMatrix) -> tuple[torch.Tensor, int]:
            w32 = np.ascontiguousarray(X.words.T).view(np.uint32)  # (cols, 2 * n64)
            ldw = -(-w32.shape[1] // 4) * 4
            host = np.zeros((w32.shape[0], ldw), dtype=np.uint32)
            host[:, :w32.shape[1]] = w32
            return torch.from_numpy(host.view(np.int32)).to(dev), ldw

        wa, lda = dev_words(A)
        wb, ldb = (wa, lda) if B is A else dev_words(B)
        out = torch.empty((n, m), dtype=torch.int64, device=dev)
        N.call("psim_mgemm_bits", D.ptr(wa), lda, D.ptr(wb), ldb, A.n_rows, m, n, D.ptr(out), m,
               D.stream_ptr())
        M = np.asfortranarray(out.cpu().numpy().T)
    _count(counter, mins=m * n * A.n_rows, adds=m * n * max(A.n_rows - 1, 0))
    return M
