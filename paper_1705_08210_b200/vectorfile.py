"""Raw vector files as run inputs.

Format (reference io.py:1-14, 55-117): headerless, n_f * n_v little-endian
elements in column order (vector i's fields contiguous), shape and precision
supplied by the caller or a manifest. Column-major on disk equals the HBM
block layout, so a rank's vector slab is one contiguous byte range of the
file (field-split slabs are a strided sub-range of each vector).

``VectorFileSpec`` is a ``Problem`` source like the reference's; when a run
loads it, ``device.load_block`` streams the rank's slab straight from the
file into pinned host chunks and copies them asynchronously into HBM
(``stream_to_device``): no full host copy, no materialised matrix.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from .domain import ConfigError, DataError, dtype_of, field_range, vector_range

CHUNK_BYTES = 256 << 20  # pinned staging chunk


def file_dtype(precision: str) -> np.dtype:
    return np.dtype("<f4" if precision == "single" else "<f8")


@dataclass(frozen=True)
class VectorFileSpec:
    """Location and shape of one raw vector file (reference io.py:55-86)."""

    path: str
    n_f: int
    n_v: int
    precision: str = "double"

    def __post_init__(self) -> None:
        if self.n_f < 1 or self.n_v < 1:
            raise ConfigError(f"vector file needs positive dims, got {self.n_f}x{self.n_v}")
        dtype_of(self.precision)

    @property
    def expected_nbytes(self) -> int:
        return self.n_f * self.n_v * file_dtype(self.precision).itemsize

    def check_size(self) -> None:
        actual = os.path.getsize(self.path)
        if actual != self.expected_nbytes:
            raise DataError(
                f"vector file {self.path}: expected {self.expected_nbytes} bytes "
                f"for {self.n_f}x{self.n_v} {self.precision}, found {actual}")

    def local_block(self, problem, grid, coords) -> np.ndarray:
        """Host read of one rank's slice (compatibility path)."""
        self._check(problem, grid)
        f0, f1 = field_range(grid, coords.p_f, self.n_f)
        v0, v1 = vector_range(grid, coords.p_v, self.n_v)
        mm = np.memmap(self.path, dtype=file_dtype(self.precision), mode="r",
                       shape=(self.n_v, self.n_f))
        return np.array(mm[v0:v1, f0:f1].T, dtype=dtype_of(problem.precision), order="F")

    def _check(self, problem, grid) -> None:
        if (problem.n_f, problem.n_v) != (self.n_f, self.n_v):
            raise ConfigError(f"problem dims ({problem.n_f}, {problem.n_v}) do not match "
                              f"file dims ({self.n_f}, {self.n_v})")
        if self.n_f % grid.n_pf or self.n_v % grid.n_pv:
            raise ConfigError(f"grid does not divide {self.n_f} fields x {self.n_v} vectors")
        self.check_size()


def write_vectors(path, matrix: np.ndarray, precision: str = "double") -> VectorFileSpec:
    """Write a fields x vectors matrix as a raw column-major file (io.py:89-95)."""
    arr = np.asfortranarray(matrix, dtype=file_dtype(precision))
    if not np.isfinite(arr).all():
        raise DataError("non-finite element in vector block")
    if (arr < 0).any():
        raise DataError("negative element in vector block")
    arr.ravel(order="F").tofile(str(path))
    return VectorFileSpec(path=str(path), n_f=arr.shape[0], n_v=arr.shape[1], precision=precision)


def is_vector_file(source) -> bool:
    return all(hasattr(source, a) for a in ("path", "n_f", "n_v", "precision", "check_size"))


def stream_to_device(spec, problem, grid, coords, data: torch.Tensor) -> None:
    """Copy the rank's slab of ``spec`` into the device block ``data``
    ((n_vp, ld) rows = vectors), through two alternating pinned chunks."""
    if hasattr(spec, "_check"):
        spec._check(problem, grid)
    else:
        spec.check_size()
    fdt = file_dtype(spec.precision)
    f0, f1 = field_range(grid, coords.p_f, spec.n_f)
    v0, v1 = vector_range(grid, coords.p_v, spec.n_v)
    n_fp = f1 - f0
    isz = fdt.itemsize
    per = max(1, CHUNK_BYTES // (spec.n_f * isz))  # vectors per chunk
    stage = [torch.empty((per, spec.n_f), dtype=data.dtype, pin_memory=True) for _ in range(2)]
    done = [None, None]
    stream = torch.cuda.current_stream()
    with open(spec.path, "rb", buffering=0) as fh:
        for k, vs in enumerate(range(v0, v1, per)):
            ve = min(v1, vs + per)
            buf = stage[k % 2]
            if done[k % 2] is not None:
                done[k % 2].synchronize()  # its previous H2D has drained
            view = buf[: ve - vs].numpy()
            fh.seek(vs * spec.n_f * isz)
            got = fh.readinto(memoryview(view).cast("B"))
            if got != (ve - vs) * spec.n_f * isz:
                raise DataError(f"short read from {spec.path}")
            data[vs - v0: ve - v0, :n_fp].copy_(buf[: ve - vs, f0:f1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            done[k % 2] = ev
    for ev in done:
        if ev is not None:
            ev.synchronize()
