"""Per-rank metric output directories.

On-disk contract of the reference (io.py:1-14, 118-371): a directory with
``metrics_<r>.bin`` for every rank of the grid -- values only, each file in
canonical tuple order, ``full`` (little-endian run dtype) or ``byte``
(floor(clamp(v, 0, 1) * 255 + 0.5)) -- and a key=value ``manifest.txt``.
No indices are stored: the owner of a tuple is a pure function of the
configuration (owns_pair / owns_triple, schedule.py:154-177, 266-310).

How this differs from the reference's implementation (same bytes on disk):

* ownership is evaluated for all tuples at once with numpy over canonical
  indices (``pair_owner_ranks`` / ``triple_owner_ranks``) instead of one
  Python call per record, so a 1e9-record directory is written at disk
  speed;
* ``byte`` mode quantises on the GPU (psim_quantize_bytes) while the values
  are still in HBM, so one byte per metric crosses PCIe, not eight;
* under ``transport="nccl"`` every process holds only its share of the
  records: write_run_output is then collective -- each process routes its
  records to the owning rank with one all-to-all (index + payload) and
  writes exactly one file, ``metrics_<rank>.bin``; rank 0 writes the
  manifest. Nothing is gathered to one process.
"""
from __future__ import annotations

import dataclasses
import math
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .domain import (
    ConfigError, DataError, DecompGrid, MetricRecord, TupleId, dtype_of, pair_unindex_np,
    triple_unindex_np,
)

OUTPUT_MODES = ("byte", "full")
MANIFEST_NAME = "manifest.txt"


def file_dtype(precision: str) -> np.dtype:
    """On-disk element type: little-endian f4 / f8 (io.py:47-48)."""
    dtype_of(precision)
    return np.dtype("<f4" if precision == "single" else "<f8")


@dataclass(frozen=True)
class MetricOutputSpec:
    """Output directory + storage mode (io.py:145-161)."""

    directory: str
    mode: str = "full"

    def __post_init__(self) -> None:
        if self.mode not in OUTPUT_MODES:
            raise ConfigError(f"output mode must be one of {OUTPUT_MODES}, got {self.mode!r}")

    def rank_path(self, rank: int) -> str:
        return os.path.join(self.directory, f"metrics_{rank}.bin")

    @property
    def manifest_path(self) -> str:
        return os.path.join(self.directory, MANIFEST_NAME)

    def unit(self, precision: str) -> int:
        return 1 if self.mode == "byte" else file_dtype(precision).itemsize


# ---------------------------------------------------------------------------
# byte quantisation (host forms; the device form is psim_quantize_bytes)


def quantize_byte(value) -> int:
    """One metric to one byte (io.py:122-127)."""
    return int(quantize_values(np.array([value], dtype=np.float64))[0])


def quantize_values(values) -> np.ndarray:
    v = np.asarray(values, dtype=np.float64)
    if not np.isfinite(v).all():
        raise DataError("cannot quantize non-finite metric value")
    return np.floor(np.clip(v, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)


def dequantize_byte(byte: int, precision: str = "double"):
    t = dtype_of(precision).type
    return t(byte) / t(255)


# ---------------------------------------------------------------------------
# ownership, vectorised over canonical indices


def pair_owner_ranks(i, j, n_v: int, grid) -> np.ndarray:
    """Owning rank of each pair i < j: owns_pair (schedule.py:154-177).

    Block pair (bi, bj) lives on slab row ``row`` at circulant step
    ``delta`` (the shorter way round the ring; an even ring's antipodal
    step goes to the lower half), replica p_r = delta mod n_pr, p_f = 0."""
    n_pv = grid.n_pv
    n_vp = n_v // n_pv
    bi, bj = np.asarray(i) // n_vp, np.asarray(j) // n_vp
    half = n_pv // 2
    fwd = (bj - bi) % n_pv
    short = fwd <= half
    row, delta = np.where(short, bi, bj), np.where(short, fwd, n_pv - fwd)
    if n_pv % 2 == 0:
        anti = fwd == half
        row = np.where(anti & (bi >= half), bj, np.where(anti, bi, row))
    same = bi == bj
    row, delta = np.where(same, bi, row), np.where(same, 0, delta)
    return grid.n_pf * (row + n_pv * (delta % grid.n_pr))


def triple_owner_ranks(i, j, k, n_v: int, grid):
    """Owning (rank, stage) of each triple i < j < k: owns_triple
    (schedule.py:266-310), with the slice permutation of _perm_of_rank
    (schedule.py:89-93) for volume blocks."""
    n_pv = grid.n_pv
    n_vp = n_v // n_pv
    i, j, k = np.asarray(i), np.asarray(j), np.asarray(k)
    bi, bj, bk = i // n_vp, j // n_vp, k // n_vp
    pair_lo = (bi == bj) & (bj != bk)     # face with the pair in the low block
    pair_hi = (bi != bj) & (bj == bk)     # face with the pair in the high block
    edge = (bi == bj) & (bj == bk)
    volume = (bi != bj) & (bj != bk)
    # the sliced local index: k for edge / low-pair faces, else i
    sl = np.where(edge | pair_lo, k - bk * n_vp, i - bi * n_vp)
    six = (6 * sl) // n_vp
    lead = np.where(pair_lo, bk, bi)
    other = np.where(pair_lo, bi, bj)
    counter = np.where(edge, six, 6 + six * (n_pv - 1) + ((other - lead) % n_pv) - 1)
    if volume.any():
        first = np.choose(six, [bi, bi, bj, bj, bk, bk])
        rest_lo = np.where(first == bi, bj, bi)
        rest_hi = np.where(first == bk, bj, bk)
        odd = (six & 1) == 1
        second, third = np.where(odd, rest_hi, rest_lo), np.where(odd, rest_lo, rest_hi)
        vol = (6 * n_pv + ((third - first) % n_pv - 1) * (n_pv - 1)
               + ((second - first) % n_pv) - 1)
        lead = np.where(volume, first, lead)
        counter = np.where(volume, vol, counter)
    stage = (sl // (n_vp // (6 * grid.n_st))) % grid.n_st
    return grid.n_pf * (lead + n_pv * (counter % grid.n_pr)), stage


def owner_ranks(arity: int, canon, n_v: int, grid):
    """(rank, stage or None) for an array of canonical indices."""
    if arity == 2:
        return pair_owner_ranks(*pair_unindex_np(canon, n_v), n_v, grid), None
    return triple_owner_ranks(*triple_unindex_np(canon, n_v), n_v, grid)


def owned_canonical(rank: int, *, arity: int, n_v: int, grid, stages=None,
                    chunk: int = 1 << 24) -> np.ndarray:
    """Canonical indices one rank's file holds, in file order (io.py:189-207)."""
    total = math.comb(n_v, arity)
    keep = []
    for a in range(0, total, chunk):
        canon = np.arange(a, min(total, a + chunk), dtype=np.int64)
        owners, stage = owner_ranks(arity, canon, n_v, grid)
        sel = owners == rank
        if arity == 3 and stages is not None:
            sel &= np.isin(stage, np.asarray(list(stages), dtype=np.int64))
        keep.append(canon[sel])
    return np.concatenate(keep) if keep else np.zeros(0, np.int64)


def owned_tuples(rank: int, *, arity: int, n_v: int, grid, stages=None):
    """TupleIds of one rank's file in order (io.py:189-207)."""
    owned = owned_canonical(rank, arity=arity, n_v=n_v, grid=grid, stages=stages)
    cols = pair_unindex_np(owned, n_v) if arity == 2 else triple_unindex_np(owned, n_v)
    for row in zip(*(c.tolist() for c in cols)):
        yield TupleId(tuple(row))


def reconstruct_index(rank: int, position: int, *, arity: int, n_v: int, grid,
                      stages=None) -> TupleId:
    """The tuple at (rank, position) of an output directory (io.py:210-228)."""
    if position < 0:
        raise IndexError(f"position must be nonnegative, got {position}")
    owned = owned_canonical(rank, arity=arity, n_v=n_v, grid=grid, stages=stages)
    if position >= owned.size:
        raise IndexError(f"rank {rank} holds no record at position {position}")
    at = owned[position:position + 1]
    cols = pair_unindex_np(at, n_v) if arity == 2 else triple_unindex_np(at, n_v)
    return TupleId(tuple(int(c[0]) for c in cols))


# ---------------------------------------------------------------------------
# per-rank files


def write_metrics(records, spec: MetricOutputSpec, rank: int, precision: str = "double") -> str:
    """One rank's records (any order) -> its file in canonical order (io.py:164-186)."""
    recs = sorted(records, key=lambda r: r.id.indices)
    os.makedirs(spec.directory, exist_ok=True)
    vals = np.array([r.value for r in recs], dtype=file_dtype(precision))
    path = spec.rank_path(rank)
    (quantize_values(vals) if spec.mode == "byte" else vals).tofile(path)
    return path


def read_metrics(spec: MetricOutputSpec, rank: int, *, arity: int, n_v: int, grid,
                 precision: str = "double", stages=None) -> list[MetricRecord]:
    """One rank's file back into records with their TupleIds (io.py:231-258)."""
    owned = owned_canonical(rank, arity=arity, n_v=n_v, grid=grid, stages=stages)
    values = _read_values(spec, rank, owned.size, precision)
    cols = pair_unindex_np(owned, n_v) if arity == 2 else triple_unindex_np(owned, n_v)
    return [MetricRecord(TupleId(tuple(row)), v)
            for row, v in zip(zip(*(c.tolist() for c in cols)), values)]


def _read_values(spec, rank, n_records, precision) -> np.ndarray:
    path = spec.rank_path(rank)
    want = n_records * spec.unit(precision)
    have = os.path.getsize(path)
    if have != want:
        raise DataError(f"metric file {path}: expected {want} bytes for {n_records} records, "
                        f"found {have}")
    dt = dtype_of(precision)
    if spec.mode == "byte":
        return np.fromfile(path, dtype=np.uint8).astype(dt) / dt.type(255)
    return np.fromfile(path, dtype=file_dtype(precision)).astype(dt)


# ---------------------------------------------------------------------------
# manifests (flat key=value text, io.py:264-306)


def write_manifest(path, entries: dict) -> None:
    text = []
    for key, value in entries.items():
        k, v = f"{key}", f"{value}"
        if "\n" in k + v or "=" in k:
            raise DataError(f"manifest entry {key!r} is not representable as key=value")
        text.append(f"{k}={v}")
    Path(path).write_text("".join(t + "\n" for t in text), encoding="ascii")


def read_manifest(path) -> dict[str, str]:
    out: dict[str, str] = {}
    for n, line in enumerate(Path(path).read_text(encoding="ascii").split("\n"), 1):
        if line:
            key, eq, value = line.partition("=")
            if not eq:
                raise DataError(f"manifest {path} line {n}: missing '='")
            out[key] = value
    return out


def grid_from_manifest(entries: dict) -> DecompGrid:
    return DecompGrid(int(entries["npf"]), int(entries["npv"]), int(entries["npr"]),
                      int(entries.get("num_stage", 1)))


def stages_from_manifest(entries: dict):
    raw = entries.get("stages", "all")
    return None if raw == "all" else tuple(int(s) for s in raw.split(","))


def manifest_entries(result, mode: str, source: dict | None = None) -> dict:
    g = result.grid
    entries = {
        "format": "metrics", "arity": result.arity, "num_field": result.n_f,
        "num_vector": result.n_v, "precision": result.precision, "metric": result.metric,
        "mode": mode, "npf": g.n_pf, "npv": g.n_pv, "npr": g.n_pr, "num_stage": g.n_st,
        "stages": "all" if result.stages is None else ",".join(str(s) for s in result.stages),
        "transport": result.transport, "kernel": result.kernel,
        "record_count": _global_count(result), "degenerate_count": result.degenerate_count,
        "checksum": f"{result.checksum.value:032x}",
    }
    entries.update({f"input_{k}": v for k, v in (source or {}).items()})
    return entries


def _global_count(result) -> int:
    if result.stages is None:
        return math.comb(result.n_v, result.arity)
    return len(result.records) if result.transport != "nccl" else _allreduce_count(result)


def _allreduce_count(result) -> int:
    import torch
    import torch.distributed as dist

    from . import device as D

    dev = _comm_device()
    t = D.to_device([len(result.records)], torch.int64, dev)
    dist.all_reduce(t)
    return int(D.to_host(t)[0])


# ---------------------------------------------------------------------------
# writing a run


def _payload(result, mode: str) -> np.ndarray:
    """This process's values in canonical order as file payload (bytes or
    little-endian values). Byte mode quantises each device piece on the GPU."""
    recs = result.records
    pieces = getattr(recs, "_pieces", None) or []
    if any(p.values is None for p in pieces):
        raise ConfigError("run was made with keep_values=False: no values to write")
    if mode == "byte" and pieces and all(getattr(p.values, "is_cuda", False) for p in pieces):
        return _device_bytes(result, pieces)
    vals = np.asarray(recs.values).astype(file_dtype(result.precision), copy=False)
    return quantize_values(vals) if mode == "byte" else vals


def _device_bytes(result, pieces) -> np.ndarray:
    import torch

    from . import _native as N
    from . import device as D
    from .records import LazyRecords

    code = D.code_of(result.precision)
    dev = pieces[0].values.device
    flag = torch.zeros(1, dtype=torch.int64, device=dev)
    byte_pieces = []
    for p in pieces:
        v = p.values.reshape(-1)
        out = torch.empty(v.numel(), dtype=torch.uint8, device=dev)
        N.call("psim_quantize_bytes", code, D.ptr(v), v.numel(), D.ptr(out), D.ptr(flag),
               D.stream_ptr())
        byte_pieces.append(dataclasses.replace(p, values=out))
    if int(flag.item()):
        raise DataError("cannot quantize non-finite metric value")
    view = LazyRecords(result.arity, result.n_v, byte_pieces, None, len(result.records),
                       np.uint8)
    return view.values


def write_run_output(result, spec: MetricOutputSpec, source: dict | None = None) -> str:
    """Write a finished run: every rank's file plus the manifest; returns the
    manifest path (io.py:310-346). Collective under ``transport="nccl"``."""
    data = _payload(result, spec.mode)  # first: reads the device pieces before they are released
    canon = result.records.canonical_indices
    grid = result.grid
    n_p = grid.n_pf * grid.n_pv * grid.n_pr
    os.makedirs(spec.directory, exist_ok=True)
    if result.transport == "nccl":
        return _write_distributed(result, spec, canon, data, source)
    if n_p == 1:
        data.tofile(spec.rank_path(0))
    else:
        owners, _ = owner_ranks(result.arity, canon, result.n_v, grid)
        order = np.argsort(owners, kind="stable")  # canonical order kept within a rank
        bounds = np.searchsorted(owners[order], np.arange(n_p + 1))
        for r in range(n_p):
            data[order[bounds[r]:bounds[r + 1]]].tofile(spec.rank_path(r))
    write_manifest(spec.manifest_path, manifest_entries(result, spec.mode, source))
    return spec.manifest_path


def _comm_device():
    import torch
    import torch.distributed as dist

    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def route_to_owners(canon: np.ndarray, payload: np.ndarray, owners: np.ndarray, world: int):
    """All-to-all: every process sends each record (canonical index + payload
    bytes) to its owning rank; returns this rank's records in canonical order.
    Works on NCCL (device buffers) and gloo (CPU, tests)."""
    import torch
    import torch.distributed as dist

    dev = _comm_device()
    order = np.argsort(owners, kind="stable")
    send_counts = np.bincount(owners, minlength=world).astype(np.int64)
    sc = torch.from_numpy(send_counts).to(dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc)
    recv_counts = rc.cpu().numpy()
    width = payload.dtype.itemsize
    idx_in = torch.from_numpy(np.ascontiguousarray(canon[order])).to(dev)
    raw = np.ascontiguousarray(payload[order]).view(np.uint8)
    pay_in = torch.from_numpy(raw).to(dev)
    n_in = int(recv_counts.sum())
    idx_out = torch.empty(n_in, dtype=torch.int64, device=dev)
    pay_out = torch.empty(n_in * width, dtype=torch.uint8, device=dev)
    dist.all_to_all_single(idx_out, idx_in, recv_counts.tolist(), send_counts.tolist())
    dist.all_to_all_single(pay_out, pay_in, (recv_counts * width).tolist(),
                           (send_counts * width).tolist())
    idx = idx_out.cpu().numpy()
    vals = pay_out.cpu().numpy().view(payload.dtype)
    keep = np.argsort(idx, kind="stable")
    return idx[keep], vals[keep]


def _write_distributed(result, spec, canon, data, source) -> str:
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    owners, _ = owner_ranks(result.arity, canon, result.n_v, result.grid)
    _, mine = route_to_owners(canon, data, owners, world)
    mine.tofile(spec.rank_path(rank))
    entries = manifest_entries(result, spec.mode, source)  # collective count first
    if rank == 0:
        write_manifest(spec.manifest_path, entries)
    dist.barrier()
    return spec.manifest_path


# ---------------------------------------------------------------------------
# reading a directory


def read_run_output(directory):
    """(manifest entries, {rank: [MetricRecord]}) of a metrics directory
    (io.py:349-371)."""
    entries = read_manifest(Path(directory) / MANIFEST_NAME)
    if entries.get("format") != "metrics":
        raise DataError(f"{directory} is not a metrics directory")
    grid = grid_from_manifest(entries)
    spec = MetricOutputSpec(str(directory), entries["mode"])
    kw = dict(arity=int(entries["arity"]), n_v=int(entries["num_vector"]), grid=grid,
              precision=entries["precision"], stages=stages_from_manifest(entries))
    n_p = grid.n_pf * grid.n_pv * grid.n_pr
    return entries, {r: read_metrics(spec, r, **kw) for r in range(n_p)}


def read_run_values(directory) -> tuple[dict, np.ndarray, np.ndarray]:
    """Whole directory as (entries, canonical indices, values), ascending
    canonical order -- the array form of read_run_output for large runs."""
    entries = read_manifest(Path(directory) / MANIFEST_NAME)
    grid = grid_from_manifest(entries)
    spec = MetricOutputSpec(str(directory), entries["mode"])
    arity, n_v = int(entries["arity"]), int(entries["num_vector"])
    stages = stages_from_manifest(entries)
    idx, vals = [], []
    for r in range(grid.n_pf * grid.n_pv * grid.n_pr):
        owned = owned_canonical(r, arity=arity, n_v=n_v, grid=grid, stages=stages)
        idx.append(owned)
        vals.append(_read_values(spec, r, owned.size, entries["precision"]))
    idx, vals = np.concatenate(idx), np.concatenate(vals)
    order = np.argsort(idx, kind="stable")
    return entries, idx[order], vals[order]
