"""Symmetry-eliminating work plans: 2-way circulant, 3-way tetrahedral.

Every unique pair / triple is produced exactly once across the grid
(coverage contract: metrics2.py:177-181, schedule.py:1-15).

2-way (schedule.py:116-142). Slab p_v handles offsets delta = 0..n_pv//2
round-robined over replicas (delta mod n_pr == p_r); delta > 0 needs the
block of slab p_v + delta, received while the own block goes to p_v - delta.
The reference keeps the even-n_pv half-offset block entirely on the lower
slab (schedule.py:130-136), which caps load balance at 67% / 80% / 89% for
n_pv = 2 / 4 / 8. Here, by default (``balance="split"``), both
slabs that already hold that block pair after the exchange compute half of
it: the lower slab its first n_vp//2 rows, the upper slab the complementary
columns of its transposed view. ``balance="reference"`` restores the
reference rule. Results and checksums are unaffected by the choice.

3-way (schedule.py:184-310). The three-phase slab walk is kept as is: six
diagonal-edge sixths, 6*(n_pv-1) face sixths, (n_pv-1)(n_pv-2) volume
slices, with the same exchanges and replica round-robin. Each unit (and each
stage sub-range of its sliced axis, schedule.py:103-109) is an interval box
I x J x K over canonical (i < j < k) ids, which is what the GPU kernel
consumes (psim_box3_t).
"""
from __future__ import annotations

from dataclasses import dataclass

from .domain import ConfigError, RankCoords, coords_of_rank, n_ranks, rank_of_coords

BALANCES = ("split", "reference")


@dataclass(frozen=True)
class Exchange:
    """Send the own block to slab ``send_to``, receive slab ``recv_from``'s."""

    kind: str  # "pair" | "face_j" | "vol_k" | "vol_j"
    step: int
    send_to: int
    recv_from: int


@dataclass(frozen=True)
class Task2:
    """Rows [r0, r1) of block ``row_block`` against columns [c0, c1) of ``col_block``.

    Ranges are block-local. ``diagonal`` tasks (row_block == col_block)
    keep only li < lj.
    """

    step: int
    row_block: int
    col_block: int
    r0: int
    r1: int
    c0: int
    c1: int

    @property
    def diagonal(self) -> bool:
        return self.row_block == self.col_block


def plan_2way(grid, coords, n_vp: int, balance: str = "split") -> tuple:
    """Ordered Exchange / Task2 events of one rank (field peers share them)."""
    if balance not in BALANCES:
        raise ConfigError(f"balance must be one of {BALANCES}, got {balance!r}")
    n_pv, p, p_r = grid.n_pv, coords.p_v, coords.p_r
    half = n_pv // 2
    out: list = []
    for delta in range(half + 1):
        if delta % grid.n_pr != p_r:
            continue
        if delta == 0:
            out.append(Task2(0, p, p, 0, n_vp, 0, n_vp))
            continue
        col = (p + delta) % n_pv
        out.append(Exchange("pair", delta, (p - delta) % n_pv, col))
        if n_pv % 2 == 0 and delta == half:
            if balance == "reference":
                if p < half:
                    out.append(Task2(delta, p, col, 0, n_vp, 0, n_vp))
            elif p < half:
                out.append(Task2(delta, p, col, 0, n_vp // 2, 0, n_vp))
            else:
                out.append(Task2(delta, p, col, 0, n_vp, n_vp // 2, n_vp))
            continue
        out.append(Task2(delta, p, col, 0, n_vp, 0, n_vp))
    return tuple(out)


def tasks_2way(grid, n_vp: int, balance: str = "split") -> dict[int, tuple[Task2, ...]]:
    """Task lists per rank (the field axis shares its slab's tasks)."""
    out = {}
    for rank in range(n_ranks(grid)):
        c = coords_of_rank(rank, grid)
        out[rank] = tuple(e for e in plan_2way(grid, c, n_vp, balance) if isinstance(e, Task2))
    return out


def owns_pair(i: int, j: int, n_v: int, grid, balance: str = "reference") -> tuple[int, int]:
    """(rank with p_f = 0, task position) computing canonical pair (i, j) under
    the given plan balance; the default is the reference's owner
    (schedule.py:154-177), the one output files are laid out by."""
    if not 0 <= i < j < n_v:
        raise ValueError(f"need 0 <= i < j < n_v, got ({i}, {j})")
    if n_v % grid.n_pv:
        raise ConfigError(f"n_pv={grid.n_pv} does not divide n_v={n_v}")
    n_vp = n_v // grid.n_pv
    for rank, tasks in tasks_2way(grid, n_vp, balance).items():
        if coords_of_rank(rank, grid).p_f:
            continue
        for pos, t in enumerate(tasks):
            for a, b in ((i, j), (j, i)):
                ra, rb = divmod(a, n_vp), divmod(b, n_vp)
                if (ra[0], rb[0]) == (t.row_block, t.col_block) and t.r0 <= ra[1] < t.r1 \
                        and t.c0 <= rb[1] < t.c1 and (not t.diagonal or ra[1] < rb[1]):
                    return rank, pos
    raise AssertionError("pair not covered")  # unreachable for a valid plan


# ---------------------------------------------------------------------------
# 3-way


@dataclass(frozen=True)
class Unit3:
    """One slice unit (schedule.py:45-59): blocks in role order and its sixth."""

    blocks: tuple[int, int, int]
    cls: str  # "edge" | "face" | "volume"
    slice_index: int
    counter: int


@dataclass(frozen=True)
class Box:
    """Canonical interval box: (i, j, k) in [i0,i1) x [j0,j1) x [k0,k1), i<j<k.

    ``blocks`` = slabs holding I, J and K (ascending)."""

    blocks: tuple[int, int, int]
    i0: int
    i1: int
    j0: int
    j1: int
    k0: int
    k1: int


def sixth_bounds(s: int, n: int) -> tuple[int, int]:
    if not 0 <= s < 6:
        raise ValueError(f"slice index must be in [0, 6), got {s}")
    return (s * n) // 6, ((s + 1) * n) // 6


def stage_range(s_t: int, s: int, n_vp: int, n_st: int) -> tuple[int, int]:
    """Sub-range of sixth s for stage s_t; all (s_t, s) tile [0, n_vp) (schedule.py:103-109)."""
    if not 0 <= s_t < n_st:
        raise ValueError(f"stage must be in [0, {n_st}), got {s_t}")
    return ((s_t + n_st * s) * n_vp) // (6 * n_st), ((s_t + 1 + n_st * s) * n_vp) // (6 * n_st)


def _perm_rank(I: int, J: int, K: int) -> int:
    """Lexicographic rank of (I, J, K) among the orderings of its blocks."""
    order = sorted((I, J, K))
    first = order.index(I)
    rest = [b for b in (I, J, K)[1:]]
    return 2 * first + (1 if rest[0] > rest[1] else 0)


def plan_3way(grid, coords) -> tuple:
    """Ordered Exchange / Unit3 events of one rank's slab (schedule.py:184-214)."""
    n_pv, n_pr, p, p_r = grid.n_pv, grid.n_pr, coords.p_v, coords.p_r
    out: list = []
    counter = 0
    for s in range(6):
        if counter % n_pr == p_r:
            out.append(Unit3((p, p, p), "edge", s, counter))
        counter += 1
    for s in range(6):
        for dj in range(1, n_pv):
            if counter % n_pr == p_r:
                J = (p + dj) % n_pv
                out.append(Exchange("face_j", counter, (p - dj) % n_pv, J))
                out.append(Unit3((p, J, J), "face", s, counter))
            counter += 1
    for dk in range(1, n_pv):
        K = (p + dk) % n_pv
        out.append(Exchange("vol_k", dk, (p - dk) % n_pv, K))
        for dj in range(1, n_pv):
            if counter % n_pr == p_r and dj != dk:
                J = (p + dj) % n_pv
                out.append(Exchange("vol_j", counter, (p - dj) % n_pv, J))
                out.append(Unit3((p, J, K), "volume", _perm_rank(p, J, K), counter))
            counter += 1
    return tuple(out)


def unit_boxes(unit: Unit3, n_vp: int, n_st: int, stages) -> list[Box]:
    """Canonical boxes covering ``unit`` for the given stages (schedule.py:231-263)."""
    out = []
    for s_t in stages:
        lo, hi = stage_range(s_t, unit.slice_index, n_vp, n_st)
        if unit.cls == "edge":
            p = unit.blocks[0]
            b = p * n_vp
            out.append(Box((p, p, p), b, b + n_vp, b, b + n_vp, b + lo, b + hi))
        elif unit.cls == "face":
            p, J, _ = unit.blocks
            if p < J:
                bp, bj = p * n_vp, J * n_vp
                out.append(Box((p, J, J), bp + lo, bp + hi, bj, bj + n_vp, bj, bj + n_vp))
            else:
                bp, bj = p * n_vp, J * n_vp
                out.append(Box((J, J, p), bj, bj + n_vp, bj, bj + n_vp, bp + lo, bp + hi))
        else:
            A, B, Cb = sorted(unit.blocks)
            ba, bb, bc = A * n_vp, B * n_vp, Cb * n_vp
            out.append(Box((A, B, Cb), ba + lo, ba + hi, bb, bb + n_vp, bc, bc + n_vp))
    return out


def merge_boxes(boxes: list[Box]) -> list[Box]:
    """Join boxes that differ only by adjacent K (or I) intervals, e.g. the
    six edge sixths of an unstaged single slab become one launch."""
    out: list[Box] = []
    for b in boxes:
        if out:
            a = out[-1]
            if (a.blocks, a.i0, a.i1, a.j0, a.j1) == (b.blocks, b.i0, b.i1, b.j0, b.j1) \
                    and a.k1 == b.k0:
                out[-1] = Box(a.blocks, a.i0, a.i1, a.j0, a.j1, a.k0, b.k1)
                continue
            if (a.blocks, a.j0, a.j1, a.k0, a.k1) == (b.blocks, b.j0, b.j1, b.k0, b.k1) \
                    and a.i1 == b.i0:
                out[-1] = Box(a.blocks, a.i0, b.i1, a.j0, a.j1, a.k0, a.k1)
                continue
        out.append(b)
    return out


def box_count(b: Box) -> int:
    """Number of (i<j<k) triples in a box (exact, host integer arithmetic)."""
    total = 0
    for j in range(b.j0, b.j1):
        r = max(0, min(b.i1, j) - b.i0)
        c = max(0, b.k1 - max(b.k0, j + 1))
        total += r * c
    return total


def owns_triple(i: int, j: int, k: int, n_v: int, grid) -> tuple[int, int, int]:
    """(rank with p_f = 0, stage, unit position) of canonical triple (i, j, k)."""
    if not 0 <= i < j < k < n_v:
        raise ValueError(f"need 0 <= i < j < k < n_v, got ({i}, {j}, {k})")
    n_vp = n_v // grid.n_pv
    for p_r in range(grid.n_pr):
        for p in range(grid.n_pv):
            c = RankCoords(0, p, p_r)
            units = [e for e in plan_3way(grid, c) if isinstance(e, Unit3)]
            for pos, u in enumerate(units):
                for s_t in range(grid.n_st):
                    for b in unit_boxes(u, n_vp, grid.n_st, (s_t,)):
                        if b.i0 <= i < b.i1 and b.j0 <= j < b.j1 and b.k0 <= k < b.k1:
                            return rank_of_coords(c, grid), s_t, pos
    raise AssertionError("triple not covered")  # unreachable for a valid plan
