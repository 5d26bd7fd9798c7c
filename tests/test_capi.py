"""The C-ABI library loads and exports every symbol include/psim.h declares
(CPU: no compute calls, only the host-side planning entry point)."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "psim.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(psim_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1705_08210_b200 import _native

    if not _native.LIB_PATH.exists():
        from paper_1705_08210_b200 import build

        build.build()
    return _native.lib()


def test_header_declares_the_abi():
    names = declared()
    for must in ("psim_czek2_block", "psim_czek3_box", "psim_mgemm", "psim_column_sums",
                 "psim_gen_random_exact", "psim_last_error", "psim_peak_minplus"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    from paper_1705_08210_b200 import _native

    for name in declared():
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, f"{name} lacks a ctypes signature"


def test_version_and_error_string(lib):
    assert lib.psim_version() == 1
    assert isinstance(lib.psim_last_error(), bytes)


def test_bad_dtype_is_config_error(lib):
    from paper_1705_08210_b200 import _native
    from paper_1705_08210_b200.domain import ConfigError

    status = lib.psim_column_sums(7, None, 1, 1, 1, None, None)
    assert status == 1
    with pytest.raises(ConfigError):
        _native.check(status)
    assert b"dtype" in lib.psim_last_error()


def test_box3_plan_counts_match_host_plan(lib):
    from paper_1705_08210_b200 import _native as N
    from paper_1705_08210_b200.plan import Box, box_count

    for box in (Box((0, 0, 0), 0, 60, 0, 60, 0, 60), Box((0, 1, 1), 0, 10, 30, 60, 30, 60),
                Box((0, 1, 2), 5, 17, 20, 40, 40, 60), Box((0, 0, 0), 0, 300, 0, 300, 250, 300)):
        b = N.Box3(i0=box.i0, i1=box.i1, j0=box.j0, j1=box.j1, k0=box.k0, k1=box.k1)
        n_out, n_tiles = C.c_int64(), C.c_int64()
        assert lib.psim_box3_plan(1, C.byref(b), C.byref(n_out), C.byref(n_tiles)) == 0
        assert n_out.value == box_count(box)
        assert n_tiles.value > 0


def _box_tiles(lib, code, box, packed):
    """Every CTA tile of one grid of a box, decoded by the kernels' own code."""
    from paper_1705_08210_b200 import _native as N

    b = N.Box3(i0=box.i0, i1=box.i1, j0=box.j0, j1=box.j1, k0=box.k0, k1=box.k1)
    out, n = (C.c_int64 * 11)(), C.c_int64()
    tiles = []
    t = 0
    while True:
        st = lib.psim_box3_tile(code, C.byref(b), packed, t, out, C.byref(n))
        if t >= n.value:
            assert st == 1  # outside the grid: ConfigError
            break
        assert st == 0
        tiles.append(tuple(out))
        t += 1
    return tiles


@pytest.mark.parametrize("code", [0, 1])
def test_box3_tiles_cover_every_triple_once(lib, code):
    """The single-pivot and two-segment grids of every box layout (PAIR
    diagonal, FLAT_COLS faces, FLAT_ROWS faces, volumes, staged / chunked
    boxes, plain) cover each (i < j < k) of the box exactly once, within the
    CTA tile shape (box3_plan.cuh)."""
    import numpy as np

    from paper_1705_08210_b200 import _native as N
    from paper_1705_08210_b200.plan import Box, box_count

    bm, bn = N.tile_shape(code)
    boxes = [
        Box((0, 0, 0), 0, 700, 0, 700, 0, 700),          # diagonal (PAIR)
        Box((0, 0, 0), 0, 700, 300, 420, 0, 700),        # pivot chunk of a diagonal
        Box((0, 1, 1), 0, 300, 300, 700, 300, 700),      # face, rows fixed (FLAT_COLS)
        Box((0, 1, 1), 50, 100, 300, 700, 300, 700),     # face sixth
        Box((0, 0, 1), 0, 400, 0, 400, 400, 700),        # face, columns fixed (FLAT_ROWS)
        Box((0, 0, 1), 0, 400, 0, 400, 650, 700),        # face sixth of the upper block
        Box((0, 1, 2), 0, 250, 250, 500, 500, 750),      # volume
        Box((0, 1, 2), 0, 130, 250, 390, 500, 529),      # volume slice, narrow K
        Box((0, 0, 0), 0, 500, 0, 500, 333, 500),        # staged diagonal (plain)
        Box((0, 1, 1), 0, 40, 300, 700, 300, 700),       # rows < one tile
        Box((0, 1, 1), 0, 300, 300, 700, 640, 700),      # K narrower than a tile
    ]
    for box in boxes:
        nI, nJ, nK = box.i1 - box.i0, box.j1 - box.j0, box.k1 - box.k0
        seen = np.zeros((nI, nJ, nK), dtype=np.int32)
        for packed in (0, 1):
            for (p0, p1, r0, r1, c0, c1, nr0, nr1, nc0, nc1, side) in _box_tiles(lib, code, box,
                                                                                   packed):
                assert 0 < nr0 + nr1 <= bm and 0 < nc0 + nc1 <= bn
                assert packed or (nr1 == 0 and nc1 == 0)
                ii = np.r_[r0:r0 + nr0, r1:r1 + nr1]
                kk = np.r_[c0:c0 + nc0, c1:c1 + nc1]
                rseg = np.r_[np.zeros(nr0, int), np.ones(nr1, int)]
                cseg = np.r_[np.zeros(nc0, int), np.ones(nc1, int)]
                seg = cseg[None, :] if side else rseg[:, None]
                jj = np.broadcast_to(np.where(seg == 1, p1, p0), (len(ii), len(kk)))
                I = np.broadcast_to(ii[:, None], jj.shape)
                K = np.broadcast_to(kk[None, :], jj.shape)
                assert ((box.i0 <= I) & (I < np.minimum(box.i1, jj))).all(), box
                assert ((np.maximum(box.k0, jj + 1) <= K) & (K < box.k1)).all(), box
                assert ((box.j0 <= jj) & (jj < box.j1)).all(), box
                seen[I - box.i0, jj - box.j0, K - box.k0] += 1  # cells of a tile are distinct
        assert seen.max() == 1, box
        assert int(seen.sum()) == box_count(box), box


def _layout(lib):
    from paper_1705_08210_b200 import _native

    buf = (C.c_int64 * 18)()
    assert "psim_abi_layout" in _native.SIGNATURES
    n = lib.psim_abi_layout(buf, 9)
    assert n == 9
    return [(buf[2 * k], buf[2 * k + 1]) for k in range(9)]


def test_ctypes_mirrors_match_the_c_structs(lib):
    """Every ctypes restatement of a public struct (the package's _native and
    the torch-free reference-side binding) has the C sizeof and the C offset
    of its last member: a field added on one side only fails here, not as
    silent memory corruption on the GPU box."""
    from paper_1705_08210_b200 import _native

    want = _layout(lib)
    for (cls, last), (size, off) in zip(_native.abi_mirrors(), want):
        assert C.sizeof(cls) == size, (cls.__name__, C.sizeof(cls), size)
        assert getattr(cls, last).offset == off, (cls.__name__, last)
    import sys

    sys.path.insert(0, str(ROOT / "integration"))
    import propsim_b200 as B

    order = {"_Problem": 2, "_Grid": 3, "_Piece": 4, "_Traffic": 5, "_Out": 6, "_Plan": 7}
    last = {"_Problem": "ld", "_Grid": "n_st", "_Piece": "v", "_Traffic": "nbytes",
            "_Out": "scratch_vals", "_Plan": "workspace_bytes"}
    for name, k in order.items():
        cls = getattr(B, name)
        assert C.sizeof(cls) == want[k][0], name
        assert getattr(cls, last[name]).offset == want[k][1], name
