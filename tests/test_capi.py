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
