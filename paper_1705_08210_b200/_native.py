"""ctypes binding of libpsim.so (the C ABI in include/psim.h).

The library is REQUIRED: there is no CPU fallback anywhere in this package.
If ``_lib/libpsim.so`` is missing, ``lib()`` raises with the build command.
Status codes map back onto the reference's exception families
(1 -> ConfigError, 2 -> DataError, 3 -> EngineError; cli.py:917-929).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .domain import ConfigError, DataError, EngineError

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libpsim.so"
if os.environ.get("PSIM_LIB"):  # A/B experiments against another in-tree build
    LIB_PATH = Path(os.environ["PSIM_LIB"]).resolve()

F32, F64 = 0, 1

c_i64 = C.c_int64
c_u64 = C.c_uint64
c_vp = C.c_void_p
c_ullp = C.POINTER(C.c_ulonglong)


class Block2(C.Structure):
    """psim_block2_t"""

    _fields_ = [
        ("W", c_vp), ("ldw", c_i64), ("V", c_vp), ("ldv", c_i64), ("n_f", c_i64),
        ("m", c_i64), ("n", c_i64), ("diagonal", C.c_int32),
        ("row_begin", c_i64), ("row_end", c_i64),
        ("s_row", c_vp), ("s_col", c_vp),
        ("g_row", c_i64), ("g_col", c_i64), ("n_v", c_i64),
        ("vals", c_vp), ("acc", c_vp),
    ]


class Box3(C.Structure):
    """psim_box3_t"""

    _fields_ = [
        ("n_f", c_i64), ("n_v", c_i64),
        ("VA", c_vp), ("ldA", c_i64), ("a0", c_i64),
        ("VB", c_vp), ("ldB", c_i64), ("b0", c_i64),
        ("VC", c_vp), ("ldC", c_i64), ("c0", c_i64),
        ("SA", c_vp), ("SB", c_vp), ("SC", c_vp),
        ("NAB", c_vp), ("ldAB", c_i64),
        ("NAC", c_vp), ("ldAC", c_i64),
        ("NBC", c_vp), ("ldBC", c_i64),
        ("i0", c_i64), ("i1", c_i64), ("j0", c_i64), ("j1", c_i64),
        ("k0", c_i64), ("k1", c_i64),
        ("vals", c_vp), ("acc", c_vp),
    ]


class Problem(C.Structure):
    """psim_problem_t"""

    _fields_ = [
        ("arity", C.c_int32), ("dtype", C.c_int32), ("n_f", c_i64), ("n_v", c_i64),
        ("input", C.c_int32), ("bits", C.c_int32), ("seed", c_u64),
        ("block", c_vp), ("ld", c_i64),
    ]


class Grid(C.Structure):
    """psim_grid_t"""

    _fields_ = [("n_pf", C.c_int32), ("n_pv", C.c_int32), ("n_pr", C.c_int32),
                ("n_st", C.c_int32)]


class Piece(C.Structure):
    """psim_piece_t"""

    _fields_ = [("kind", c_i64), ("offset", c_i64), ("count", c_i64), ("v", c_i64 * 8)]


PHASES = 6


class Traffic(C.Structure):
    """psim_traffic_t"""

    _fields_ = [("messages", c_i64 * PHASES), ("elements", c_i64 * PHASES),
                ("nbytes", c_i64 * PHASES)]


class Out(C.Structure):
    """psim_out_t"""

    _fields_ = [
        ("vals", c_vp), ("pieces", C.POINTER(Piece)), ("sums", c_vp),
        ("rank_traffic", C.POINTER(Traffic)),
        ("n_pieces", c_i64), ("n_vals", c_i64), ("checksum", c_u64 * 2),
        ("count", c_i64), ("degenerate", c_i64), ("local_count", c_i64),
        ("elapsed", C.c_double), ("traffic", Traffic),
        ("kernel_seconds", C.c_double), ("kernel_grids", c_i64),
        ("scratch_piece", c_i64), ("scratch_vals", c_vp),
    ]


class Msg(C.Structure):
    """psim_msg_t"""

    _fields_ = [("group", C.c_int32), ("op", C.c_int32), ("peer", C.c_int32),
                ("what", C.c_int32), ("bytes", c_i64), ("slot", c_i64)]


MSG_BLOCK, MSG_SUMS, MSG_TASK, MSG_TABLE, MSG_BOX = range(5)


class Plan(C.Structure):
    """psim_plan_t"""

    _fields_ = [("n_pieces", c_i64), ("n_vals", c_i64), ("workspace_bytes", c_i64)]


INPUT_RANDOM_EXACT, INPUT_ANALYTIC, INPUT_UNIFORM, INPUT_DEVICE, INPUT_HOST = range(5)
RUN_BALANCE_REFERENCE, RUN_VALUES_SCRATCH, RUN_NO_STREAM = 1, 2, 4


# ctypes mirrors of the public structs in psim_abi_layout order (checked
# against the library's sizeof / offsetof by tests/test_capi.py)
def abi_mirrors():
    return [(Block2, "acc"), (Box3, "acc"), (Problem, "ld"), (Grid, "n_st"), (Piece, "v"),
            (Traffic, "nbytes"), (Out, "scratch_vals"), (Plan, "workspace_bytes"),
            (Msg, "slot")]


# name -> (restype, argtypes); every symbol declared in include/psim.h
SIGNATURES = {
    "psim_version": (C.c_int, []),
    "psim_last_error": (C.c_char_p, []),
    "psim_abi_layout": (C.c_int, [C.POINTER(c_i64), C.c_int]),
    "psim_device_info": (C.c_int, [C.POINTER(C.c_int)] * 3),
    "psim_tile_shape": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "psim_gen_random_exact": (
        C.c_int, [C.c_int, c_u64, C.c_int, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "psim_gen_analytic": (C.c_int, [C.c_int, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "psim_gen_uniform": (
        C.c_int, [C.c_int, c_u64, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "psim_check_block": (C.c_int, [C.c_int, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "psim_column_sums": (C.c_int, [C.c_int, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "psim_mgemm": (
        C.c_int,
        [C.c_int, c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, C.c_int, c_vp, c_i64, C.c_int,
         c_vp]),
    "psim_czek2_block": (C.c_int, [C.c_int, C.POINTER(Block2), c_vp]),
    "psim_czek2_tasks": (C.c_int, [C.c_int, C.POINTER(Block2), C.c_int, c_vp]),
    "psim_pack_bits": (C.c_int, [C.c_int, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "psim_sorenson2_block": (C.c_int, [C.c_int, C.POINTER(Block2), c_vp]),
    "psim_czek2_from_numerators": (
        C.c_int,
        [C.c_int, c_vp, c_i64, c_i64, c_i64, c_i64, C.c_int, c_vp, c_vp, c_i64, c_i64, c_i64,
         c_vp, c_vp, c_vp]),
    "psim_fold_add": (C.c_int, [C.c_int, c_vp, c_vp, c_i64, c_vp]),
    "psim_czek2_streamed": (C.c_int, [C.c_int, C.POINTER(Block2), c_vp, c_i64, c_i64, c_vp,
                                      c_vp, c_vp]),
    "psim_stream_stats": (C.c_int, [C.POINTER(C.c_uint64), C.c_int]),
    "psim_stream_error": (C.c_int, [C.POINTER(C.c_uint)]),
    "psim_launch_count": (C.c_int, [C.POINTER(C.c_uint64), C.c_int]),
    "psim_quantize_bytes": (C.c_int, [C.c_int, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "psim_box3_plan": (C.c_int, [C.c_int, C.POINTER(Box3), C.POINTER(c_i64), C.POINTER(c_i64)]),
    "psim_mgemm_bits": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64,
                                  c_vp]),
    "psim_min_columns": (C.c_int, [C.c_int, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "psim_box3_tile": (C.c_int, [C.c_int, C.POINTER(Box3), C.c_int, c_i64, C.POINTER(c_i64),
                                 C.POINTER(c_i64)]),
    "psim_czek3_box": (C.c_int, [C.c_int, C.POINTER(Box3), c_vp]),
    "psim_czek3_box_numerators": (C.c_int, [C.c_int, C.POINTER(Box3), c_vp]),
    "psim_czek3_from_numerators": (
        C.c_int, [C.c_int, C.POINTER(Box3), c_vp, c_i64, c_i64, c_vp, c_vp]),
    "psim_nccl_unique_id": (C.c_int, [c_vp]),
    "psim_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, c_vp, C.POINTER(c_vp)]),
    "psim_ctx_destroy": (C.c_int, [c_vp]),
    "psim_run_plan": (C.c_int, [c_vp, C.POINTER(Problem), C.POINTER(Grid), C.c_int, C.c_int,
                                C.POINTER(Plan)]),
    "psim_run_pieces": (C.c_int, [c_vp, C.POINTER(Problem), C.POINTER(Grid), C.c_int, C.c_int,
                                  C.POINTER(Plan), C.POINTER(Piece), c_i64]),
    "psim_run_comms": (C.c_int, [c_vp, C.POINTER(Problem), C.POINTER(Grid), C.c_int, C.c_int,
                                 C.POINTER(Msg), c_i64, C.POINTER(c_i64)]),
    "psim_run2": (C.c_int, [c_vp, C.POINTER(Problem), C.POINTER(Grid), C.c_int, c_vp, c_i64,
                            C.POINTER(Out), c_vp]),
    "psim_run3": (C.c_int, [c_vp, C.POINTER(Problem), C.POINTER(Grid), C.c_int, C.c_int, c_vp,
                            c_i64, C.POINTER(Out), c_vp]),
    "psim_malloc": (C.c_int, [C.POINTER(c_vp), c_i64, C.c_int]),
    "psim_free": (C.c_int, [c_vp, C.c_int]),
    "psim_memcpy": (C.c_int, [c_vp, c_vp, c_i64]),
    "psim_checksum": (C.c_int, [C.c_int, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "psim_peak_minplus": (
        C.c_int, [C.c_int, C.c_int, c_i64, C.POINTER(C.c_double), C.POINTER(C.c_double), c_vp]),
}

_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Load libpsim.so once; fail loudly when it has not been built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise ImportError(
                        f"libpsim.so not found at {LIB_PATH}; build it with "
                        "`python -m paper_1705_08210_b200.build` (no CPU fallback exists)"
                    )
                handle = C.CDLL(str(LIB_PATH))
                for name, (res, args) in SIGNATURES.items():
                    if os.environ.get("PSIM_LIB") and not hasattr(handle, name):
                        continue  # an older build under A/B test
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib().psim_last_error().decode(errors="replace")
    if status == 1:
        raise ConfigError(msg)
    if status == 2:
        raise DataError(msg)
    raise EngineError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


_shapes: dict = {}


def tile_shape(code: int) -> tuple[int, int]:
    """(rows, cols) of the min-plus CTA tile for a dtype code."""
    if code not in _shapes:
        r, c = C.c_int(), C.c_int()
        call("psim_tile_shape", code, C.byref(r), C.byref(c))
        _shapes[code] = (r.value, c.value)
    return _shapes[code]


def launch_count(reset: bool = False) -> int:
    """Kernel launches libpsim issued in this process (psim_launch_count)."""
    n = C.c_uint64(0)
    call("psim_launch_count", C.byref(n), 1 if reset else 0)
    return n.value
