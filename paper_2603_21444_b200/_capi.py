"""ctypes binding of the drop-in C ABI ``include/spg/capi.h`` (libspgb200.so).

The shared library is built in-tree (``make`` / ``__graft_entry__.build()``);
importing this module never compiles anything. There is no CPU fallback: if the
library or a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPG_LIB_PATH") or os.path.join(_HERE, "lib", "libspgb200.so")
CXX_LIB_PATH = os.path.join(_HERE, "lib", "libspgsim_b200.so")

# Every symbol declared in include/spg/capi.h (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "spg_last_error", "spg_version", "spg_device_count", "spg_init", "spg_finalize", "spg_ctx_stream", "spg_ctx_synchronize",
    "spg_ctx_device", "spg_timing_enable", "spg_timing_reset", "spg_timing_read", "spg_csr_upload",
    "spg_csr_zeros", "spg_csr_shape", "spg_csr_upload_into", "spg_csr_download", "spg_csr_check", "spg_csr_free", "spg_result_checksum",
    "spg_csr_device_ptrs", "spg_spgemm", "spg_spgemm_products", "spg_spgeam", "spg_spgeam_inplace",
    "spg_vconcat", "spg_csr_extract", "spg_csr_copy", "spg_tile_rects", "spg_partition", "spg_reassemble", "spg_spgemm_host", "spg_spgemm_host_to_host", "spg_column_normalize", "spg_prune", "spg_elementwise_power", "spg_mcl_poststep",
    "spg_trident_grid", "spg_trident_spgemm", "spg_summa_spgemm", "spg_oned_spgemm",
    "spg_trident_spgemm_ex", "spg_summa_spgemm_ex",
    "spg_host_register", "spg_host_unregister",
    "spg_csr_ipc_export", "spg_csr_ipc_open", "spg_csr_make_shareable", "spg_trident_rank",
]

STATUS = {
    0: "SPG_OK", 1: "SPG_ERROR", 2: "SPG_DIMENSION_ERROR", 3: "SPG_PARAMETER_ERROR", 4: "SPG_GRID_ERROR",
    5: "SPG_INCOMPLETE_TILE_SET", 6: "SPG_ROUTING_ERROR", 7: "SPG_SCHEDULE_ERROR", 8: "SPG_DEADLOCK_ERROR",
    20: "SPG_CUDA_ERROR", 21: "SPG_OOM", 22: "SPG_NO_DEVICE",
}

IPC_BYTES = 256


class LedgerCell(C.Structure):
    _fields_ = [("messages", C.c_uint64), ("nnz", C.c_uint64), ("bytes", C.c_uint64)]


class Event(C.Structure):
    """spg_event (capi.h): one measured TimelineEvent (engine.hpp:25-38)."""
    _fields_ = [("type", C.c_int32), ("src", C.c_int32), ("dst", C.c_int32), ("round", C.c_int32),
                ("operand", C.c_int32), ("link", C.c_int32), ("t_start", C.c_double), ("t_end", C.c_double),
                ("nnz", C.c_int64), ("bytes", C.c_int64)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built; run `make` (or __graft_entry__.build()) first")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, f64, st = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_int
    P = C.POINTER
    L.spg_last_error.restype = C.c_char_p
    L.spg_version.restype = C.c_char_p
    sig = {
        "spg_device_count": (st, [P(i32)]),
        "spg_init": (st, [i32, P(vp)]),
        "spg_finalize": (st, [vp]),
        "spg_ctx_stream": (vp, [vp]),
        "spg_ctx_synchronize": (st, [vp]),
        "spg_ctx_device": (i32, [vp]),
        "spg_timing_enable": (st, [vp, i32]),
        "spg_timing_reset": (st, [vp]),
        "spg_timing_read": (i32, [vp, C.c_char_p, C.c_size_t, P(i64), P(f64), i32]),
        "spg_csr_upload": (st, [vp, i64, i64, vp, vp, i32, vp, P(vp)]),
        "spg_csr_zeros": (st, [vp, i64, i64, P(vp)]),
        "spg_csr_shape": (st, [vp, P(i64), P(i64), P(i64)]),
        "spg_csr_upload_into": (st, [vp, vp, vp, vp, vp]),
        "spg_csr_download": (st, [vp, vp, vp, vp, i32, vp]),
        "spg_csr_check": (st, [vp, vp]),
        "spg_csr_free": (st, [vp]),
        "spg_csr_device_ptrs": (st, [vp, P(vp), P(vp), P(vp)]),
        "spg_spgemm": (st, [vp, vp, vp, P(vp)]),
        "spg_spgemm_products": (st, [vp, vp, vp, P(i64)]),
        "spg_spgeam": (st, [vp, vp, vp, P(vp)]),
        "spg_spgeam_inplace": (st, [vp, P(vp), vp]),
        "spg_vconcat": (st, [vp, P(vp), i32, P(vp)]),
        "spg_csr_extract": (st, [vp, vp, i64, i64, i64, i64, P(vp)]),
        "spg_result_checksum": (st, [vp, vp, P(i64), P(C.c_uint64)]),
        "spg_tile_rects": (st, [i64, i64, i32, i32, i32, P(i64)]),
        "spg_partition": (st, [P(vp), i32, vp, i32, i32, i32, P(vp)]),
        "spg_reassemble": (st, [vp, P(vp), i32, i64, i64, i32, i32, i32, P(vp)]),
        "spg_csr_copy": (st, [vp, vp, P(vp)]),
        "spg_spgemm_host": (st, [vp, i64, i64, vp, vp, vp, i64, i64, vp, vp, vp, i32, P(vp)]),
        "spg_spgemm_host_to_host": (st, [vp, i64, i64, vp, vp, vp, i64, i64, vp, vp, vp, i32, i32, i64, vp, vp, vp,
                                         P(i64)]),
        "spg_column_normalize": (st, [vp, vp]),
        "spg_prune": (st, [vp, vp, f64, P(vp)]),
        "spg_elementwise_power": (st, [vp, vp, f64]),
        "spg_mcl_poststep": (st, [vp, vp, f64, f64, P(vp)]),
        "spg_trident_grid": (st, [i32, i32, P(i32)]),
        "spg_trident_spgemm": (st, [P(vp), i32, P(vp), P(vp), i32, i32, i32, i32, P(vp), P(LedgerCell), P(f64)]),
        "spg_oned_spgemm": (st, [P(vp), i32, P(vp), P(vp), i32, i32, i32, i32, P(vp), P(LedgerCell), P(f64)]),
        "spg_summa_spgemm": (st, [P(vp), i32, P(vp), P(vp), i32, i32, i32, i32, P(vp), P(LedgerCell), P(f64)]),
        "spg_trident_spgemm_ex": (st, [P(vp), i32, P(vp), P(vp), i32, i32, i32, i32, P(f64), i32, P(vp),
                                       P(LedgerCell), P(f64), P(Event), i32, P(i32), P(f64)]),
        "spg_summa_spgemm_ex": (st, [P(vp), i32, P(vp), P(vp), i32, i32, i32, i32, P(vp), P(LedgerCell), P(f64),
                                     P(Event), i32, P(i32), P(f64)]),
        "spg_host_register": (st, [vp, C.c_size_t]),
        "spg_host_unregister": (st, [vp]),
        "spg_csr_ipc_export": (st, [vp, C.c_char_p]),
        "spg_csr_ipc_open": (st, [vp, C.c_char_p, P(vp)]),
        "spg_csr_make_shareable": (st, [vp, vp, P(vp)]),
        "spg_trident_rank": (st, [vp, i32, i32, i32, P(vp), P(vp), P(vp), P(f64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


class SpgError(RuntimeError):
    """Raised for a non-OK spg_status; ``.status`` is the numeric code and
    ``.kind`` the reference exception class name it maps to."""

    KIND = {1: "Error", 2: "DimensionError", 3: "ParameterError", 4: "GridError", 5: "IncompleteTileSet",
            6: "RoutingError", 7: "ScheduleError", 8: "DeadlockError", 20: "CudaError", 21: "OutOfMemory",
            22: "NoDevice"}

    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.kind = self.KIND.get(status, "Error")


def check(status: int) -> None:
    if status != 0:
        raise SpgError(status, lib().spg_last_error().decode(errors="replace"))
