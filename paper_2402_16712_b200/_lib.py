"""ctypes binding of the C ABI in include/l1b200.h (libl1b200.so, built in-tree).

There is deliberately no fallback: if the shared library is missing or does
not export the ABI, importing the device path raises.  The library is built
by ``paper_2402_16712_b200.build.build()`` (nvcc, sm_100a) and is loaded from
the package directory so the GPU box uses the in-tree artefact.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("L1B200_LIB") or os.path.join(_HERE, "csrc", "libl1b200.so")

# Every symbol include/l1b200.h declares (tests check the export list).
ABI_SYMBOLS = (
    "l1b_status_string",
    "l1b_version",
    "l1b_workspace_bytes",
    "l1b_prepare",
    "l1b_fit_pivots",
    "l1b_fit_pivot_list",
    "l1b_bound_pivots",
    "l1b_bound_pivot_sums",
    "l1b_bound_pivot_list",
    "l1b_argmin",
    "l1b_residual_exact",
    "l1b_deflate",
    "l1b_absmax",
    "l1b_prepared_absmax",
    "l1b_host_copy",
    "l1b_upload",
    "l1b_selftest_divide",
    "l1b_kernel_launches",
    "l1b_dfma_probe",
    "l1b_fit_stats",
    "l1b_set_probe",
    "l1b_straggler_records",
    "l1b_bound_columns",
    "l1b_fit_pivot_list_seeded",
    "l1b_bound_pivot_list_continue",
    "l1b_bound_pivots_multi",
    "l1b_pivot_breakpoints",
    "l1b_pivot_tableau",
    "l1b_certify_columns",
    "l1b_bound_entries",
    "l1b_fit_entries_seeded",
    "l1b_residual_exact_batch",
    "l1b_fit_line",
    "l1b_fit_lines",
    "l1b_csv_read",
    "l1b_csv_free",
    "l1b_merge_path",
    "l1b_merge_path_device",
    "l1b_snap_events",
    "l1b_set_steer",
    "l1b_brute_force_columns",
    "l1b_last_bound_ms",
    "l1b_atoms_probe",
)

# double (*)(double top, void* ctx): the sharded fit's upper-bound exchange hook
UB_EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_double, ctypes.c_void_p)
UB_EXCHANGE_VEC_FN = ctypes.CFUNCTYPE(None, ctypes.POINTER(ctypes.c_double), ctypes.c_int32, ctypes.c_void_p)

L1B_OK = 0
L1B_EINVAL = -1
L1B_ECUDA = -2
L1B_ENOMEM = -3
L1B_EFALLBACK = -5
L1B_EINTERNAL = -4

_lib = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_sz = ctypes.c_size_t


class L1BError(RuntimeError):
    """A CUDA-side failure reported by the C ABI."""


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name in ABI_SYMBOLS:
        if not hasattr(lib, name):
            raise ImportError(f"{LIB_PATH} does not export {name}")
    lib.l1b_status_string.restype = ctypes.c_char_p
    lib.l1b_status_string.argtypes = [ctypes.c_int]
    lib.l1b_version.restype = ctypes.c_int
    lib.l1b_version.argtypes = []
    lib.l1b_workspace_bytes.restype = _sz
    lib.l1b_workspace_bytes.argtypes = [_i64, _i64, _i32, _i64]
    lib.l1b_prepare.restype = ctypes.c_int
    lib.l1b_prepare.argtypes = [_vp, _i64, _i64, _vp, _sz, _vp]
    lib.l1b_fit_pivots.restype = ctypes.c_int
    lib.l1b_fit_pivots.argtypes = [_vp, _i64, _i64, ctypes.POINTER(ctypes.c_double), _i32,
                                   _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    lib.l1b_fit_pivot_list.restype = ctypes.c_int
    lib.l1b_fit_pivot_list.argtypes = [_vp, _i64, _i64, ctypes.POINTER(ctypes.c_double), _i32,
                                       ctypes.POINTER(ctypes.c_int64), _i64, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    lib.l1b_bound_pivots.restype = ctypes.c_int
    lib.l1b_bound_pivots.argtypes = [_vp, _i64, _i64, ctypes.c_double, _i64, _i64, _i64, _vp, _vp, _vp, _sz, _vp]
    lib.l1b_bound_pivot_sums.restype = ctypes.c_int
    lib.l1b_bound_pivot_sums.argtypes = [_vp, _i64, _i64, ctypes.c_double, _i64, _i64, _i64, _i32, _vp, _vp, _vp,
                                         _sz, _vp]
    lib.l1b_bound_pivot_list.restype = ctypes.c_int
    lib.l1b_bound_pivot_list.argtypes = [_vp, _i64, _i64, ctypes.c_double, ctypes.POINTER(ctypes.c_int64), _i64,
                                         _i32, _vp, _vp, _vp, _sz, _vp]
    lib.l1b_argmin.restype = ctypes.c_int
    lib.l1b_argmin.argtypes = [_vp, _i32, _i64, _vp, _vp, _vp]
    lib.l1b_residual_exact.restype = ctypes.c_int
    lib.l1b_residual_exact.argtypes = [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _sz, _vp]
    lib.l1b_deflate.restype = ctypes.c_int
    lib.l1b_deflate.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp]
    lib.l1b_absmax.restype = ctypes.c_int
    lib.l1b_absmax.argtypes = [_vp, _i64, _i64, _vp, _vp]
    lib.l1b_host_copy.restype = ctypes.c_int
    lib.l1b_host_copy.argtypes = [_vp, _vp, ctypes.c_size_t, ctypes.c_int32]
    lib.l1b_upload.restype = ctypes.c_int
    lib.l1b_upload.argtypes = [_vp, _vp, ctypes.c_size_t, _vp, _vp, ctypes.c_size_t, ctypes.c_int32, _vp]
    lib.l1b_prepared_absmax.restype = ctypes.c_int
    lib.l1b_prepared_absmax.argtypes = [_vp, _i64, _i64, ctypes.c_size_t, _vp, _vp]
    lib.l1b_selftest_divide.restype = ctypes.c_int
    lib.l1b_selftest_divide.argtypes = [ctypes.c_uint64, _i64, _vp, _vp]
    lib.l1b_kernel_launches.restype = ctypes.c_uint64
    lib.l1b_kernel_launches.argtypes = []
    lib.l1b_dfma_probe.restype = ctypes.c_int
    lib.l1b_dfma_probe.argtypes = [_i64, _i32, _i32, _vp, _vp]
    lib.l1b_fit_stats.restype = ctypes.c_int
    lib.l1b_fit_stats.argtypes = [_i64, _i64, _i64, _vp, _sz, _vp, _vp]
    lib.l1b_straggler_records.restype = ctypes.c_int
    lib.l1b_straggler_records.argtypes = [_i64, _i64, _i64, _vp, _sz, _vp, _i64, _vp]
    lib.l1b_bound_columns.restype = ctypes.c_int
    lib.l1b_bound_columns.argtypes = [_i64, _i64, _i64, _vp, _sz, _vp, _vp, _vp]
    lib.l1b_fit_pivot_list_seeded.restype = ctypes.c_int
    lib.l1b_fit_pivot_list_seeded.argtypes = [_vp, _i64, _i64, ctypes.c_double, _vp, _i64, _vp, _i64, _vp, _vp,
                                              _vp, _vp, _vp, _sz, _vp]
    lib.l1b_bound_pivot_list_continue.restype = ctypes.c_int
    lib.l1b_bound_pivot_list_continue.argtypes = [_vp, _i64, _i64, ctypes.c_double, _vp, _i64, _vp, _i64, _vp,
                                                  _vp, _vp, _sz, _vp]
    lib.l1b_bound_pivots_multi.restype = ctypes.c_int
    lib.l1b_bound_pivots_multi.argtypes = [_vp, _i64, _i64, _vp, ctypes.c_int32, _i64, _i64, _i64, _vp, _vp, _vp,
                                           _vp, _sz, _vp]
    lib.l1b_pivot_tableau.restype = ctypes.c_int
    lib.l1b_pivot_tableau.argtypes = [_vp, _i64, _i64, _i64, _i64, ctypes.POINTER(ctypes.c_int64), _vp, _vp, _vp, _vp,
                                      _i64, _vp, _sz, _vp]
    lib.l1b_pivot_breakpoints.restype = ctypes.c_int
    lib.l1b_pivot_breakpoints.argtypes = [_vp, _i64, _i64, _i64, ctypes.POINTER(ctypes.c_int64), _vp, _vp, _vp, _i64,
                                          _vp, _sz, _vp]
    lib.l1b_certify_columns.restype = ctypes.c_int
    lib.l1b_certify_columns.argtypes = [_vp, _i64, _i64, _i64, _vp, ctypes.c_double, _vp, _vp, _sz, _vp]
    lib.l1b_bound_entries.restype = ctypes.c_int
    lib.l1b_bound_entries.argtypes = [_vp, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp]
    lib.l1b_fit_entries_seeded.restype = ctypes.c_int
    lib.l1b_fit_entries_seeded.argtypes = [_vp, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _sz,
                                           _vp]
    lib.l1b_residual_exact_batch.restype = ctypes.c_int
    lib.l1b_residual_exact_batch.argtypes = [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _sz, _vp]
    lib.l1b_fit_line.restype = ctypes.c_int
    lib.l1b_fit_line.argtypes = [_vp, _i64, _i64, ctypes.c_double, _i64, _i64, _i64, ctypes.c_int32, UB_EXCHANGE_FN,
                                 _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    lib.l1b_fit_lines.restype = ctypes.c_int
    lib.l1b_fit_lines.argtypes = [_vp, _i64, _i64, _vp, _i32, _i64, _i64, _i64, UB_EXCHANGE_VEC_FN, _vp, _vp, _vp, _sz,
                                  _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    lib.l1b_csv_read.restype = ctypes.c_int
    lib.l1b_csv_read.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32,
                                 ctypes.POINTER(ctypes.POINTER(ctypes.c_double)), ctypes.POINTER(ctypes.c_int64),
                                 ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_char_p)]
    lib.l1b_csv_free.restype = None
    lib.l1b_csv_free.argtypes = [_vp]
    lib.l1b_merge_path.restype = ctypes.c_int
    lib.l1b_merge_path.argtypes = [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _i64,
                                   _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    lib.l1b_merge_path_device.restype = ctypes.c_int
    lib.l1b_merge_path_device.argtypes = [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp,
                                          ctypes.POINTER(ctypes.c_void_p), _vp, _vp, _sz, _vp]
    lib.l1b_set_steer.restype = ctypes.c_int
    lib.l1b_set_steer.argtypes = [_vp, _i32]
    lib.l1b_snap_events.restype = ctypes.c_int
    lib.l1b_snap_events.argtypes = [_vp, _i64, _vp, _i64, ctypes.c_double, _vp, _vp]
    lib.l1b_brute_force_columns.restype = ctypes.c_int
    lib.l1b_brute_force_columns.argtypes = [_vp, _i64, _i64, _i64, ctypes.c_double, _vp, _vp, _vp]
    lib.l1b_last_bound_ms.restype = ctypes.c_int
    lib.l1b_last_bound_ms.argtypes = [ctypes.POINTER(ctypes.c_float)]
    lib.l1b_atoms_probe.restype = ctypes.c_int
    lib.l1b_atoms_probe.argtypes = [_i64, ctypes.c_int32, ctypes.c_int32, _vp, _vp]
    lib.l1b_set_probe.restype = ctypes.c_int
    lib.l1b_set_probe.argtypes = [_vp]
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    """Map a C ABI status to the reference's exception types."""
    if status == L1B_OK:
        return
    msg = load().l1b_status_string(status).decode()
    if status == L1B_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise L1BError(f"{what}: {msg} ({status})")
