"""ctypes binding of include/fw_capi.h and the error mapping of errors.hpp."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libfw_b200.so"


def library_path() -> str:
    # FW_LIBRARY: an alternative build of the same library (A/B timing of kernel variants)
    return os.environ.get("FW_LIBRARY") or os.path.join(_HERE, "lib", LIB_NAME)


# ---- errors: one class per fwave::Error subtype the path raises (errors.hpp:10-60)


class Error(RuntimeError):
    code = -1


class GridMismatch(Error):
    code = 2


class NegativeM(Error):
    code = 3


class OrderOutOfRange(Error):
    code = 4


class DeviationTooLarge(Error):
    code = 5


class GammaOutOfRange(Error):
    code = 6


class BlowupDetected(Error):
    code = 7


class OddSize(Error):
    code = 8


class EmptyInterval(Error):
    code = 9


class DimOutOfRange(Error):
    code = 10


class MemoryBudgetExceeded(Error):
    code = 17


class NotConstantOrder(Error):
    code = 18


class DimUnsupported(Error):
    code = 19


class NonpositiveFrequency(Error):
    code = 20


class OutOfMemory(Error):
    code = 11


class CudaError(Error):
    code = 12


class Unsupported(Error):
    code = 13


class PicardDiverged(Error):
    code = 15


class CgStagnated(Error):
    code = 16


class ArgumentError(Error, ValueError):
    code = 1


_BY_CODE = {c.code: c for c in (ArgumentError, GridMismatch, NegativeM, OrderOutOfRange,
                                 DeviationTooLarge, GammaOutOfRange, BlowupDetected, OddSize,
                                 EmptyInterval, DimOutOfRange, OutOfMemory, CudaError, Unsupported,
                                 PicardDiverged, CgStagnated, MemoryBudgetExceeded, NotConstantOrder,
                                 DimUnsupported, NonpositiveFrequency)}


class OpInfo(C.Structure):
    _fields_ = [("dim", C.c_int), ("J", C.c_int * 3), ("M", C.c_int), ("constant_order", C.c_int),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("s0", C.c_double),
                ("smin", C.c_double), ("smax", C.c_double), ("N", C.c_size_t),
                ("N_half", C.c_size_t), ("device_bytes", C.c_size_t)]


_lib = None

_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def load_library():
    """Load lib/libfw_b200.so (built by __graft_entry__.build()).  Raises if absent:
    there is no CPU fallback for any compute entry point."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    lib.fw_last_error.restype = C.c_char_p
    lib.fw_version.restype = C.c_int
    lib.fw_ctx_create.argtypes = [C.c_int, C.POINTER(_vp)]
    lib.fw_ctx_destroy.argtypes = [_vp]
    lib.fw_ctx_destroy.restype = None
    lib.fw_ctx_sync.argtypes = [_vp]
    lib.fw_ctx_stream.argtypes = [_vp]
    lib.fw_ctx_stream.restype = _vp
    lib.fw_ctx_launches.argtypes = [_vp]
    lib.fw_ctx_launches.restype = C.c_longlong
    lib.fw_op_create.argtypes = [_vp, C.c_int, _ip, _dp, _dp, _dp, _dp, C.c_int, C.POINTER(_vp)]
    lib.fw_op_create_from_tables.argtypes = [_vp, C.c_int, _ip, _dp, _dp, C.c_int, C.c_double,
                                             C.c_int, _dp, C.POINTER(_dp), C.POINTER(_dp),
                                             C.POINTER(_vp)]
    lib.fw_op_destroy.argtypes = [_vp]
    lib.fw_op_destroy.restype = None
    lib.fw_op_info.argtypes = [_vp, C.POINTER(OpInfo)]
    lib.fw_op_path.argtypes = [_vp]
    lib.fw_ricker_initial.argtypes = [C.c_int, _ip, _dp, _dp, C.c_double, _dp, _dp]
    lib.fw_grid_dft.argtypes = [_vp, C.c_int, _ip, _dp, C.c_int]
    lib.fw_dense_create.argtypes = [_vp, C.c_int, _ip, _dp, _dp, _dp, C.c_ulonglong, C.POINTER(_vp)]
    lib.fw_dense_destroy.argtypes = [_vp]
    lib.fw_dense_destroy.restype = None
    lib.fw_dense_apply.argtypes = [_vp, _dp, _dp]
    lib.fw_dense_entries.argtypes = [_vp, _dp]
    lib.fw_apply_toeplitz.argtypes = [_vp, C.c_int, _ip, _dp, _dp, _dp, _dp, _dp]
    lib.fw_truncation_indicator.argtypes = [C.c_int, C.c_double, C.c_double, _dp]
    lib.fw_ctx_device.argtypes = [_vp]
    lib.fw_nccl_unique_id.argtypes = [C.c_char_p]
    lib.fw_slab_seis_create.argtypes = [_vp, C.c_char_p, C.c_int, C.c_int, _ip, _dp, _dp, _dp, _dp, C.c_double,
                                        C.c_int, _dp, _dp, C.c_double, C.c_double, C.POINTER(_vp)]
    lib.fw_slab_seis_destroy.argtypes = [_vp]
    lib.fw_slab_seis_destroy.restype = None
    lib.fw_slab_seis_step.argtypes = [_vp, C.c_int]
    lib.fw_slab_seis_get.argtypes = [_vp, _dp, _dp, _dp, C.POINTER(C.c_long)]
    lib.fw_slab_seis_info.argtypes = [_vp, C.POINTER(C.c_size_t), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.fw_op_create_slab.argtypes = [_vp, _ip, _dp, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]
    lib.fw_ipc_alloc.argtypes = [_vp, C.c_size_t, C.POINTER(_vp)]
    lib.fw_ipc_free.argtypes = [_vp, _vp]
    lib.fw_stage_seis_update_peers.argtypes = ([_vp, C.c_longlong, C.c_double] + [_vp] * 10
                                               + [C.c_double, C.c_int, _vp, C.c_int, _vp])
    lib.fw_grid_dft_device.argtypes = [_vp, C.c_int, _ip, _vp, C.c_int]
    lib.fw_grid_forward.argtypes = [_vp, C.c_int, _ip, _dp, _dp]
    lib.fw_grid_inverse.argtypes = [_vp, C.c_int, _ip, _dp, _dp, _dp]
    lib.fw_apply_constant_order.argtypes = [_vp, C.c_int, _ip, _dp, _dp, _dp, C.c_double, _dp, _dp]
    lib.fw_apply_constant_order_spectrum.argtypes = [_vp, C.c_int, _ip, _dp, _dp, _dp, C.c_double, _dp]
    lib.fw_apply.argtypes = [_vp, _dp, _dp, C.c_int, _dp]
    lib.fw_apply_device.argtypes = [_vp, _vp, _vp, C.c_int, _vp]
    lib.fw_apply_batch_device.argtypes = [C.POINTER(_vp), C.c_int, C.POINTER(_vp), C.POINTER(_vp)]
    lib.fw_seis_create.argtypes = [_vp, C.c_int, _ip, _dp, _dp, _dp, _dp, C.c_double, C.c_int,
                                   _dp, _dp, C.c_double, C.c_double, C.POINTER(_vp)]
    lib.fw_seis_destroy.argtypes = [_vp]
    lib.fw_seis_destroy.restype = None
    lib.fw_seis_step.argtypes = [_vp, C.c_int]
    lib.fw_seis_enqueue.argtypes = [_vp, C.c_int]
    lib.fw_seis_get.argtypes = [_vp, _dp, _dp, _dp, C.POINTER(C.c_long)]
    lib.fw_seis_set_current.argtypes = [_vp, _dp]
    lib.fw_seis_step_io.argtypes = [_vp, _dp, C.c_int, _dp]
    lib.fw_seis_step_io_async.argtypes = [_vp, _dp, C.c_int, _dp]
    lib.fw_seis_wait.argtypes = [_vp]
    lib.fw_seis_current_device.argtypes = [_vp]
    lib.fw_seis_current_device.restype = _vp
    lib.fw_seis_ops.argtypes = [_vp, C.POINTER(_vp), C.POINTER(_vp)]
    lib.fw_seis_medium.argtypes = [_vp, _dp, _dp, _dp]
    lib.fw_tsfp2_create.argtypes = [_vp, C.c_int, _ip, _dp, _dp, _dp, C.c_int, C.c_double, C.c_int,
                                    _dp, _dp, C.c_double, C.c_double, C.POINTER(_vp)]
    lib.fw_tsfp2_destroy.argtypes = [_vp]
    lib.fw_tsfp2_destroy.restype = None
    lib.fw_tsfp2_step.argtypes = [_vp, C.c_int]
    lib.fw_tsfp2_get.argtypes = [_vp, _dp, _dp, C.POINTER(C.c_long)]
    lib.fw_wave_create.argtypes = [_vp, C.c_int, C.c_int, _ip, _dp, _dp, _dp, C.c_int, C.c_double, C.c_int, _dp,
                                   _dp, C.c_double, C.c_double, C.c_int, C.c_double, C.c_int, C.c_double,
                                   C.POINTER(_vp)]
    lib.fw_wave_destroy.argtypes = [_vp]
    lib.fw_wave_destroy.restype = None
    lib.fw_wave_step.argtypes = [_vp, C.c_int]
    lib.fw_wave_get.argtypes = [_vp, _dp, _dp, C.POINTER(C.c_long), C.POINTER(C.c_long)]
    lib.fw_rfftn.argtypes = [_vp, C.c_int, _ip, _dp, _dp]
    lib.fw_irfftn.argtypes = [_vp, C.c_int, _ip, _dp, _dp]
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load_library().fw_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, Error)(msg)


EXPORTED_SYMBOLS = [
    "fw_last_error", "fw_version", "fw_ctx_create", "fw_ctx_destroy", "fw_ctx_sync", "fw_ctx_stream",
    "fw_ctx_launches", "fw_ctx_trace", "fw_op_create", "fw_op_create_from_tables", "fw_op_destroy", "fw_op_info",
    "fw_apply", "fw_apply_device", "fw_apply_batch_device", "fw_stage_c2c_scatter", "fw_ipc_handle", "fw_ipc_open", "fw_ipc_close",
    "fw_medium_coefficients", "fw_stage_seis_start", "fw_stage_seis_update", "fw_seis_create", "fw_seis_destroy",
    "fw_seis_step", "fw_seis_enqueue", "fw_seis_get", "fw_seis_set_current", "fw_seis_step_io",
    "fw_seis_step_io_async", "fw_seis_wait",
    "fw_seis_current_device", "fw_seis_ops", "fw_seis_medium", "fw_tsfp2_create",
    "fw_tsfp2_destroy", "fw_tsfp2_step", "fw_tsfp2_get", "fw_wave_create", "fw_wave_destroy", "fw_wave_step",
    "fw_wave_get", "fw_rfftn", "fw_irfftn", "fw_op_path", "fw_ricker_initial", "fw_grid_dft", "fw_grid_dft_device",
    "fw_grid_forward", "fw_grid_inverse", "fw_apply_constant_order", "fw_apply_constant_order_spectrum",
    "fw_dense_create", "fw_dense_destroy", "fw_dense_apply", "fw_dense_entries", "fw_apply_toeplitz",
    "fw_truncation_indicator", "fw_ctx_device", "fw_nccl_unique_id", "fw_slab_seis_create", "fw_slab_seis_destroy",
    "fw_slab_seis_step", "fw_slab_seis_get", "fw_slab_seis_info", "fw_op_create_slab", "fw_stage_seis_update_peers", "fw_ipc_alloc", "fw_ipc_free",
]
