"""ctypes binding of libcbg.so (the C ABI declared in include/cbg.h).

The product path is the in-tree ``libcbg.so`` (CUDA kernels for sm_100a + the
C++ runtime). There is no fallback: if the library is missing, importing this
module raises, and every compute call fails loudly when no B200 is visible.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CBG_LIB selects an instrumented build (e.g. libcbg_trace.so) for debugging only
LIB_PATH = os.path.join(_HERE, os.environ.get("CBG_LIB", "libcbg.so"))

# ---- status codes / enums (include/cbg.h) -----------------------------------
OK, ERR_INVALID_INPUT, ERR_CONFIG, ERR_CUDA, ERR_OOM, ERR_UNSUPPORTED = range(6)
LAYER_CONV, LAYER_ACT, LAYER_POOL, LAYER_ADD, LAYER_CONCAT, LAYER_UPSAMPLE = range(6)
POLICY_DETECT, POLICY_PROPAGATE, POLICY_REUSE1X1 = range(3)
MODE_FEEDFORWARD, MODE_CLOSEDLOOP = range(2)
FWD_FORCE_FULL = 1
FWD_RECORD_WORST_CASE = 2
FWD_BROADCAST_INPUT = 8
FWD_INPUT_ON_DEVICE = 4


class ConvSpecC(C.Structure):
    _fields_ = [
        ("in_channels", C.c_int), ("out_channels", C.c_int),
        ("kernel_h", C.c_int), ("kernel_w", C.c_int),
        ("stride", C.c_int), ("padding", C.c_int),
        ("out_h", C.c_int), ("out_w", C.c_int),
        ("weights", C.POINTER(C.c_float)), ("bias", C.POINTER(C.c_float)),
    ]


class LayerDescC(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("name", C.c_char_p),
        ("n_from", C.c_int), ("from_", C.POINTER(C.c_char_p)),
        ("conv", ConvSpecC), ("fuse_relu", C.c_int),
        ("pool_size", C.c_int), ("pool_stride", C.c_int),
        ("pool_out_h", C.c_int), ("pool_out_w", C.c_int),
        ("act_slope", C.c_float), ("upsample", C.c_int),
    ]


class NetworkSpecC(C.Structure):
    _fields_ = [
        ("in_channels", C.c_int), ("in_height", C.c_int), ("in_width", C.c_int),
        ("n_layers", C.c_int), ("layers", C.POINTER(LayerDescC)),
    ]


class SyntheticConfigC(C.Structure):
    _fields_ = [
        ("height", C.c_int), ("width", C.c_int), ("channels", C.c_int), ("n_frames", C.c_int),
        ("n_objects", C.c_int), ("object_size", C.c_int),
        ("velocity_y", C.c_int), ("velocity_x", C.c_int),
        ("noise_std", C.c_float), ("seed", C.c_uint32),
    ]


class NodeInfoC(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("name", C.c_char * 64),
        ("n_inputs", C.c_int), ("inputs", C.c_int * 8),
        ("out_channels", C.c_int), ("out_height", C.c_int), ("out_width", C.c_int),
        ("in_channels", C.c_int), ("in_height", C.c_int), ("in_width", C.c_int),
        ("policy", C.c_int), ("fuse_relu", C.c_int), ("tau", C.c_float),
        ("ops_per_pixel", C.c_int64),
    ]


class LayerStatsC(C.Structure):
    _fields_ = [
        ("changed_px", C.c_int64), ("total_px", C.c_int64),
        ("eff_ops", C.c_int64), ("propagated_px", C.c_int64),
    ]


class EvalSequenceC(C.Structure):
    _fields_ = [("n_frames", C.c_int), ("frames", C.c_void_p), ("references", C.c_void_p), ("ref_channels", C.c_int)]


class CalibConfigC(C.Structure):
    _fields_ = [
        ("initial_tau", C.c_double), ("growth_factor", C.c_double), ("per_layer_budget", C.c_double),
        ("budget_overrides", C.c_void_p), ("n_budget_overrides", C.c_int),
        ("metric", C.c_int), ("aggregation", C.c_int), ("max_steps", C.c_int),
    ]


class CalibTracePointC(C.Structure):
    _fields_ = [("layer", C.c_int), ("tau", C.c_double), ("loss", C.c_double)]


class TradeoffRowC(C.Structure):
    _fields_ = [("factor", C.c_double), ("loss", C.c_double), ("total_eff_ops", C.c_int64), ("wall_ns", C.c_int64)]


# every symbol include/cbg.h declares: (name, restype, argtypes)
_vp = C.c_void_p
_P = C.POINTER
SIGNATURES = {
    "cbg_last_error": (C.c_char_p, []),
    "cbg_abi_version": (C.c_int, []),
    "cbg_device_available": (C.c_int, []),
    "cbg_ctx_create": (C.c_int, [C.c_int, _P(_vp)]),
    "cbg_ctx_destroy": (None, [_vp]),
    "cbg_ctx_sync": (C.c_int, [_vp]),
    "cbg_ctx_stream": (_vp, [_vp]),
    "cbg_ctx_copy_stream": (_vp, [_vp]),
    "cbg_gen_synthetic": (C.c_int, [_P(SyntheticConfigC), _vp, _vp]),
    "cbg_fill_random_weights": (C.c_int, [_P(NetworkSpecC), C.c_uint32, _P(_vp), _P(_vp)]),
    "cbg_net_validate": (C.c_int, [_P(NetworkSpecC), _vp, C.c_int, _vp, C.c_int]),
    "cbg_net_create": (C.c_int, [_vp, _P(NetworkSpecC), _vp, C.c_int, _vp, C.c_int, C.c_int, _P(_vp)]),
    "cbg_net_destroy": (None, [_vp]),
    "cbg_net_clone": (C.c_int, [_vp, _P(_vp)]),
    "cbg_net_node_count": (C.c_int, [_vp, _P(C.c_int)]),
    "cbg_net_stream_count": (C.c_int, [_vp, _P(C.c_int)]),
    "cbg_net_node_info": (C.c_int, [_vp, C.c_int, _P(NodeInfoC)]),
    "cbg_net_forward": (C.c_int, [_vp, _vp, C.c_uint]),
    "cbg_net_forward_u8": (C.c_int, [_vp, _vp, C.c_uint]),
    "cbg_net_reset": (C.c_int, [_vp, C.c_int]),
    "cbg_net_set_thresholds": (C.c_int, [_vp, _vp, C.c_int]),
    "cbg_net_set_stream_thresholds": (C.c_int, [_vp, C.c_int, _vp, C.c_int]),
    "cbg_select_thresholds": (C.c_int, [_vp, _P(EvalSequenceC), C.c_int, _P(CalibConfigC), _vp, _vp,
                                        _P(CalibTracePointC), C.c_int, _P(C.c_int)]),
    "cbg_sweep_threshold_factor": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int, _P(EvalSequenceC), C.c_int, C.c_int,
                                             _P(TradeoffRowC)]),
    "cbg_net_thresholds": (C.c_int, [_vp, _vp, C.c_int]),
    "cbg_net_set_dense": (C.c_int, [_vp, C.c_int]),
    "cbg_net_read_output": (C.c_int, [_vp, C.c_int, C.c_int, _vp]),
    "cbg_net_read_state": (C.c_int, [_vp, C.c_int, C.c_int, _vp]),
    "cbg_net_read_changes": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _vp, _P(C.c_int64)]),
    "cbg_net_read_worst_case": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _P(C.c_int64)]),
    "cbg_net_read_stats": (C.c_int, [_vp, C.c_int, _P(LayerStatsC), C.c_int]),
    "cbg_net_read_counts": (C.c_int, [_vp, _vp]),
    "cbg_conv_create": (C.c_int, [_vp, _P(ConvSpecC), C.c_float, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_int, _P(_vp)]),
    "cbg_conv_destroy": (None, [_vp]),
    "cbg_conv_out_dims": (C.c_int, [_vp, _P(C.c_int), _P(C.c_int)]),
    "cbg_conv_forward": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int64, C.c_uint, _P(C.c_int64)]),
    "cbg_conv_read_output": (C.c_int, [_vp, _vp]),
    "cbg_conv_read_state": (C.c_int, [_vp, _vp]),
    "cbg_conv_read_changes": (C.c_int, [_vp, _vp, _vp, _P(C.c_int64)]),
    "cbg_conv_read_worst_case": (C.c_int, [_vp, _vp, _P(C.c_int64)]),
    "cbg_conv_set_tau": (C.c_int, [_vp, C.c_float]),
    "cbg_pool_create": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  _P(_vp)]),
    "cbg_pool_destroy": (None, [_vp]),
    "cbg_pool_forward": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int64, C.c_int]),
    "cbg_pool_read_output": (C.c_int, [_vp, _vp]),
    "cbg_pool_read_changes": (C.c_int, [_vp, _vp, _vp, _P(C.c_int64)]),
    "cbg_net_last_launches": (C.c_int, [_vp, _P(C.c_int)]),
    "cbg_net_set_kernel_timing": (C.c_int, [_vp, C.c_int]),
    "cbg_net_timing_report": (C.c_int, [_vp, C.c_char_p, C.c_int]),
    "cbg_net_copy_output_async": (C.c_int, [_vp, C.c_int, _vp]),
    "cbg_net_copy_output_detached": (C.c_int, [_vp, C.c_int, _vp]),
    "cbg_net_output_bytes": (C.c_int, [_vp, C.c_int, _P(C.c_int64)]),
    "cbg_net_output_delta_bytes": (C.c_int, [_vp, C.c_int, _P(C.c_int64)]),
    "cbg_host_alloc": (C.c_int, [C.c_int64, _P(_vp)]),
    "cbg_host_free": (None, [_vp]),
    "cbg_net_copy_output_delta": (C.c_int, [_vp, C.c_int, _vp]),
    "cbg_net_last_delta_dma_bytes": (C.c_int, [_vp, _P(C.c_int64)]),
    "cbg_net_apply_output_delta": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int, C.c_int]),
    "cbg_net_copy_counts_async": (C.c_int, [_vp, _vp, _vp]),
    "cbg_net_count_slots": (C.c_int, [_vp, _P(C.c_int)]),
    "cbg_net_detect_slots": (C.c_int, [_vp, _vp]),
    "cbg_ctx_set_persistent_sms": (C.c_int, [_vp, C.c_int]),
    "cbg_net_kernel_labels": (C.c_int, [_vp, C.c_uint, C.c_char_p, C.c_int]),
    "cbg_debug_gemm_trace": (C.c_int, [_vp, C.c_int]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class CbgError(RuntimeError):
    """Base of the errors raised from cbg status codes."""

    code = ERR_CUDA


class InvalidInputError(CbgError):
    """cbi::InvalidInputError (reference common.hpp:11-15)."""

    code = ERR_INVALID_INPUT


class ConfigError(CbgError):
    """cbi::ConfigError (reference common.hpp:17-21)."""

    code = ERR_CONFIG


class CudaError(CbgError):
    code = ERR_CUDA


class OutOfMemoryError(CbgError):
    code = ERR_OOM


class UnsupportedError(CbgError):
    code = ERR_UNSUPPORTED


_ERRORS = {ERR_INVALID_INPUT: InvalidInputError, ERR_CONFIG: ConfigError, ERR_CUDA: CudaError,
           ERR_OOM: OutOfMemoryError, ERR_UNSUPPORTED: UnsupportedError}


def check(status: int) -> None:
    if status != OK:
        msg = lib.cbg_last_error().decode(errors="replace")
        raise _ERRORS.get(status, CbgError)(msg)


def fptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None
