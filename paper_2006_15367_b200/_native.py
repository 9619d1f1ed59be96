"""ctypes binding of the C ABI in ``include/hfmm_gpu.h``.

The product path has no CPU fallback: if the native library is missing the
import of any entry point raises, and device calls on a machine without a GPU
return HFMM_ERR_NO_DEVICE which is raised as :class:`NoDeviceError`.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HFMM_LIB_PATH: an alternative build of the same library (A/B dev tools only)
LIB_PATH = os.environ.get("HFMM_LIB_PATH") or os.path.join(_HERE, "_lib", "libhfmm_b200.so")

HFMM_OK = 0


class HfmmError(RuntimeError):
    """Base class; ``status`` holds the hfmm_status code."""

    status = -1


class InvalidArgument(HfmmError, ValueError):  # std::invalid_argument
    status = 1


class OutOfRange(HfmmError, IndexError):  # std::out_of_range
    status = 2


class DomainError(HfmmError, ArithmeticError):  # std::domain_error
    status = 3


class LogicError(HfmmError):  # std::logic_error
    status = 4


class LengthError(HfmmError):  # std::length_error
    status = 5


class CudaError(HfmmError):
    status = 6


class NoDeviceError(HfmmError):
    status = 7


_BY_STATUS = {c.status: c for c in (InvalidArgument, OutOfRange, DomainError, LogicError,
                                     LengthError, CudaError, NoDeviceError)}


class RunConfigC(ctypes.Structure):
    _fields_ = [
        ("lambda_", ctypes.c_double),
        ("digits", ctypes.c_double),
        ("leaf_lambda", ctypes.c_double),
        ("num_ranks", ctypes.c_int32),
        ("policy", ctypes.c_int32),
        ("buffer_limit", ctypes.c_uint64),
        ("one_particle_per_leaf", ctypes.c_int32),
        ("top_level", ctypes.c_int32),
        ("d_override", ctypes.c_int32),
        ("scheduler", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("partition_weight", ctypes.c_int32),
        ("setup_device", ctypes.c_int32),
    ]


class TimingC(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 8), ("kernel_launches", ctypes.c_int64)]


_lib = None

_P = ctypes.c_void_p
_SIG = {
    "hfmm_run_config_default": (None, [ctypes.POINTER(RunConfigC)]),
    "hfmm_last_error": (ctypes.c_char_p, []),
    "hfmm_setup_build": (ctypes.c_int, [_P, _P, ctypes.c_size_t, ctypes.POINTER(RunConfigC),
                                        ctypes.POINTER(_P)]),
    "hfmm_setup_destroy": (None, [_P]),
    "hfmm_setup_import_begin": (ctypes.c_int, [ctypes.POINTER(RunConfigC), ctypes.POINTER(_P)]),
    "hfmm_setup_import_put": (ctypes.c_int, [_P, ctypes.c_char_p, _P, ctypes.c_size_t]),
    "hfmm_setup_import_end": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "hfmm_setup_import_abort": (None, [_P]),
    "hfmm_world_create": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.POINTER(_P)]),
    "hfmm_world_destroy": (None, [_P]),
    "hfmm_world_set_charges": (ctypes.c_int, [_P, _P]),
    "hfmm_world_run_phase": (ctypes.c_int, [_P, ctypes.c_int]),
    "hfmm_world_evaluate": (ctypes.c_int, [_P, _P, _P, _P]),
    "hfmm_world_potentials": (ctypes.c_int, [_P, _P]),
    "hfmm_world_get_expansion": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, ctypes.c_size_t]),
    "hfmm_setup_get": (ctypes.c_int, [_P, ctypes.c_char_p, _P, ctypes.c_size_t,
                                      ctypes.POINTER(ctypes.c_size_t)]),
    "hfmm_gpu_create": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    "hfmm_gpu_destroy": (None, [_P]),
    "hfmm_gpu_evaluate": (ctypes.c_int, [_P, _P, _P, ctypes.POINTER(TimingC)]),
    "hfmm_gpu_evaluate_device": (ctypes.c_int, [_P, _P, _P, _P]),
    "hfmm_gpu_last_timing": (ctypes.c_int, [_P, ctypes.POINTER(TimingC)]),
    "hfmm_gpu_set_charges": (ctypes.c_int, [_P, _P]),
    "hfmm_gpu_run_phase": (ctypes.c_int, [_P, ctypes.c_int]),
    "hfmm_gpu_get_expansion": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _P, ctypes.c_size_t]),
    "hfmm_gpu_get_potentials_sorted": (ctypes.c_int, [_P, _P, ctypes.c_size_t]),
    "hfmm_gpu_exchange_sizes": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "hfmm_gpu_pack": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]),
    "hfmm_gpu_unpack": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]),
    "hfmm_gpu_run_level": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int]),
    "hfmm_gpu_set_stream": (ctypes.c_int, [_P, _P]),
    "hfmm_gpu_synchronize": (ctypes.c_int, [_P]),
    "hfmm_gpu_load_charges_device": (ctypes.c_int, [_P, _P]),
    "hfmm_gpu_particle_range": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "hfmm_gpu_store_potentials_device": (ctypes.c_int, [_P, _P]),
    "hfmm_gpu_launch_count": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64)]),
    "hfmm_gpu_set_overlap": (ctypes.c_int, [_P, ctypes.c_int]),
    "hfmm_evaluate_potential": (ctypes.c_int, [_P, _P, ctypes.c_size_t, ctypes.POINTER(RunConfigC),
                                               ctypes.c_int, _P]),
    "hfmm_gpu_direct": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _P, ctypes.c_size_t, ctypes.c_double,
                                       ctypes.c_int, _P]),
    "hfmm_resample_matrix": (ctypes.c_int, [ctypes.c_int64, ctypes.c_double, ctypes.c_int64,
                                            ctypes.c_double, _P]),
    "hfmm_m2m_operands": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, ctypes.POINTER(ctypes.c_int)]),
    "hfmm_l2l_operands": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _P, _P,
                                         ctypes.POINTER(ctypes.c_int)]),
    "hfmm_generate_inputs": (None, [ctypes.c_int, ctypes.c_size_t, ctypes.c_double, ctypes.c_uint64,
                                    _P, _P]),
}

EXPORTED_SYMBOLS = tuple(_SIG)


def lib() -> ctypes.CDLL:
    """Loads libhfmm_b200.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"native library {LIB_PATH} is missing; run __graft_entry__.build() "
                "(there is no CPU fallback for the MLFMA engine)")
        h = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIG.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(status: int) -> None:
    if status == HFMM_OK:
        return
    msg = lib().hfmm_last_error().decode(errors="replace")
    raise _BY_STATUS.get(status, HfmmError)(msg or f"hfmm status {status}")


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return ctypes.c_void_p(a.ctypes.data)
