"""ctypes view of libdmpq's C ABI (include/dmpq.h). Argument marshalling only.

The library is built in-tree (``paper_2603_18742_b200/libdmpq.so``) by
``paper_2603_18742_b200.build``. There is no fallback: if it cannot be loaded,
every entry point raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdmpq.so")

c_int, c_float, c_double, c_void_p, c_uint32, c_size_t = (
    ctypes.c_int, ctypes.c_float, ctypes.c_double, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_size_t)

DMPQ_OK, DMPQ_EINVAL, DMPQ_ESHAPE, DMPQ_EALIGN, DMPQ_EZERONORM, DMPQ_ECUDA, DMPQ_EUNSUPPORTED = range(7)
STATUS_NAMES = ["DMPQ_OK", "DMPQ_EINVAL", "DMPQ_ESHAPE", "DMPQ_EALIGN", "DMPQ_EZERONORM", "DMPQ_ECUDA",
                "DMPQ_EUNSUPPORTED"]
FMT_INT8, FMT_NVFP4, FMT_BF16 = 0, 1, 2
QF_LAYERNORM, QF_WRITE_H, QF_HADAMARD = 1, 2, 4
PACK_HADAMARD = 1
EP_BIAS, EP_GELU_TANH, EP_RESIDUAL, EP_TDC_REFRESH, EP_QUANT_NVFP4 = 1, 2, 4, 8, 16
TDC_SKIP, TDC_REFRESH = 0, 1
TDC_COMPUTE, TDC_DECIDE_SKIP = 0, 1
GAMMA_L1, GAMMA_L2 = 0, 1
TDC_METRIC_COS, TDC_METRIC_REL_L2 = 0, 1
STATS_LEN = 7


class Weights(ctypes.Structure):
    _fields_ = [("n", c_int), ("k", c_int), ("fp4_codes", c_void_p), ("fp4_sf", c_void_p), ("fp4_g", c_void_p),
                ("i8_codes", c_void_p), ("i8_scale", c_void_p), ("bias", c_void_p), ("bf16_w", c_void_p),
                ("fp4_g_col", c_void_p), ("i8_rcp", c_void_p)]


class Act(ctypes.Structure):
    _fields_ = [("fmt", c_int), ("m", c_int), ("k", c_int), ("codes", c_void_p), ("sf", c_void_p), ("g", c_void_p),
                ("row_scale", c_void_p), ("scale_block", c_int)]


class QuantOpts(ctypes.Structure):
    _fields_ = [("flags", c_uint32), ("ln_eps", c_float), ("h_out", c_void_p), ("ldh", c_int),
                ("row_abs_sum", c_void_p), ("amax_in", c_void_p)]


class Epilogue(ctypes.Structure):
    _fields_ = [("flags", c_uint32), ("gate", c_void_p), ("residual", c_void_p), ("ldr", c_int),
                ("tdc_x_in", c_void_p), ("tdc_delta", c_void_p), ("tdc_stats", c_void_p), ("tdc_workspace", c_void_p),
                ("run_if", c_void_p), ("run_if_value", c_int), ("q_out", c_void_p), ("q_amax", c_void_p)]


class BlockStats(ctypes.Structure):
    _fields_ = [("sum_abs_d", c_double), ("sum_abs_x", c_double), ("sum_d2", c_double), ("sum_x2", c_double),
                ("dot_dd", c_double), ("sum_dn2", c_double), ("sum_dp2", c_double)]

    @classmethod
    def from_seq(cls, v):
        return cls(*[float(x) for x in v])

    def as_list(self):
        return [self.sum_abs_d, self.sum_abs_x, self.sum_d2, self.sum_x2, self.dot_dd, self.sum_dn2, self.sum_dp2]


class TdcNvfp4Cache(ctypes.Structure):
    _fields_ = [("codes", c_void_p), ("sf", c_void_p), ("g", c_void_p)]


class TdcState(ctypes.Structure):
    _fields_ = [("t_p", c_int), ("e_tp", c_double), ("e_acc", c_double), ("last", c_int), ("n_computed", c_int)]


class TdcConfig(ctypes.Structure):
    _fields_ = [("rho", c_double), ("tau", c_double), ("n_max", c_int), ("metric", c_int)]


# every function the header declares (checked against include/dmpq.h by the tests)
_SIGNATURES = {
    "dmpq_last_error": ([], ctypes.c_char_p),
    "dmpq_version": ([], ctypes.c_char_p),
    "dmpq_prepare": ([], c_int),
    "dmpq_sf_bytes": ([c_int, c_int], c_size_t),
    "tdc_workspace_bytes": ([c_int, c_int], c_size_t),
    "dmpq_gemm_tdc_workspace_bytes": ([], c_size_t),
    "dmpq_pack_weights": ([c_void_p, c_int, c_int, ctypes.POINTER(Weights), c_void_p], c_int),
    "dmpq_pack_weights_ex": ([c_void_p, c_int, c_int, c_uint32, ctypes.POINTER(Weights), c_void_p], c_int),
    "dmpq_cast_int8": ([ctypes.POINTER(Weights), c_void_p, c_void_p], c_int),
    "dmpq_derive_tau": ([c_double, c_double, c_double, c_double], c_double),
    "dmpq_predict": ([ctypes.POINTER(BlockStats), ctypes.POINTER(c_double), c_int, c_int, c_int, c_int,
                      ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(c_double)], c_int),
    "dmpq_quantize_act": ([c_void_p, c_int, c_int, c_int, ctypes.POINTER(QuantOpts), ctypes.POINTER(Act),
                           ctypes.POINTER(Act), c_void_p, c_void_p], c_int),
    "dmpq_outlier_gate": ([c_void_p, c_int, c_void_p, c_double, c_double, c_void_p, c_void_p, c_void_p], c_int),
    "dmpq_outlier_ratio": ([c_double, c_double, c_double], c_double),
    "dmpq_global_scale": ([c_void_p, c_float, c_void_p, c_int, c_void_p], c_int),
    "dmpq_outlier_reduce": ([c_void_p, c_int, c_int, c_void_p, c_void_p], c_int),
    "dmpq_purify": ([ctypes.POINTER(c_double), c_int, c_int, c_double, ctypes.POINTER(ctypes.c_uint8)], None),
    "dmpq_gemm": ([ctypes.POINTER(Act), ctypes.POINTER(Weights), ctypes.POINTER(Epilogue), c_void_p, c_int, c_void_p,
                   c_void_p, c_void_p], c_int),
    "tdc_step": ([c_int, c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p], c_int),
    "tdc_step_nvfp4": ([c_int, c_void_p, c_void_p, ctypes.POINTER(TdcNvfp4Cache), c_void_p, c_void_p, c_int, c_int,
                        c_void_p, c_void_p, c_void_p], c_int),
    "tdc_delta_amax": ([c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p], c_int),
    "tdc_init": ([ctypes.POINTER(TdcState)], None),
    "tdc_decide": ([ctypes.POINTER(TdcState), ctypes.POINTER(TdcConfig), c_int], c_int),
    "tdc_update": ([ctypes.POINTER(TdcState), ctypes.POINTER(TdcConfig), c_int, c_int, ctypes.POINTER(BlockStats)], None),
}

_lib = None


class DmpqError(RuntimeError):
    def __init__(self, fn: str, status: int, detail: str):
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{fn} -> {name}: {detail}")
        self.status = status


def lib() -> ctypes.CDLL:
    """Load libdmpq.so (raises if it has not been built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; build it with `python -m paper_2603_18742_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def check(fn: str, status: int, allow=()) -> int:
    if status != DMPQ_OK and status not in allow:
        raise DmpqError(fn, status, lib().dmpq_last_error().decode())
    return status


def exported_names():
    return list(_SIGNATURES)
