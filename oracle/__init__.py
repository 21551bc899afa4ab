"""CPU oracle for the DMPQ + TDC hot path of 6Bit-Diffusion (arxiv 2603.18742).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package. It shares no code with the CUDA path (``paper_2603_18742_b200``) and
neither imports the other.

Numerics live in ``dmpq_oracle.c`` (plain C loops, no FMA contraction, exhaustive
nearest-value conversions); the scalar decision logic (Eqs. 6, 7, 10, 11) lives
in :mod:`oracle.decisions`. This module is the numpy marshalling around the C
library. Citations: ``P:<line>`` = /root/reference/PAPER.md, ``S:<line>`` =
SPEC.md, ``Rn`` = reading n in DESIGN.md §3.

Parity status of each function is listed in DESIGN.md §4 ("pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .decisions import (  # noqa: F401  (re-export)
    FMT_BF16,
    FMT_INT8,
    FMT_NVFP4,
    purify_route,
    TdcConfig,
    TdcState,
    derive_tau_gamma,
    gamma_from_stats,
    route_block,
    tdc_decide,
    tdc_update,
    cosine_error_from_stats,
    prediction_error_from_stats,
    rel_l2_error_from_stats,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dmpq_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math",
           "-fexcess-precision=standard", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle C library in-tree (gcc). Returns the .so path."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *_CFLAGS, _SRC, "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I, F, LL = ctypes.c_int, ctypes.c_float, ctypes.c_longlong
        L.oracle_bf16_to_f32.argtypes, L.oracle_bf16_to_f32.restype = [ctypes.c_uint16], F
        L.oracle_f32_to_bf16.argtypes, L.oracle_f32_to_bf16.restype = [F], ctypes.c_uint16
        L.oracle_e4m3_decode.argtypes, L.oracle_e4m3_decode.restype = [ctypes.c_uint8], ctypes.c_double
        L.oracle_e4m3_encode_nonneg.argtypes, L.oracle_e4m3_encode_nonneg.restype = [F], ctypes.c_uint8
        L.oracle_e2m1_decode.argtypes, L.oracle_e2m1_decode.restype = [ctypes.c_uint8], ctypes.c_double
        L.oracle_e2m1_encode.argtypes, L.oracle_e2m1_encode.restype = [F], ctypes.c_uint8
        L.oracle_nvfp4_quantize.argtypes = [P, I, I, I, F, P, P]
        L.oracle_nvfp4_dequantize.argtypes = [P, P, I, I, F, P]
        L.oracle_global_scale.argtypes, L.oracle_global_scale.restype = [F, F], F
        L.oracle_sf_offset.argtypes, L.oracle_sf_offset.restype = [I, I, I], LL
        L.oracle_int8_quantize_rows.argtypes = [P, I, I, I, P, P]
        L.oracle_fht128_f32.argtypes = [P, P, LL]
        L.oracle_nvfp4_quantize_f32.argtypes = [P, I, I, F, P, P]
        L.oracle_int8_quantize_rows_f32.argtypes = [P, I, I, P, P]
        L.oracle_int8_quantize_blocks_f32.argtypes = [P, I, I, I, P, P]
        L.oracle_gemm_int8_blocks.argtypes = [P, P, I, P, P, P, I, I, I, I, I, P]
        L.oracle_pack_weights_hadamard.argtypes = [P, I, I, P, P, P, P, P, P]
        L.oracle_pack_weights.argtypes = [P, I, I, P, P, P, P, P]
        L.oracle_gemm_int8.argtypes, L.oracle_gemm_int8.restype = [P, P, P, P, P, I, I, I, I, I, P, P], I
        L.oracle_gemm_nvfp4.argtypes = [P, P, F, P, P, F, P, I, I, I, I, I, P]
        L.oracle_block_stats.argtypes = [P, P, P, LL, P, P]
        L.oracle_gemm_bf16.argtypes = [P, P, P, I, I, I, I, I, P]
        L.oracle_outlier_ratio.argtypes, L.oracle_outlier_ratio.restype = [P, LL, LL], ctypes.c_double
        L.oracle_tdc_skip.argtypes = [P, P, LL, P]
        L.oracle_amax_bf16.argtypes, L.oracle_amax_bf16.restype = [P, LL], F
        L.oracle_cache_dequant.argtypes = [P, P, F, LL, P]
        L.oracle_tdc_skip_nvfp4.argtypes = [P, P, P, F, LL, P]
        L.oracle_block_stats_nvfp4.argtypes = [P, P, P, P, F, I, I, F, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle inputs must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _u16(x: np.ndarray) -> np.ndarray:
    """bf16 payload as uint16 bits (accepts uint16 arrays or torch-exported views)."""
    x = np.ascontiguousarray(x)
    assert x.dtype == np.uint16, "bf16 tensors are passed as their uint16 bit patterns"
    return x


# ----------------------------------------------------------------------------- scalars

def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    """bf16 bits -> float32 values (storage widening, exact)."""
    return (np.asarray(bits, dtype=np.uint32) << 16).view(np.float32)


def f32_to_bf16(v: float) -> int:
    return int(lib().oracle_f32_to_bf16(float(v)))


def e4m3_decode(code: int) -> float:
    return float(lib().oracle_e4m3_decode(code))


def e4m3_encode(v: float) -> int:
    return int(lib().oracle_e4m3_encode_nonneg(v))


def e2m1_decode(nib: int) -> float:
    return float(lib().oracle_e2m1_decode(nib))


def e2m1_encode(v: float) -> int:
    return int(lib().oracle_e2m1_encode(v))


def global_scale(amax: float, div: float) -> float:
    """g = max(fl(amax/div), FLT_MIN) (reading R3)."""
    return float(lib().oracle_global_scale(amax, div))


def sf_offset(r: int, c: int, k: int) -> int:
    return int(lib().oracle_sf_offset(r, c, k))


def sf_swizzled_bytes(m: int, k: int) -> int:
    """Size of the swizzled scale buffer: rows padded to 128, scale cols to 4."""
    kc = ((k // 16) + 3) // 4 * 4
    return ((m + 127) // 128) * 128 * kc


def sf_swizzle(sf_logical: np.ndarray, m: int, k: int) -> np.ndarray:
    """Scatter logical [m x k/16] scales into the device layout (padding = 0)."""
    out = np.zeros(sf_swizzled_bytes(m, k), dtype=np.uint8)
    for r in range(m):
        for c in range(k // 16):
            out[sf_offset(r, c, k)] = sf_logical[r, c]
    return out


def sf_unswizzle(sf_dev: np.ndarray, m: int, k: int) -> np.ndarray:
    """Gather the device-layout scales back into logical [m x k/16]."""
    r = np.arange(m)[:, None]
    c = np.arange(k // 16)[None, :]
    kc = ((k // 16) + 3) // 4 * 4
    off = ((r // 128) * (kc // 4) + c // 4) * 512 + (r % 32) * 16 + ((r % 128) // 32) * 4 + (c % 4)
    return np.asarray(sf_dev)[off]


# ----------------------------------------------------------------------------- tensors

def nvfp4_quantize(x_bf16: np.ndarray, g: float):
    """NVFP4 quantization of a bf16 [m x k] matrix (Eq. 2, reading R3/R4).

    Returns (codes uint8 [m, k/2], sf uint8 [m, k/16] logical)."""
    x = _u16(x_bf16)
    m, k = x.shape
    assert k % 16 == 0
    codes = np.zeros((m, k // 2), dtype=np.uint8)
    sf = np.zeros((m, k // 16), dtype=np.uint8)
    lib().oracle_nvfp4_quantize(_p(x), m, k, k, float(g), _p(codes), _p(sf))
    return codes, sf


def nvfp4_dequantize(codes: np.ndarray, sf: np.ndarray, g: float) -> np.ndarray:
    m = codes.shape[0]
    k = codes.shape[1] * 2
    out = np.zeros((m, k), dtype=np.float64)
    lib().oracle_nvfp4_dequantize(_p(np.ascontiguousarray(codes)), _p(np.ascontiguousarray(sf)),
                                  m, k, float(g), _p(out))
    return out


def int8_quantize(x_bf16: np.ndarray):
    """Per-token symmetric INT8 (reading R2). Returns (codes int8 [m,k], scale f32 [m])."""
    x = _u16(x_bf16)
    m, k = x.shape
    codes = np.zeros((m, k), dtype=np.int8)
    scale = np.zeros(m, dtype=np.float32)
    lib().oracle_int8_quantize_rows(_p(x), m, k, k, _p(codes), _p(scale))
    return codes, scale


def pack_weights(w_bf16: np.ndarray):
    """Offline weight packing (reading R7). Returns a dict of the packed forms
    (scales in LOGICAL layout)."""
    w = _u16(w_bf16)
    n, k = w.shape
    out = dict(
        fp4_codes=np.zeros((n, k // 2), dtype=np.uint8),
        fp4_sf=np.zeros((n, k // 16), dtype=np.uint8),
        fp4_g=np.zeros(1, dtype=np.float32),
        i8_codes=np.zeros((n, k), dtype=np.int8),
        i8_scale=np.zeros(n, dtype=np.float32),
    )
    lib().oracle_pack_weights(_p(w), n, k, _p(out["fp4_codes"]), _p(out["fp4_sf"]), _p(out["fp4_g"]),
                              _p(out["i8_codes"]), _p(out["i8_scale"]))
    out["fp4_g"] = float(out["fp4_g"][0])
    return out


def fht128(x) -> np.ndarray:
    """Sylvester block Hadamard y = H_128 x over 128-element blocks of the last axis
    (reading R14: entries +-1, the 1/128 normalization rides on the weights),
    fp32 butterflies in the fixed stage order."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    assert x.shape[-1] % 128 == 0
    y = np.empty_like(x)
    lib().oracle_fht128_f32(_p(x), _p(y), x.size)
    return y


def nvfp4_quantize_f32(x32: np.ndarray, g: float):
    x = np.ascontiguousarray(x32, dtype=np.float32)
    m, k = x.shape
    codes = np.zeros((m, k // 2), dtype=np.uint8)
    sf = np.zeros((m, k // 16), dtype=np.uint8)
    lib().oracle_nvfp4_quantize_f32(_p(x), m, k, float(g), _p(codes), _p(sf))
    return codes, sf


def int8_quantize_f32(x32: np.ndarray):
    x = np.ascontiguousarray(x32, dtype=np.float32)
    m, k = x.shape
    codes = np.zeros((m, k), dtype=np.int8)
    scale = np.zeros(m, dtype=np.float32)
    lib().oracle_int8_quantize_rows_f32(_p(x), m, k, _p(codes), _p(scale))
    return codes, scale


def int8_quantize_blocks_f32(x32: np.ndarray, block: int = 128):
    """Per-block symmetric INT8 of FP32 rows (reading R17). Returns (codes int8 [m, k],
    scales f32 [m, k/block])."""
    x = np.ascontiguousarray(x32, dtype=np.float32)
    m, k = x.shape
    assert k % block == 0
    codes = np.zeros((m, k), dtype=np.int8)
    scale = np.zeros((m, k // block), dtype=np.float32)
    lib().oracle_int8_quantize_blocks_f32(_p(x), m, k, block, _p(codes), _p(scale))
    return codes, scale


def gemm_int8_blocks(a, s_a, w, s_w, bias, block: int = 128, rows=None) -> np.ndarray:
    """GEMM over per-block INT8 activations (R17): exact per-block integer sums, FP64 scaling."""
    a = np.ascontiguousarray(a, dtype=np.int8)
    w = np.ascontiguousarray(w, dtype=np.int8)
    m, k = a.shape
    n = w.shape[0]
    r0, r1 = (0, m) if rows is None else rows
    y = np.zeros((r1 - r0, n), dtype=np.float64)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    lib().oracle_gemm_int8_blocks(_p(a), _p(np.ascontiguousarray(s_a, dtype=np.float32)), block, _p(w),
                                  _p(np.ascontiguousarray(s_w, dtype=np.float32)), _p(b), m, n, k, r0, r1, _p(y))
    return y


def pack_weights_hadamard(w_bf16: np.ndarray):
    """Weight pack with the offline block-Hadamard rotation of every row (R14)."""
    w = _u16(w_bf16)
    n, k = w.shape
    out = dict(
        fp4_codes=np.zeros((n, k // 2), dtype=np.uint8),
        fp4_sf=np.zeros((n, k // 16), dtype=np.uint8),
        fp4_g=np.zeros(1, dtype=np.float32),
        i8_codes=np.zeros((n, k), dtype=np.int8),
        i8_scale=np.zeros(n, dtype=np.float32),
    )
    scratch = np.zeros((n, k), dtype=np.float32)
    lib().oracle_pack_weights_hadamard(_p(w), n, k, _p(out["fp4_codes"]), _p(out["fp4_sf"]), _p(out["fp4_g"]),
                                       _p(out["i8_codes"]), _p(out["i8_scale"]), _p(scratch))
    out["fp4_g"] = float(out["fp4_g"][0])
    return out


def gemm_int8(a, s_a, w, s_w, bias, rows=None):
    """INT8 GEMM + epilogue (reading R8). Returns (acc int32 [r,n], y float32 [r,n])."""
    a = np.ascontiguousarray(a, dtype=np.int8)
    w = np.ascontiguousarray(w, dtype=np.int8)
    m, k = a.shape
    n = w.shape[0]
    r0, r1 = (0, m) if rows is None else rows
    acc = np.zeros((r1 - r0, n), dtype=np.int32)
    y = np.zeros((r1 - r0, n), dtype=np.float32)
    s_a = np.ascontiguousarray(s_a, dtype=np.float32)
    s_w = np.ascontiguousarray(s_w, dtype=np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    ovf = lib().oracle_gemm_int8(_p(a), _p(s_a), _p(w), _p(s_w), _p(b), m, n, k, r0, r1, _p(acc), _p(y))
    assert ovf == 0, "int32 accumulator overflow"
    return acc, y


def gemm_nvfp4(a_codes, a_sf, g_a, w_codes, w_sf, g_w, bias, rows=None) -> np.ndarray:
    """NVFP4 GEMM + epilogue, fp64 accumulation over the same codes (reading R3)."""
    a_codes = np.ascontiguousarray(a_codes, dtype=np.uint8)
    w_codes = np.ascontiguousarray(w_codes, dtype=np.uint8)
    m, kh = a_codes.shape
    k = kh * 2
    n = w_codes.shape[0]
    r0, r1 = (0, m) if rows is None else rows
    y = np.zeros((r1 - r0, n), dtype=np.float64)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    lib().oracle_gemm_nvfp4(_p(a_codes), _p(np.ascontiguousarray(a_sf, dtype=np.uint8)), float(g_a),
                            _p(w_codes), _p(np.ascontiguousarray(w_sf, dtype=np.uint8)), float(g_w),
                            _p(b), m, n, k, r0, r1, _p(y))
    return y


def gemm_bf16(x_bf16, w_bf16, bias, rows=None) -> np.ndarray:
    """BF16 fallback GEMM of the PDR gate (R15), fp64 accumulation."""
    x = _u16(x_bf16)
    w = _u16(w_bf16)
    m, k = x.shape
    n = w.shape[0]
    r0, r1 = (0, m) if rows is None else rows
    y = np.zeros((r1 - r0, n), dtype=np.float64)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    lib().oracle_gemm_bf16(_p(x), _p(w), _p(b), m, n, k, r0, r1, _p(y))
    return y


def outlier_ratio(x_bf16, stride: int = 1) -> float:
    """R_outlier = max|X| / mean|X|."""
    x = _u16(x_bf16).reshape(-1)
    return float(lib().oracle_outlier_ratio(_p(x), x.size, stride))


def block_stats(x_in, x_out, delta_prev=None):
    """Predictor + TDC refresh statistics (Eqs. 3, 8, 9). Returns (delta_new bf16 bits, st[7])."""
    xi = _u16(x_in).reshape(-1)
    xo = _u16(x_out).reshape(-1)
    dp = None if delta_prev is None else _u16(delta_prev).reshape(-1)
    dn = np.zeros_like(xi)
    st = np.zeros(7, dtype=np.float64)
    lib().oracle_block_stats(_p(xi), _p(xo), _p(dp), xi.size, _p(dn), _p(st))
    return dn.reshape(np.shape(x_in)), st


def tdc_skip(x_in, delta):
    """TDC skip: X_out = bf16(X_in + Delta_tp)."""
    xi = _u16(x_in).reshape(-1)
    d = _u16(delta).reshape(-1)
    out = np.zeros_like(xi)
    lib().oracle_tdc_skip(_p(xi), _p(d), xi.size, _p(out))
    return out.reshape(np.shape(x_in))


def amax_bf16(x) -> float:
    xi = _u16(x).reshape(-1)
    return float(lib().oracle_amax_bf16(_p(xi), xi.size))


# ----------------------------------------------------------------------------- compressed delta cache (R16)

def cache_dequant(codes, sf, g: float) -> np.ndarray:
    """dq = fl32(dec(code) * fl32(dec(s_b) * g)) of an NVFP4-compressed delta cache (R16)."""
    c = np.ascontiguousarray(codes, dtype=np.uint8)
    f = np.ascontiguousarray(sf, dtype=np.uint8)
    n = c.size * 2
    out = np.zeros(n, dtype=np.float32)
    lib().oracle_cache_dequant(_p(c), _p(f), float(g), n, _p(out))
    return out.reshape(c.shape[0], -1) if c.ndim == 2 else out


def tdc_skip_nvfp4(x_in, codes, sf, g: float):
    """TDC skip with the compressed cache (R16): X_out = bf16(X_in + dq)."""
    xi = _u16(x_in).reshape(-1)
    out = np.zeros_like(xi)
    lib().oracle_tdc_skip_nvfp4(_p(xi), _p(np.ascontiguousarray(codes, dtype=np.uint8)),
                                _p(np.ascontiguousarray(sf, dtype=np.uint8)), float(g), xi.size, _p(out))
    return out.reshape(np.shape(x_in))


def block_stats_nvfp4(x_in, x_out, codes_prev, sf_prev, g_prev: float, g_new: float):
    """Refresh with the compressed cache (Eqs. 3, 8, 9; R16). Returns
    (codes_new [m, h/2], sf_new [m, h/16], st[7], amax |d|)."""
    xi = _u16(x_in)
    xo = _u16(x_out)
    m, h = xi.shape
    cn = np.zeros((m, h // 2), dtype=np.uint8)
    sn = np.zeros((m, h // 16), dtype=np.uint8)
    st = np.zeros(7, dtype=np.float64)
    am = np.zeros(1, dtype=np.float32)
    lib().oracle_block_stats_nvfp4(_p(xi), _p(xo), _p(np.ascontiguousarray(codes_prev, dtype=np.uint8)),
                                   _p(np.ascontiguousarray(sf_prev, dtype=np.uint8)), float(g_prev), m, h, float(g_new),
                                   _p(cn), _p(sn), _p(st), _p(am))
    return cn, sn, st, float(am[0])
