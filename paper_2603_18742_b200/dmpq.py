"""Python binding of libdmpq with the C ABI's names (include/dmpq.h).

Argument marshalling only: torch supplies device memory and the current CUDA
stream; every step of the hot path runs in libdmpq's sm_100a kernels. There is
no CPU or eager-PyTorch fallback — a missing library or GPU raises.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import torch

from . import _lib as L

__all__ = [
    "PackedWeights", "QuantAct", "dmpq_pack_weights", "dmpq_predict", "dmpq_derive_tau", "dmpq_quantize_act",
    "dmpq_global_scale", "dmpq_gemm", "dmpq_cast_int8", "tdc_step", "tdc_decide", "tdc_update", "tdc_new_state", "sf_bytes",
    "tdc_workspace_bytes", "FMT_INT8", "FMT_NVFP4", "FMT_BF16",
]

FMT_INT8, FMT_NVFP4, FMT_BF16 = L.FMT_INT8, L.FMT_NVFP4, L.FMT_BF16


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _check_dev(t: torch.Tensor, name: str, dtype=None):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (libdmpq has no CPU path)")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


def sf_bytes(rows: int, k: int) -> int:
    return int(L.lib().dmpq_sf_bytes(rows, k))


def tdc_workspace_bytes(m: int, h: int) -> int:
    return int(L.lib().tdc_workspace_bytes(m, h))


# --------------------------------------------------------------------------- weights

@dataclass
class PackedWeights:
    n: int
    k: int
    fp4_codes: torch.Tensor
    fp4_sf: torch.Tensor
    fp4_g: torch.Tensor
    i8_codes: torch.Tensor | None          # None: NVFP4-only residency (INT8 cast per GEMM, dmpq_cast_int8)
    i8_scale: torch.Tensor
    bias: torch.Tensor | None
    c: L.Weights = field(default=None, repr=False)
    hadamard: bool = False
    bf16_w: torch.Tensor | None = None     # unquantised weights for the PDR BF16 fallback (R15)
    i8_rcp: torch.Tensor | None = None     # r_w = fl(127 / max|W^|) per row (the cast's INT8 scale)
    g_col: torch.Tensor | None = None

    def keep_bf16(self, W: torch.Tensor):
        self.bf16_w = W.contiguous()
        self.c.bf16_w = self.bf16_w.data_ptr()
        return self

    @classmethod
    def empty(cls, n: int, k: int, device, bias: torch.Tensor | None = None, int8_resident: bool = True):
        d = dict(device=device)
        return cls._from_tensors(
            n, k, torch.empty((n, k // 2), dtype=torch.uint8, **d), torch.zeros(sf_bytes(n, k), dtype=torch.uint8, **d),
            torch.zeros(1, dtype=torch.float32, **d),
            torch.empty((n, k), dtype=torch.int8, **d) if int8_resident else None,
            torch.empty(n, dtype=torch.float32, **d),
            None if bias is None else bias.to(device=device, dtype=torch.float32).contiguous(), None, False,
            i8_rcp=torch.empty(n, dtype=torch.float32, **d))

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in
                   (self.fp4_codes, self.fp4_sf, self.fp4_g, self.i8_codes, self.i8_scale, self.i8_rcp) if t is not None)

    @classmethod
    def _from_tensors(cls, n, k, codes, sf, g, i8, i8s, bias, bf16_w, hadamard, g_col=None, i8_rcp=None):
        pw = cls(n, k, codes, sf, g, i8, i8s, bias, hadamard=hadamard, bf16_w=bf16_w, i8_rcp=i8_rcp, g_col=g_col)
        pw.c = L.Weights(n, k, codes.data_ptr(), sf.data_ptr(), g.data_ptr(), _ptr_or_none(i8), i8s.data_ptr(),
                         _ptr_or_none(bias), _ptr_or_none(bf16_w), _ptr_or_none(g_col), _ptr_or_none(i8_rcp))
        return pw


def _ptr_or_none(t):
    return None if t is None else t.data_ptr()


def dmpq_concat_weights(pws: list) -> tuple:
    """Pack several layers over the same input side by side along n (e.g. Q, K, V): returns the
    concatenated PackedWeights (each layer keeps its own NVFP4 g_w through fp4_g_col, so one GEMM
    gives the separate GEMMs' outputs bit for bit) and per-layer views into it (same contents as
    the inputs, which can then be freed). Needs every n % 128 == 0 (whole scale-atom row tiles)."""
    k = pws[0].k
    if any(p.k != k or p.n % 128 for p in pws) or len({p.hadamard for p in pws}) != 1:
        raise ValueError("dmpq_concat_weights: equal k, n % 128 == 0 and one Hadamard setting required")
    has_bias = all(p.bias is not None for p in pws)
    has_bf16 = all(p.bf16_w is not None for p in pws)
    if not has_bias and any(p.bias is not None for p in pws):
        raise ValueError("dmpq_concat_weights: bias on some layers but not on others")
    if not has_bf16 and any(p.bf16_w is not None for p in pws):
        raise ValueError("dmpq_concat_weights: bf16_w kept on some layers but not on others")
    n = sum(p.n for p in pws)
    if len({p.i8_codes is None for p in pws}) != 1 or len({p.i8_rcp is None for p in pws}) != 1:
        raise ValueError("dmpq_concat_weights: mixed INT8 residency")
    codes = torch.cat([p.fp4_codes for p in pws])
    sf = torch.cat([p.fp4_sf for p in pws])
    i8 = None if pws[0].i8_codes is None else torch.cat([p.i8_codes for p in pws])
    i8s = torch.cat([p.i8_scale for p in pws])
    rcp = None if pws[0].i8_rcp is None else torch.cat([p.i8_rcp for p in pws])
    bias = torch.cat([p.bias for p in pws]) if has_bias else None
    bf16_w = torch.cat([p.bf16_w for p in pws]) if has_bf16 else None
    g_col = torch.cat([p.fp4_g.expand(p.n) for p in pws]).contiguous()
    cat = PackedWeights._from_tensors(n, k, codes, sf, g_col[:1], i8, i8s, bias, bf16_w, pws[0].hadamard, g_col,
                                      i8_rcp=rcp)
    views, r0, s0 = [], 0, 0
    sl = lambda t, a, b: None if t is None else t[a:b]
    for p in pws:
        ns = p.fp4_sf.numel()
        views.append(PackedWeights._from_tensors(
            p.n, k, codes[r0:r0 + p.n], sf[s0:s0 + ns], g_col[r0:r0 + 1], sl(i8, r0, r0 + p.n), i8s[r0:r0 + p.n],
            sl(bias, r0, r0 + p.n), sl(bf16_w, r0, r0 + p.n), p.hadamard, i8_rcp=sl(rcp, r0, r0 + p.n)))
        r0 += p.n
        s0 += ns
    return cat, views


def dmpq_pack_weights(W: torch.Tensor, bias: torch.Tensor | None = None, hadamard: bool = False,
                      keep_bf16: bool = False, int8_resident: bool = True) -> PackedWeights:
    """Offline pack of nn.Linear weights W [n, k] (bf16, CUDA) in both formats (R7);
    hadamard=True rotates every row by the block FHT first (R14). int8_resident=False keeps
    only the NVFP4 form (+ the per-row INT8 scales): INT8 codes are then cast per GEMM
    (dmpq_cast_int8, P:184's on-the-fly cast)."""
    _check_dev(W, "W", torch.bfloat16)
    W = W.contiguous()
    n, k = W.shape
    pw = PackedWeights.empty(n, k, W.device, bias, int8_resident=int8_resident)
    if hadamard:
        L.check("dmpq_pack_weights_ex", L.lib().dmpq_pack_weights_ex(_ptr(W), n, k, L.PACK_HADAMARD, ctypes.byref(pw.c),
                                                                     _stream(W.device)))
    else:
        L.check("dmpq_pack_weights", L.lib().dmpq_pack_weights(_ptr(W), n, k, ctypes.byref(pw.c), _stream(W.device)))
    pw.hadamard = hadamard
    if keep_bf16:
        pw.keep_bf16(W)
    return pw


def dmpq_cast_int8(W: PackedWeights, scratch: torch.Tensor) -> PackedWeights:
    """On-the-fly NVFP4 -> INT8 weight cast (NEXT-4b): writes W's INT8 codes into `scratch`
    (int8, >= n*k elements, reused across layers) and returns W viewed with i8_codes = scratch."""
    _check_dev(scratch, "scratch", torch.int8)
    if scratch.numel() < W.n * W.k:
        raise ValueError("dmpq_cast_int8: scratch too small")
    i8 = scratch.view(-1)[: W.n * W.k].view(W.n, W.k)
    L.check("dmpq_cast_int8", L.lib().dmpq_cast_int8(ctypes.byref(W.c), _ptr(i8), _stream(scratch.device)))
    v = PackedWeights._from_tensors(W.n, W.k, W.fp4_codes, W.fp4_sf, W.fp4_g, i8, W.i8_scale, W.bias, W.bf16_w,
                                    W.hadamard, W.g_col, i8_rcp=W.i8_rcp)
    return v


# --------------------------------------------------------------------------- activations

@dataclass
class QuantAct:
    fmt: int
    m: int
    k: int
    codes: torch.Tensor
    sf: torch.Tensor | None = None
    g: torch.Tensor | None = None
    row_scale: torch.Tensor | None = None
    c: L.Act = field(default=None, repr=False)

    scale_block: int = 0

    @classmethod
    def empty(cls, fmt: int, m: int, k: int, device, g: torch.Tensor | None = None, scale_block: int = 0):
        """scale_block (INT8 only): 0 per-token scales [m] (R2); 128 per-block scales [m, k/128] (R17)."""
        d = dict(device=device)
        if fmt == FMT_NVFP4:
            if g is None:
                raise ValueError("an NVFP4 activation needs its global scale tensor g (R3)")
            a = cls(fmt, m, k, torch.empty((m, k // 2), dtype=torch.uint8, **d),
                    sf=torch.empty(sf_bytes(m, k), dtype=torch.uint8, **d), g=g)
            a.c = L.Act(fmt, m, k, a.codes.data_ptr(), a.sf.data_ptr(), g.data_ptr(), None)
        else:
            if scale_block not in (0, 128) or (scale_block and k % scale_block):
                raise ValueError("scale_block must be 0 or 128 (dividing k)")
            a = cls(fmt, m, k, torch.empty((m, k), dtype=torch.int8, **d),
                    row_scale=torch.empty((m, k // scale_block) if scale_block else m, dtype=torch.float32, **d),
                    scale_block=scale_block)
            a.c = L.Act(fmt, m, k, a.codes.data_ptr(), None, None, a.row_scale.data_ptr(), scale_block)
        return a

    @classmethod
    def bf16(cls, X: torch.Tensor):
        """The unquantised activation itself, for the BF16 (PDR fallback) GEMM path."""
        _check_dev(X, "X", torch.bfloat16)
        if not X.is_contiguous():   # the BF16 GEMM's A tensor map has row stride k (include/dmpq.h dmpq_act)
            raise ValueError("a BF16 activation must be dense (row stride k)")
        m, k = X.shape
        a = cls(FMT_BF16, m, k, X)
        a.c = L.Act(FMT_BF16, m, k, X.data_ptr(), None, None, None)
        return a


def dmpq_quantize_act(X: torch.Tensor, out_i8: QuantAct | None = None, out_fp4: QuantAct | None = None,
                      amax_out: torch.Tensor | None = None, layernorm: bool = False, ln_eps: float = 1e-6,
                      h_out: torch.Tensor | None = None, hadamard: bool = False,
                      row_abs_sum: torch.Tensor | None = None, amax_in: torch.Tensor | None = None):
    """Quantize X [m, k] (bf16, CUDA, row stride X.stride(0)) into the given outputs (Eq. 2 / P:115)."""
    _check_dev(X, "X", torch.bfloat16)
    if X.stride(1) != 1:
        raise ValueError("X rows must be contiguous")
    m, k = X.shape
    opts = None
    flags = (L.QF_LAYERNORM if layernorm else 0) | (L.QF_WRITE_H if h_out is not None else 0) | \
        (L.QF_HADAMARD if hadamard else 0)
    if flags or row_abs_sum is not None or amax_in is not None:
        opts = L.QuantOpts(flags, ln_eps, None if h_out is None else h_out.data_ptr(),
                           0 if h_out is None else h_out.stride(0),
                           None if row_abs_sum is None else row_abs_sum.data_ptr(),
                           None if amax_in is None else amax_in.data_ptr())
    L.check("dmpq_quantize_act", L.lib().dmpq_quantize_act(
        _ptr(X), m, k, X.stride(0), None if opts is None else ctypes.byref(opts),
        None if out_i8 is None else ctypes.byref(out_i8.c), None if out_fp4 is None else ctypes.byref(out_fp4.c),
        _ptr(amax_out), _stream(X.device)))
    return out_i8, out_fp4


def dmpq_outlier_reduce(row_sums: torch.Tensor, out: torch.Tensor):
    """out[s] = sum_r row_sums[s, r] in FP64, fixed order (PDR statistics, R15)."""
    seg, m = row_sums.shape
    L.check("dmpq_outlier_reduce", L.lib().dmpq_outlier_reduce(_ptr(row_sums), m, seg, _ptr(out), _stream(row_sums.device)))
    return out


def dmpq_outlier_ratio(max_abs: float, sum_abs: float, count: float) -> float:
    """R = max|x| / mean|x|; 1 for an all-zero input."""
    return float(L.lib().dmpq_outlier_ratio(float(max_abs), float(sum_abs), float(count)))


def dmpq_outlier_gate(row_abs_sum: torch.Tensor, amax_in: torch.Tensor, count: float, tau_outlier: float,
                      flag_out: torch.Tensor, sum_out: torch.Tensor | None = None):
    """Current-input PDR gate on the device (R18): flag_out[0] = R > tau_outlier."""
    L.check("dmpq_outlier_gate", L.lib().dmpq_outlier_gate(
        _ptr(row_abs_sum), row_abs_sum.numel(), _ptr(amax_in), float(count), float(tau_outlier), _ptr(sum_out),
        _ptr(flag_out), _stream(row_abs_sum.device)))
    return flag_out


def dmpq_purify(fmts, ratios, prev_skipped: bool, tau_outlier: float = 25.0):
    """Purified Cache Refresh gate (R15): BF16 if ratio > tau_outlier, INT8 after a skip."""
    n = len(fmts)
    f = (ctypes.c_uint8 * max(n, 1))(*fmts)
    r = None if ratios is None else (ctypes.c_double * n)(*[float(x) for x in ratios])
    L.lib().dmpq_purify(r, n, int(bool(prev_skipped)), float(tau_outlier), f)
    return [int(f[i]) for i in range(n)]


def dmpq_global_scale(amax: torch.Tensor, div: float, g_out: torch.Tensor):
    """g = max(fl(amax/div), FLT_MIN) on the device (R3)."""
    _check_dev(amax, "amax", torch.float32)
    L.check("dmpq_global_scale", L.lib().dmpq_global_scale(_ptr(amax), div, _ptr(g_out), amax.numel(),
                                                           _stream(amax.device)))
    return g_out


# --------------------------------------------------------------------------- GEMM

def dmpq_gemm(A: QuantAct, W: PackedWeights, Y: torch.Tensor | None = None, Y32: torch.Tensor | None = None,
              acc: torch.Tensor | None = None, bias: bool = True, gelu: bool = False,
              residual: torch.Tensor | None = None, gate: torch.Tensor | None = None,
              tdc_x_in: torch.Tensor | None = None, tdc_delta: torch.Tensor | None = None,
              tdc_stats: torch.Tensor | None = None, tdc_workspace: torch.Tensor | None = None,
              run_if: torch.Tensor | None = None, run_if_value: int = 0,
              quant_out: QuantAct | None = None, quant_amax: torch.Tensor | None = None):
    """Y = epilogue(A @ W^T) on tcgen05 (kind::i8 or kind::mxf4nvf4). With tdc_x_in / tdc_delta /
    tdc_stats / tdc_workspace the epilogue also runs the TDC refresh of X_out = Y (fused tdc_step)."""
    flags = (L.EP_BIAS if (bias and W.bias is not None) else 0) | (L.EP_GELU_TANH if gelu else 0)
    if residual is not None:
        flags |= L.EP_RESIDUAL
    if quant_out is not None:   # producer-fused NVFP4 quantization of bf16(Y) (NEXT-2)
        flags |= L.EP_QUANT_NVFP4
    if tdc_x_in is not None:
        flags |= L.EP_TDC_REFRESH
        for t_, n_ in ((tdc_x_in, "tdc_x_in"), (tdc_delta, "tdc_delta")):
            _check_dev(t_, n_, torch.bfloat16)
    ep = None
    if flags or run_if is not None:   # run_if: int32 device flag, the GEMM runs iff *run_if == run_if_value (R18)
        ep = L.Epilogue(flags, _ptr(gate), _ptr(residual), 0 if residual is None else residual.stride(0),
                        _ptr(tdc_x_in), _ptr(tdc_delta), _ptr(tdc_stats), _ptr(tdc_workspace), _ptr(run_if),
                        int(run_if_value), None if quant_out is None else ctypes.addressof(quant_out.c),
                        _ptr(quant_amax))
    if Y is not None:
        _check_dev(Y, "Y", torch.bfloat16)
    L.check("dmpq_gemm", L.lib().dmpq_gemm(
        ctypes.byref(A.c), ctypes.byref(W.c), None if ep is None else ctypes.byref(ep), _ptr(Y),
        0 if Y is None else Y.stride(0), _ptr(Y32), _ptr(acc), _stream(A.codes.device)))
    return Y


def dmpq_gemm_tdc_workspace_bytes() -> int:
    return int(L.lib().dmpq_gemm_tdc_workspace_bytes())


# --------------------------------------------------------------------------- predictor (host-pure)

def dmpq_derive_tau(alpha: float, beta: float, tau_rel: float, eps_slope: float = 1e-8) -> float:
    return float(L.lib().dmpq_derive_tau(alpha, beta, tau_rel, eps_slope))


def dmpq_predict(stats, tau_gamma, t: int, prev_skipped: bool, metric: int = L.GAMMA_L1):
    """Eq. 7 routing of one block's layers. Returns (fmts list, gamma or nan, status)."""
    n = len(tau_gamma)
    taus = (ctypes.c_double * n)(*[float(x) for x in tau_gamma])
    fmts = (ctypes.c_uint8 * max(n, 1))()
    gamma = ctypes.c_double(0.0)
    st = None if stats is None else (stats if isinstance(stats, L.BlockStats) else L.BlockStats.from_seq(stats))
    rc = L.lib().dmpq_predict(None if st is None else ctypes.byref(st), taus, n, t, int(bool(prev_skipped)), metric,
                              fmts, ctypes.byref(gamma))
    L.check("dmpq_predict", rc, allow=(L.DMPQ_EZERONORM,))
    return [int(fmts[i]) for i in range(n)], gamma.value, rc


# --------------------------------------------------------------------------- TDC

def tdc_step(mode: int, x_in: torch.Tensor, x_out: torch.Tensor, delta: torch.Tensor,
             stats_out: torch.Tensor | None = None, workspace: torch.Tensor | None = None):
    """SKIP: x_out = x_in + delta. REFRESH: delta <- x_out - x_in, FP64 stats (Eqs. 3/8/9)."""
    m, h = x_in.shape
    L.check("tdc_step", L.lib().tdc_step(mode, _ptr(x_in), _ptr(x_out), _ptr(delta), m, h, _ptr(stats_out),
                                         _ptr(workspace), _stream(x_in.device)))


class DeltaCacheNvfp4:
    """NVFP4-compressed delta cache of one block (R16): codes [m, h/2], row-major
    E4M3 scales [m, h/16], and the device global scale it was written with. Zeroed."""

    def __init__(self, m: int, h: int, device):
        self.m, self.h = m, h
        self.codes = torch.zeros(m, h // 2, dtype=torch.uint8, device=device)
        self.sf = torch.zeros(m, h // 16, dtype=torch.uint8, device=device)
        self.g = torch.zeros(1, dtype=torch.float32, device=device)

    def c(self) -> L.TdcNvfp4Cache:
        return L.TdcNvfp4Cache(_ptr(self.codes), _ptr(self.sf), _ptr(self.g))

    def nbytes(self) -> int:
        return self.codes.numel() + self.sf.numel() + 4


def tdc_step_nvfp4(mode: int, x_in: torch.Tensor, x_out: torch.Tensor, cache: DeltaCacheNvfp4,
                   g_new: torch.Tensor | None = None, amax_out: torch.Tensor | None = None,
                   stats_out: torch.Tensor | None = None, workspace: torch.Tensor | None = None):
    """tdc_step with the NVFP4-compressed cache (R16). SKIP: x_out = x_in + dq(cache).
    REFRESH: stats vs dq(cache), cache <- NVFP4(x_out - x_in; g_new), amax |d| -> amax_out."""
    m, h = x_in.shape
    c = cache.c()
    L.check("tdc_step_nvfp4", L.lib().tdc_step_nvfp4(mode, _ptr(x_in), _ptr(x_out), ctypes.byref(c), _ptr(g_new),
                                                     _ptr(amax_out), m, h, _ptr(stats_out), _ptr(workspace),
                                                     _stream(x_in.device)))


def tdc_delta_amax(x_in: torch.Tensor, x_out: torch.Tensor, amax_out: torch.Tensor):
    """max |x_out - x_in| max-reduced into amax_out (bootstraps a compressed cache's scale)."""
    m, h = x_in.shape
    L.check("tdc_delta_amax", L.lib().tdc_delta_amax(_ptr(x_in), _ptr(x_out), m, h, _ptr(amax_out),
                                                     _stream(x_in.device)))


def tdc_new_state() -> L.TdcState:
    st = L.TdcState()
    L.lib().tdc_init(ctypes.byref(st))
    return st


def tdc_decide(st: L.TdcState, cfg: L.TdcConfig, t: int) -> int:
    return int(L.lib().tdc_decide(ctypes.byref(st), ctypes.byref(cfg), t))


def tdc_update(st: L.TdcState, cfg: L.TdcConfig, t: int, decision: int, stats=None) -> None:
    g = None if stats is None else (stats if isinstance(stats, L.BlockStats) else L.BlockStats.from_seq(stats))
    L.lib().tdc_update(ctypes.byref(st), ctypes.byref(cfg), t, decision, None if g is None else ctypes.byref(g))
