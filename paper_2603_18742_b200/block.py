"""Synthetic video-DiT block stack driven through libdmpq.

One block = the six DMPQ linear layers of a DiT block (attention Q/K/V/O
projections and the two FFN layers) with minimal glue:

    h  = LN(X_in)                       (fused into the quantizer)
    q, k, v = Q(h), K(h), V(h)          (one shared quantized h per format)
    a  = v                              (attention stand-in: attention is out of scope)
    X_mid = X_in + g1 * O(a)            (gated residual fused in O's epilogue)
    h2 = LN(X_mid)                      (fused into the quantizer)
    f  = GELU_tanh(FFN1(h2))            (fused epilogue)
    X_out = X_mid + g2 * FFN2(f)        (fused epilogue)

wrapped by the paper's per-step control:
  - TDC (Eqs. 10-11): Skip -> X_out = X_in + Delta_tp (tdc_step SKIP);
    Compute -> run the block, then tdc_step REFRESH (Delta, FP64 statistics);
  - DMPQ routing (Eq. 7): per-layer NVFP4 / INT8 from the block's
    Gamma_{t-1} (dmpq_predict), NVFP4 global scales from the previous step's amax
    (delayed policy, R3).
Token sharding (shard.py): each rank owns a contiguous row range; the per-step
statistics and maxima are combined across ranks with ONE slot-packed SUM all-reduce
(an exact all-gather), after which every rank takes identical decisions.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import dmpq as D
from . import synth
from .shard import SlotBuffer, combine_host, exchange_device

LAYERS = ("q", "k", "v", "o", "ffn1", "ffn2")
NVTX = os.environ.get("DMPQ_NVTX") == "1"   # NVTX ranges per step and block (for nsys / ncu range filters)
N_STATS = L.STATS_LEN + 4      # per block: 7 TDC/predictor sums + sum|x| of the 4 layer inputs (PDR, R15)
SLOT_OF_LAYER = (0, 0, 0, 1, 2, 3)   # activation tensor each layer consumes
N_SLOTS = 4


def default_tau_gamma(tau_rel: float = 0.0025, beta: float = 0.001):
    """Per-layer thresholds from synthetic calibration slopes alpha_j = 0.1 (1 + j/2)
    through Eq. 6 (tau_rel, beta as stated; the paper's single-threshold setting
    tau_Gamma = 0.015 is layer 0)."""
    return [D.dmpq_derive_tau(0.1 * (1 + j / 2), beta, tau_rel) for j in range(len(LAYERS))]


@dataclass
class BlockWeights:
    layers: list            # 6 PackedWeights (Q, K, V are views into qkv)
    g1: torch.Tensor        # [H] fp32 gate of the attention residual
    g2: torch.Tensor        # [H] fp32 gate of the FFN residual
    qkv: D.PackedWeights = None   # Q, K, V side by side (one GEMM when they share a format)

    def nbytes(self):
        return sum(w.nbytes() for w in self.layers)


def make_block_weights(H: int, F: int, seed: int, device, gate_scale: float, hadamard: bool = False,
                       keep_bf16: bool = False, fuse_qkv: bool = True, int8_resident: bool = True) -> BlockWeights:
    shapes = [(H, H), (H, H), (H, H), (H, H), (F, H), (H, F)]
    layers = []
    for j, (n, k) in enumerate(shapes):
        if torch.device(device).type == "cuda" and n * k > 4_000_000:
            w, b = synth.linear_weight_device(n, k, seed * 16 + j, device)
        else:
            w, b = synth.linear_weight(n, k, seed * 16 + j)
        layers.append(D.dmpq_pack_weights(w.to(device), b.to(device), hadamard=hadamard, keep_bf16=keep_bf16,
                                          int8_resident=int8_resident))
        if not keep_bf16:
            del w
    qkv = None
    if fuse_qkv:   # needs H % 128 == 0 (whole scale-atom row tiles per layer)
        qkv, layers[0:3] = D.dmpq_concat_weights(layers[0:3])
    g = torch.Generator(device="cpu")
    g.manual_seed(seed * 16 + 15)
    g1 = (gate_scale * (0.5 + torch.rand(H, generator=g))).to(device)
    g2 = (gate_scale * (0.5 + torch.rand(H, generator=g))).to(device)
    return BlockWeights(layers, g1, g2, qkv)


class Workspace:
    """Activation buffers for one block evaluation of m rows (reused by every block)."""

    def __init__(self, m: int, H: int, F: int, device, g_table: torch.Tensor, int8_block: int = 0):
        self.m, self.H, self.F = m, H, F
        e = dict(dtype=torch.bfloat16, device=device)
        self.qkv = torch.empty(m, 3 * H, **e)    # Q | K | V outputs (Q, K unused by the stand-in attention)
        self.qk = self.qkv[:, :H]
        self.v = self.qkv[:, 2 * H:]             # strided view (row stride 3H): quantizer input only
        self.v_dense = torch.empty(m, H, **e)     # V when the O projection runs the BF16 GEMM (dense A, R15)
        self.x_mid = torch.empty(m, H, **e)
        self.f = torch.empty(m, F, **e)
        self.g_table = g_table                     # [n_blocks, 4] fp32 NVFP4 global scales
        self.acts = {}
        for slot, k in enumerate((H, H, H, F)):
            self.acts[(slot, D.FMT_INT8)] = D.QuantAct.empty(D.FMT_INT8, m, k, device, scale_block=int8_block)
            self.acts[(slot, D.FMT_NVFP4)] = D.QuantAct.empty(D.FMT_NVFP4, m, k, device, g=g_table[0, slot:slot + 1])
        self.tdc_ws = torch.zeros(D.tdc_workspace_bytes(m, H), dtype=torch.uint8, device=device)
        # fused refresh in the FFN2 epilogue (zero-filled once; the kernel resets its counter)
        self.tdc_gemm_ws = torch.zeros(D.dmpq_gemm_tdc_workspace_bytes(), dtype=torch.uint8, device=device)
        self.h1 = torch.empty(m, H, **e)          # LN outputs, materialised only for BF16-routed layers (R15)
        self.h2 = torch.empty(m, H, **e)

    def act(self, slot: int, fmt: int, block: int) -> D.QuantAct:
        a = self.acts[(slot, fmt)]
        if fmt == D.FMT_NVFP4:
            # point the activation's global scale at this block's slot of the g table
            a.g = self.g_table[block, slot:slot + 1]
            a.c.g = a.g.data_ptr()
        return a


@dataclass
class StepRecord:
    t: int
    decisions: list = field(default_factory=list)   # per block: 0 compute / 1 skip
    fmts: list = field(default_factory=list)        # per block: list of 6 formats (None if skipped)
    gammas: list = field(default_factory=list)
    linear_flops: float = 0.0


class DiTStack:
    """n_blocks synthetic DiT blocks on this rank's m_local token rows."""

    def __init__(self, n_blocks: int, H: int, F: int, m_local: int, device, seed: int = 0,
                 tdc_cfg=(0.001, 0.003, 2), tau_gamma=None, gate_scales=None, tdc_enabled: bool = True,
                 force_fmt: int | None = None, group=None, hadamard: bool = False, pdr: bool = False,
                 tau_outlier: float = 25.0, m_total: int | None = None, cache_nvfp4: bool = False,
                 fuse_refresh: bool = False, fuse_qkv: bool = True, int8_cast: bool = False, int8_block: bool = False,
                 fuse_quant: bool = False, overlap_refresh: bool = False, g_policy: str = "delayed"):
        self.nb, self.H, self.F, self.m = n_blocks, H, F, m_local
        self.device = torch.device(device)
        self.cfg = L.TdcConfig(*tdc_cfg)
        self.tau = tau_gamma if tau_gamma is not None else default_tau_gamma()
        self.tdc_enabled = tdc_enabled
        self.force_fmt = force_fmt
        self.group = group
        self.hadamard = hadamard      # online block-Hadamard smoothing (R14)
        # Purified Cache Refresh outlier gate: True / "delayed" = R from the block's last
        # computed step over all ranks, decided on the host (R15); "current" = R of this step's
        # layer input, decided on the device, both GEMM kinds enqueued and predicated (R18)
        self.pdr = bool(pdr)
        self.pdr_current = pdr == "current"
        self.tau_outlier = tau_outlier
        self.cache_nvfp4 = cache_nvfp4  # NVFP4-compressed delta cache (R16)
        # bf16 cache, optional: the TDC refresh runs in the FFN2 GEMM's epilogue (
        # measured slower than the streaming refresh kernel)
        self.fuse_refresh = fuse_refresh and not cache_nvfp4
        self.fuse_qkv = fuse_qkv      # one Q|K|V GEMM when the three layers share a format
        self.m_total = m_total if m_total is not None else m_local
        # P:184's residency: weights NVFP4 only, INT8 codes cast on the fly per INT8 GEMM into one
        # shared scratch (NEXT-4b; dmpq_cast_int8)
        self.int8_cast = int8_cast
        # per-block symmetric INT8 activations over the 128-element Hadamard blocks (R17,
        # NEXT-1) instead of per-token INT8 (R2); needs the Hadamard option
        if int8_block and not hadamard:
            raise ValueError("per-block INT8 (R17) is defined on the Hadamard blocks: needs hadamard=True")
        self.int8_block = int8_block
        # NVFP4 per-tensor scale (R3): "delayed" = max(fl(amax_{t-1}/1344), FLT_MIN) from the previous
        # step's (all-rank) amax, the default; "current" = an amax-only pass over this input first,
        # then max(fl(amax/2688), FLT_MIN) -- one extra read of each NVFP4-quantized tensor, and a
        # per-tensor cross-rank maximum inside the block under sharding, so single-rank only
        if g_policy not in ("delayed", "current"):
            raise ValueError("g_policy must be 'delayed' or 'current'")
        if g_policy == "current" and group is not None and torch.distributed.get_world_size(group) > 1:
            raise ValueError("g_policy='current' is single-rank (it needs a cross-rank max per NVFP4 tensor)")
        self.g_policy = g_policy
        # producer-fused quantization (NEXT-2): FFN1's epilogue writes the NVFP4 codes of the
        # FFN2 input directly (no bf16 f round trip, no standalone quantizer) when FFN2 is routed
        # NVFP4; built for the plain quantizer (the Hadamard blocks do not fit the epilogue, DESIGN 5.7)
        # (not with the "current" g policy: FFN2's global scale would need f's amax before f exists)
        self.fuse_quant = fuse_quant and not hadamard and not pdr and g_policy == "delayed"
        if gate_scales is None:
            gate_scales = [0.004 * (1 + (b % 5)) for b in range(n_blocks)]
        self.blocks = [make_block_weights(H, F, seed * 1000 + b, self.device, gate_scales[b], hadamard, keep_bf16=pdr,
                                          fuse_qkv=fuse_qkv, int8_resident=not int8_cast) for b in range(n_blocks)]
        self.i8_scratch = torch.empty(max(3 * H * H, F * H) if int8_cast else 0, dtype=torch.int8, device=self.device)
        self.g_table = torch.ones(n_blocks, N_SLOTS, dtype=torch.float32, device=self.device)
        self.g_cur_amax = torch.zeros(n_blocks, N_SLOTS, dtype=torch.float32, device=self.device)
        # one buffer for the per-step MAX all-reduce: [0] amax of the quantised values (NVFP4 global
        # scales, R3); [1] max|x| of the layer inputs (PDR, R15); then max|d| of each block's last
        # refresh (compressed delta cache, R16; kept across steps: skipped blocks do not refresh)
        self.amax_all = torch.zeros(2 * n_blocks * N_SLOTS + n_blocks, dtype=torch.float32, device=self.device)
        self.amax = self.amax_all[:2 * n_blocks * N_SLOTS].view(2, n_blocks, N_SLOTS)
        self.delta_amax = self.amax_all[2 * n_blocks * N_SLOTS:]
        self.g_delta = torch.zeros(n_blocks, dtype=torch.float32, device=self.device)
        self.row_abs = torch.zeros(n_blocks * N_SLOTS, m_local, dtype=torch.float32, device=self.device)
        self.ws = Workspace(m_local, H, F, self.device, self.g_table, int8_block=128 if int8_block else 0)
        if cache_nvfp4:
            self.delta = [D.DeltaCacheNvfp4(m_local, H, self.device) for _ in range(n_blocks)]
        else:
            self.delta = [torch.zeros(m_local, H, dtype=torch.bfloat16, device=self.device) for _ in range(n_blocks)]
        world = 1 if group is None else torch.distributed.get_world_size(group)
        self.world = world
        self.rank = 0 if group is None else torch.distributed.get_rank(group)
        # the per-step exchange buffer: this rank's FP64 statistics and fp32 maxima in its own slot,
        # one SUM all-reduce per step (shard.py)
        self.slots = SlotBuffer(world, self.rank, n_blocks * N_STATS, self.amax_all.numel(), self.device)
        self.stats_slots = self.slots.stats.view(world, n_blocks, N_STATS)
        self.ratio = [None] * n_blocks          # PDR outlier ratio per slot from the block's last compute
        # TDC refresh of block b on a side stream, overlapped with block b + 1 (it only reads block b's
        # input and output, which a ring of three activation buffers keeps alive until block b + 2;
        # joined at the end of the step). bf16 cache, separate refresh kernel only. Off by default:
        # measured step time unchanged (104.6 vs 104.6 ms; the power-capped step does the same work).
        self.overlap_refresh = overlap_refresh and not cache_nvfp4 and not self.fuse_refresh
        self.x_buf = [torch.empty(m_local, H, dtype=torch.bfloat16, device=self.device)
                      for _ in range(3 if self.overlap_refresh else 2)]
        self.refresh_stream = torch.cuda.Stream(device=self.device) if self.overlap_refresh else None
        self.refresh_graphs = [None] * n_blocks
        self.ev_out = [torch.cuda.Event() for _ in range(n_blocks)] if self.overlap_refresh else None
        self.ev_refreshed = [torch.cuda.Event() for _ in range(n_blocks)] if self.overlap_refresh else None
        self.tdc = [D.tdc_new_state() for _ in range(n_blocks)]
        self.prev_stats = [None] * n_blocks     # global stats of the block's last step (None if skipped)
        self.prev_skipped = [False] * n_blocks
        self.records: list[StepRecord] = []
        self.launches = 0                       # libdmpq kernel launches issued (bench's gpu_launches)
        self.timing = False                     # record CUDA events around every GEMM (roofline)
        self.kernel_events = {"quantize": [], "tdc": [], "exchange": [], "cast": []}   # breakdown of the step
        self.hbm_bytes = {"quantize": 0.0, "tdc": 0.0, "cast": 0.0}   # algorithmic HBM bytes of those kernels (timing passes)
        self.gemm_events = {D.FMT_INT8: [], D.FMT_NVFP4: [], D.FMT_BF16: []}
        self.gemm_flops = {D.FMT_INT8: 0.0, D.FMT_NVFP4: 0.0, D.FMT_BF16: 0.0}
        self.capture = None                     # dict -> per-stage clones for the parity tests
        # CUDA graphs: one per (block, decision, formats) pattern, captured on first use and
        # replayed afterwards (pointers are static per block; the step input is copied into x_in0)
        self.use_graphs = False
        self.graphs = [dict() for _ in range(n_blocks)]
        self.graph_pool = None
        self.x_in0 = torch.empty(m_local, H, dtype=torch.bfloat16, device=self.device)
        self.pdr_sums = torch.zeros(n_blocks * N_SLOTS, dtype=torch.float64, device=self.device)
        self.pdr_flags = torch.zeros(n_blocks, N_SLOTS, dtype=torch.int32, device=self.device)   # R18 device gate

    def _cap(self, key, t):
        if self.capture is not None:
            self.capture[key] = t.detach().clone()

    def _cap_act(self, key, a):
        if self.capture is not None and a is not None:
            d = {"codes": a.codes.clone()}
            if a.fmt == D.FMT_NVFP4:
                d.update(sf=a.sf.clone(), g=a.g.clone())
            else:
                d.update(row_scale=a.row_scale.clone())
            self.capture[key] = d

    # ------------------------------------------------------------------ one block
    def _ev(self, kind):
        """Context manager: CUDA events around a region when timing is on (breakdown)."""
        stack = self

        class _C:
            def __enter__(self_):
                if stack.timing:
                    self_.s = torch.cuda.Event(enable_timing=True)
                    self_.s.record()

            def __exit__(self_, *a):
                if stack.timing:
                    e = torch.cuda.Event(enable_timing=True)
                    e.record()
                    stack.kernel_events[kind].append((self_.s, e))
        return _C()

    def breakdown_s(self):
        return {k: sum(s.elapsed_time(e) for s, e in v) * 1e-3 for k, v in self.kernel_events.items()}

    def _quant(self, b, slot, src, fmts_needed, layernorm=False, h_buf=None):
        """Quantize one activation tensor into the formats its consumers need (plus PDR
        statistics); returns {fmt: QuantAct} with FMT_BF16 -> the bf16 tensor itself."""
        with self._ev("quantize"):
            return self._quant_impl(b, slot, src, fmts_needed, layernorm, h_buf)

    def _quant_impl(self, b, slot, src, fmts_needed, layernorm, h_buf):
        ws = self.ws
        want_h = layernorm and (D.FMT_BF16 in fmts_needed or self.capture is not None or self.pdr_current)
        a8 = ws.act(slot, D.FMT_INT8, b) if D.FMT_INT8 in fmts_needed else None
        a4 = ws.act(slot, D.FMT_NVFP4, b) if D.FMT_NVFP4 in fmts_needed else None
        if a4 is not None and self.g_policy == "current":   # R3 "current": amax pass, then g from it
            am = self.g_cur_amax[b, slot:slot + 1]
            am.zero_()
            D.dmpq_quantize_act(src, amax_out=am, layernorm=layernorm, hadamard=self.hadamard)
            D.dmpq_global_scale(am, 2688.0, self.g_table[b, slot:slot + 1])
            if self.timing:
                self.hbm_bytes["quantize"] += 2 * src.numel()
        D.dmpq_quantize_act(src, out_i8=a8, out_fp4=a4, amax_out=self.amax[0, b, slot:slot + 1], layernorm=layernorm,
                            h_out=h_buf if want_h else None, hadamard=self.hadamard,
                            row_abs_sum=self.row_abs[b * N_SLOTS + slot] if self.pdr else None,
                            amax_in=self.amax[1, b, slot:slot + 1] if self.pdr else None)
        if self.timing:   # algorithmic HBM bytes of this launch (the bench's in-step quantizer GB/s)
            m, k = src.shape
            nb = 2 * m * k + (2 * m * k if want_h else 0)
            if a4 is not None:
                nb += m * k // 2 + m * k // 16
            if a8 is not None:
                nb += m * k + 4 * (m * k // 128 if a8.scale_block else m)
            self.hbm_bytes["quantize"] += nb
        out = {D.FMT_INT8: a8, D.FMT_NVFP4: a4}
        if D.FMT_BF16 in fmts_needed:
            out[D.FMT_BF16] = D.QuantAct.bf16(h_buf if layernorm else src)
        return out

    def _gate(self, b, slot, k):
        """R18: this step's outlier ratio of the slot's input on the device -> pdr_flags[b, slot]."""
        with self._ev("quantize"):
            D.dmpq_outlier_gate(self.row_abs[b * N_SLOTS + slot], self.amax[1, b, slot:slot + 1], float(self.m * k),
                                self.tau_outlier, self.pdr_flags[b, slot:slot + 1])

    def _gemm_gated(self, b, slot, q, fmt, w, **kw):
        """Both GEMM kinds of one layer, predicated on the device gate (R18): the quantized one
        runs iff pdr_flags[b, slot] == 0, the BF16 one iff it is 1."""
        flag = self.pdr_flags[b, slot:slot + 1]
        self._gemm(q[fmt], w, run_if=flag, run_if_value=0, **kw)
        self._gemm(q[D.FMT_BF16], w, run_if=flag, run_if_value=1, **kw)

    def _compute_block_current(self, b: int, x_in: torch.Tensor, x_out: torch.Tensor, fmts) -> float:
        """One block with the current-input PDR gate (R18): each layer input's quantizer
        also writes the statistics (and the dense bf16 input), a one-CTA kernel takes the BF16 /
        quantized decision on the device, and both GEMM kinds are enqueued, predicated on it."""
        W, ws, H, F = self.blocks[b], self.ws, self.H, self.F
        q0 = self._quant(b, 0, x_in, set(fmts[0:3]) | {D.FMT_BF16}, layernorm=True, h_buf=ws.h1)
        self._gate(b, 0, H)
        if self.capture is not None:
            self._cap("x_in", x_in); self._cap("h1", ws.h1)
            self._cap_act("a0_i8", q0[D.FMT_INT8]); self._cap_act("a0_f4", q0[D.FMT_NVFP4])
        for j, out in ((0, ws.qk), (1, ws.qkv[:, H:2 * H]), (2, ws.v_dense)):   # V dense: O may run BF16
            self._gemm_gated(b, 0, q0, fmts[j], W.layers[j], Y=out)
            self._cap(f"y{j}", out)
        q1 = self._quant(b, 1, ws.v_dense, {fmts[3], D.FMT_BF16})
        self._gate(b, 1, H)
        self._cap_act("a1", q1[fmts[3]])
        self._gemm_gated(b, 1, q1, fmts[3], W.layers[3], Y=ws.x_mid, residual=x_in, gate=W.g1)
        self._cap("x_mid", ws.x_mid)
        q2 = self._quant(b, 2, ws.x_mid, {fmts[4], D.FMT_BF16}, layernorm=True, h_buf=ws.h2)
        self._gate(b, 2, H)
        self._cap("h2", ws.h2)
        self._cap_act("a2", q2[fmts[4]])
        self._gemm_gated(b, 2, q2, fmts[4], W.layers[4], Y=ws.f, gelu=True)
        self._cap("f", ws.f)
        q3 = self._quant(b, 3, ws.f, {fmts[5], D.FMT_BF16})
        self._gate(b, 3, F)
        self._cap_act("a3", q3[fmts[5]])
        self._gemm_gated(b, 3, q3, fmts[5], W.layers[5], Y=x_out, residual=ws.x_mid, gate=W.g2)
        self._cap("x_out", x_out)
        return 2.0 * self.m * (4 * H * H + 2 * H * F)

    def _compute_block(self, b: int, x_in: torch.Tensor, x_out: torch.Tensor, fmts, refresh_stats=None) -> float:
        if self.pdr_current:
            return self._compute_block_current(b, x_in, x_out, fmts)
        W, ws, H, F, m = self.blocks[b], self.ws, self.H, self.F, self.m
        cap = self.capture is not None
        # attention input: LN fused into the quantizer, one pass for every format Q/K/V need
        q0 = self._quant(b, 0, x_in, set(fmts[0:3]), layernorm=True, h_buf=ws.h1)
        if cap:
            self._cap("x_in", x_in); self._cap("h1", ws.h1)
            self._cap_act("a0_i8", q0[D.FMT_INT8]); self._cap_act("a0_f4", q0[D.FMT_NVFP4])
        # the BF16 GEMM reads its A operand densely (row stride k): a BF16-routed O projection
        # gets V in its own buffer instead of the strided Q|K|V view
        v = ws.v_dense if fmts[3] == D.FMT_BF16 else ws.v
        if self.fuse_qkv and fmts[0] == fmts[1] == fmts[2] and v is ws.v:
            # one GEMM over the side-by-side Q | K | V weights (per-layer NVFP4 g_w per column)
            self._gemm(q0[fmts[0]], W.qkv, Y=ws.qkv)
            for j in range(3):
                self._cap(f"y{j}", ws.qkv[:, j * H:(j + 1) * H])
        else:
            for j, out in ((0, ws.qk), (1, ws.qkv[:, H:2 * H]), (2, v)):
                self._gemm(q0[fmts[j]], W.layers[j], Y=out)
                self._cap(f"y{j}", out)
        # O projection on the attention stand-in a = v, gated residual in the epilogue
        q1 = self._quant(b, 1, v, {fmts[3]})
        if fmts[3] != D.FMT_BF16:
            self._cap_act("a1", q1[fmts[3]])
        self._gemm(q1[fmts[3]], W.layers[3], Y=ws.x_mid, residual=x_in, gate=W.g1)
        self._cap("x_mid", ws.x_mid)
        # FFN
        q2 = self._quant(b, 2, ws.x_mid, {fmts[4]}, layernorm=True, h_buf=ws.h2)
        if cap:
            self._cap("h2", ws.h2)
            if fmts[4] != D.FMT_BF16:
                self._cap_act("a2", q2[fmts[4]])
        if self.fuse_quant and fmts[5] == D.FMT_NVFP4:
            a3 = ws.act(3, D.FMT_NVFP4, b)
            self._gemm(q2[fmts[4]], W.layers[4], Y=ws.f if cap else None, gelu=True, quant_out=a3,
                       quant_amax=self.amax[0, b, 3:4])
            q3 = {D.FMT_NVFP4: a3}
        else:
            self._gemm(q2[fmts[4]], W.layers[4], Y=ws.f, gelu=True)
            q3 = None
        self._cap("f", ws.f)
        if q3 is None:
            q3 = self._quant(b, 3, ws.f, {fmts[5]})
        if fmts[5] != D.FMT_BF16:
            self._cap_act("a3", q3[fmts[5]])
        tdc = {}
        if refresh_stats is not None:   # fused TDC refresh of X_out (Eq. 8) in this epilogue
            tdc = dict(tdc_x_in=x_in, tdc_delta=self.delta[b], tdc_stats=refresh_stats, tdc_workspace=ws.tdc_gemm_ws)
        self._gemm(q3[fmts[5]], W.layers[5], Y=x_out, residual=ws.x_mid, gate=W.g2, **tdc)
        self._cap("x_out", x_out)
        return 2.0 * m * (4 * H * H + 2 * H * F)

    def _gemm(self, a, w, **kw):
        if a.fmt == D.FMT_INT8 and self.int8_cast:   # rebuild this layer's INT8 codes from its NVFP4 form
            with self._ev("cast"):
                w = D.dmpq_cast_int8(w, self.i8_scratch)
            if self.timing:   # NVFP4 codes + scales read, INT8 codes written
                self.hbm_bytes["cast"] += 1.5625 * w.n * w.k
        if self.timing:
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            D.dmpq_gemm(a, w, **kw)
            e.record()
            self.gemm_events[a.fmt].append((s, e))
            self.gemm_flops[a.fmt] += 2.0 * a.m * w.n * w.k
        else:
            D.dmpq_gemm(a, w, **kw)

    def gemm_time_s(self):
        """Sum of the recorded GEMM durations per format (seconds) and launch counts."""
        out = {}
        for f, evs in self.gemm_events.items():
            out[f] = (sum(s.elapsed_time(e) for s, e in evs) * 1e-3, len(evs))
        return out

    def reset_timing(self):
        self.hbm_bytes = {"quantize": 0.0, "tdc": 0.0, "cast": 0.0}
        self.kernel_events = {"quantize": [], "tdc": [], "exchange": [], "cast": []}
        self.gemm_events = {D.FMT_INT8: [], D.FMT_NVFP4: [], D.FMT_BF16: []}
        self.gemm_flops = {D.FMT_INT8: 0.0, D.FMT_NVFP4: 0.0, D.FMT_BF16: 0.0}

    # ------------------------------------------------------------------ one timestep
    def reset_state(self):
        """Back to t = 0: TDC states, routing history, caches, global scales."""
        for bi in range(self.nb):
            self.tdc[bi] = D.tdc_new_state()
            self.prev_stats[bi] = None
            self.prev_skipped[bi] = False
            self.ratio[bi] = None
            if self.cache_nvfp4:
                for t_ in (self.delta[bi].codes, self.delta[bi].sf, self.delta[bi].g):
                    t_.zero_()
            else:
                self.delta[bi].zero_()
        self.g_table.fill_(1.0)
        self.amax_all.zero_()
        self.g_delta.zero_()
        self.records = []

    def _tdc_bytes(self, refresh: bool):
        if self.timing:   # refresh: X_in, X_out, Delta_prev read + Delta_new written; skip: X_in, Delta read + X_out
            self.hbm_bytes["tdc"] += (8 if refresh else 6) * self.m * self.H if not self.cache_nvfp4 else \
                (4 + 2 * 0.5625 if refresh else 4.5625) * self.m * self.H

    def _refresh(self, b, x_in, x_out):
        """tdc_step(REFRESH) of block b (bf16 cache): Delta_b, the block's FP64 statistics."""
        self._tdc_bytes(True)
        with self._ev("tdc"):
            D.tdc_step(L.TDC_REFRESH, x_in, x_out, self.delta[b], self.stats_slots[self.rank, b, :L.STATS_LEN],
                       self.ws.tdc_ws)

    def _block_work(self, b, x_in, x_out, d, fmts, first=False, refresh=True):
        """Enqueue one block's kernels (capturable: no host sync, no allocation). refresh=False leaves
        a computed block's TDC refresh to the caller (overlapped on the side stream)."""
        if d == L.TDC_DECIDE_SKIP:
            self._tdc_bytes(False)
            with self._ev("tdc"):
                if self.cache_nvfp4:
                    D.tdc_step_nvfp4(L.TDC_SKIP, x_in, x_out, self.delta[b])
                else:
                    D.tdc_step(L.TDC_SKIP, x_in, x_out, self.delta[b])
            return 0.0
        st = self.stats_slots[self.rank, b, :L.STATS_LEN]
        if self.fuse_refresh:
            return self._compute_block(b, x_in, x_out, fmts, refresh_stats=st)
        flops = self._compute_block(b, x_in, x_out, fmts)
        if not refresh:
            return flops
        self._tdc_bytes(True)
        with self._ev("tdc"):
            if self.cache_nvfp4:
                am, g = self.delta_amax[b:b + 1], self.g_delta[b:b + 1]
                am.zero_()
                if first:   # no previous refresh: bootstrap the cache's global scale from the current amax
                    D.tdc_delta_amax(x_in, x_out, am)
                    D.dmpq_global_scale(am, 1344.0, g)
                D.tdc_step_nvfp4(L.TDC_REFRESH, x_in, x_out, self.delta[b], g_new=g, amax_out=am, stats_out=st,
                                 workspace=self.ws.tdc_ws)
            else:
                D.tdc_step(L.TDC_REFRESH, x_in, x_out, self.delta[b], st, self.ws.tdc_ws)
        return flops

    def step(self, x0: torch.Tensor, t: int) -> torch.Tensor:
        """Run all blocks at timestep t on this rank's rows; returns the last output
        (a view of an internal buffer). Call end_step(t) afterwards."""
        rec = StepRecord(t)
        self.amax.zero_()
        self.slots.zero_()
        graphs = self.use_graphs and not self.timing and self.capture is None
        overlap = self.overlap_refresh and self.capture is None
        if graphs and x0.data_ptr() != self.x_in0.data_ptr():
            self.x_in0.copy_(x0)
            x0 = self.x_in0
        x_in = x0
        main = torch.cuda.current_stream(self.device)
        if overlap:   # this step's refreshes start after the statistics slots were zeroed
            self.refresh_stream.wait_stream(main)
        pending = set()   # blocks whose refresh of this step was enqueued on the side stream
        if NVTX:
            torch.cuda.nvtx.range_push(f"dmpq step t={t}")
        for b in range(self.nb):
            if NVTX:
                if b:
                    torch.cuda.nvtx.range_pop()
                torch.cuda.nvtx.range_push(f"block {b}")
            x_out = self.x_buf[b % len(self.x_buf)]
            if overlap and (b - 2) in pending:   # block b overwrites the buffers refresh(b - 2) reads
                main.wait_event(self.ev_refreshed[b - 2])
            d = D.tdc_decide(self.tdc[b], self.cfg, t) if self.tdc_enabled else L.TDC_COMPUTE
            fmts, gamma = None, float("nan")
            if d != L.TDC_DECIDE_SKIP:
                if self.force_fmt is not None:
                    fmts = [self.force_fmt] * 6
                else:
                    fmts, gamma, _ = D.dmpq_predict(self.prev_stats[b], self.tau, t, self.prev_skipped[b])
                    if self.pdr_current:   # post-skip INT8 now; the BF16 choice is taken on the device (R18)
                        fmts = D.dmpq_purify(fmts, None, self.prev_skipped[b], self.tau_outlier)
                    elif self.pdr and self.ratio[b] is not None:
                        fmts = D.dmpq_purify(fmts, [self.ratio[b][s] for s in SLOT_OF_LAYER], self.prev_skipped[b],
                                             self.tau_outlier)
            first = self.cache_nvfp4 and d != L.TDC_DECIDE_SKIP and self.tdc[b].n_computed == 0
            if graphs:
                key = (d, None if fmts is None else tuple(fmts), first)
                g = self.graphs[b].get(key)
                if g is None:
                    # capture on a side stream without a device-wide sync (torch.cuda.graph's
                    # context manager synchronises; this runs mid-step on first use of a pattern)
                    if self.graph_pool is None:
                        L.check("dmpq_prepare", L.lib().dmpq_prepare())
                        self.graph_pool = torch.cuda.graph_pool_handle()
                        self.capture_stream = torch.cuda.Stream(device=self.device)
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.stream(self.capture_stream):
                        g.capture_begin(pool=self.graph_pool)
                        self._block_work(b, x_in, x_out, d, fmts, first, refresh=not overlap)
                        g.capture_end()
                    self.graphs[b][key] = g
                g.replay()
                flops = 0.0 if d == L.TDC_DECIDE_SKIP else 2.0 * self.m * (4 * self.H * self.H + 2 * self.H * self.F)
            else:
                flops = self._block_work(b, x_in, x_out, d, fmts, first, refresh=not overlap)
            if overlap and d != L.TDC_DECIDE_SKIP:   # the refresh of block b on the side stream
                self.ev_out[b].record(main)
                rs = self.refresh_stream
                rs.wait_event(self.ev_out[b])
                with torch.cuda.stream(rs):
                    if graphs:
                        if self.refresh_graphs[b] is None:
                            g = torch.cuda.CUDAGraph()
                            with torch.cuda.stream(self.capture_stream):
                                g.capture_begin(pool=self.graph_pool)
                                self._refresh(b, x_in, x_out)
                                g.capture_end()
                            self.refresh_graphs[b] = g
                        self.refresh_graphs[b].replay()
                    else:
                        self._refresh(b, x_in, x_out)
                    self.ev_refreshed[b].record(rs)
                pending.add(b)
            if d == L.TDC_DECIDE_SKIP:
                self.launches += 1
            else:   # 4 quantizers + 6 GEMMs + refresh, fewer when fused, +2 for a cache bootstrap
                qkv1 = self.fuse_qkv and fmts[0] == fmts[1] == fmts[2] and fmts[3] != D.FMT_BF16 and not self.pdr_current
                self.launches += 11 - (1 if self.fuse_refresh else 0) - (2 if qkv1 else 0) + (2 if first else 0)
                if self.fuse_quant and fmts[5] == D.FMT_NVFP4:   # FFN2's quantizer runs inside FFN1
                    self.launches -= 1
                if self.pdr_current:   # + 4 device gates + the predicated-off GEMM of every layer
                    self.launches += 4 + 6
                if self.g_policy == "current":   # amax pass + global scale per NVFP4-quantized input
                    nv = [any(f == D.FMT_NVFP4 for f in fmts[0:3]), fmts[3] == D.FMT_NVFP4, fmts[4] == D.FMT_NVFP4,
                          fmts[5] == D.FMT_NVFP4]
                    self.launches += 2 * sum(nv)
                if self.int8_cast:   # one cast per INT8 GEMM launch
                    i8 = [f == D.FMT_INT8 for f in fmts]
                    self.launches += (int(i8[0]) if qkv1 else sum(i8[0:3])) + sum(i8[3:6])
            rec.linear_flops += flops
            rec.fmts.append(None if d == L.TDC_DECIDE_SKIP else fmts)
            rec.gammas.append(gamma)
            rec.decisions.append(d)
            x_in = x_out
        if overlap:   # join: the exchange and the next step see every refresh
            main.wait_stream(self.refresh_stream)
        if NVTX:
            if self.nb:
                torch.cuda.nvtx.range_pop()
            torch.cuda.nvtx.range_pop()
        self.records.append(rec)
        return x_in

    def end_step(self, t: int):
        """Per-step exchange + host decisions: combine the statistics and maxima of all ranks
        (one slot-packed SUM all-reduce = exact all-gather), copy them to the host once,
        update TDC (Eq. 10) and the NVFP4 global scales (R3)."""
        with self._ev("exchange"):
            if self.pdr:   # per-slot sum|x| of this rank's rows -> its stats slot (FP64, fixed order)
                D.dmpq_outlier_reduce(self.row_abs, self.pdr_sums)
                self.stats_slots[self.rank, :, L.STATS_LEN:] = self.pdr_sums.view(self.nb, N_SLOTS)
                self.launches += 1
            # one SUM all-reduce of the slot buffer (statistics + maxima): every rank then holds
            # every rank's partial sums and the global maxima
            exchange_device(self.slots, self.amax_all, self.group)
            # next step's NVFP4 global scales from the (all-rank) amax of this step (R3, delayed policy)
            if self.g_policy == "delayed":
                D.dmpq_global_scale(self.amax[0].view(-1), 1344.0, self.g_table.view(-1))
                self.launches += 1
            if self.cache_nvfp4:   # delta-cache scales for each block's next refresh (same delayed policy)
                D.dmpq_global_scale(self.delta_amax, 1344.0, self.g_delta)
                self.launches += 1
        # the D2H copy inside synchronises the stream (one exchange per step)
        stats = combine_host(self.slots).reshape(self.nb, N_STATS)
        if self.pdr:
            amax_in = self.amax[1].cpu().numpy().astype(np.float64)
        if self.pdr_current:   # the device gate's decisions of this step -> the step record
            flags = self.pdr_flags.cpu().numpy()
            rec = self.records[-1]
            for b in range(self.nb):
                if rec.fmts[b] is not None:
                    rec.fmts[b] = [D.FMT_BF16 if flags[b, SLOT_OF_LAYER[j]] else f for j, f in enumerate(rec.fmts[b])]
        rec = self.records[-1]
        for b in range(self.nb):
            d = rec.decisions[b]
            if d == L.TDC_DECIDE_SKIP:
                D.tdc_update(self.tdc[b], self.cfg, t, d, None)
                self.prev_stats[b] = None
                self.prev_skipped[b] = True
            else:
                st = L.BlockStats.from_seq(stats[b][:L.STATS_LEN])
                D.tdc_update(self.tdc[b], self.cfg, t, d, st)
                self.prev_stats[b] = st
                self.prev_skipped[b] = False
                if self.pdr:   # R = max|x| / mean|x| of each layer input over all tokens (R15)
                    ks = (self.H, self.H, self.H, self.F)
                    self.ratio[b] = [D.dmpq_outlier_ratio(amax_in[b, s], stats[b][L.STATS_LEN + s], self.m_total * ks[s])
                                     for s in range(N_SLOTS)]
        return stats

    def mix(self, records=None):
        """Realised NVFP4 / INT8 / skip mix over the given step records."""
        records = self.records if records is None else records
        n4 = n8 = n16 = sk = 0
        for r in records:
            for f in r.fmts:
                if f is None:
                    sk += 1
                else:
                    n4 += sum(1 for x in f if x == D.FMT_NVFP4)
                    n8 += sum(1 for x in f if x == D.FMT_INT8)
                    n16 += sum(1 for x in f if x == D.FMT_BF16)
        tot_layers = max(1, n4 + n8 + n16)
        nblk = max(1, sum(len(r.fmts) for r in records))
        return {"nvfp4_layer_frac": n4 / tot_layers, "int8_layer_frac": n8 / tot_layers,
                "bf16_layer_frac": n16 / tot_layers, "skip_block_frac": sk / nblk}
