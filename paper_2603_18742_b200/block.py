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
statistics are combined across ranks with one slot-packed SUM all-reduce (stats)
and one MAX all-reduce (amax), after which every rank takes identical decisions.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import dmpq as D
from . import synth
from .shard import exchange

LAYERS = ("q", "k", "v", "o", "ffn1", "ffn2")
SLOT_OF_LAYER = (0, 0, 0, 1, 2, 3)   # activation tensor each layer consumes
N_SLOTS = 4


def default_tau_gamma(tau_rel: float = 0.0025, beta: float = 0.001):
    """Per-layer thresholds from synthetic calibration slopes alpha_j = 0.1 (1 + j/2)
    through Eq. 6 (tau_rel, beta as stated; the paper's single-threshold setting
    tau_Gamma = 0.015 is layer 0)."""
    return [D.dmpq_derive_tau(0.1 * (1 + j / 2), beta, tau_rel) for j in range(len(LAYERS))]


@dataclass
class BlockWeights:
    layers: list            # 6 PackedWeights
    g1: torch.Tensor        # [H] fp32 gate of the attention residual
    g2: torch.Tensor        # [H] fp32 gate of the FFN residual

    def nbytes(self):
        return sum(w.nbytes() for w in self.layers)


def make_block_weights(H: int, F: int, seed: int, device, gate_scale: float, hadamard: bool = False) -> BlockWeights:
    shapes = [(H, H), (H, H), (H, H), (H, H), (F, H), (H, F)]
    layers = []
    for j, (n, k) in enumerate(shapes):
        if torch.device(device).type == "cuda" and n * k > 4_000_000:
            w, b = synth.linear_weight_device(n, k, seed * 16 + j, device)
        else:
            w, b = synth.linear_weight(n, k, seed * 16 + j)
        layers.append(D.dmpq_pack_weights(w.to(device), b.to(device), hadamard=hadamard))
        del w
    g = torch.Generator(device="cpu")
    g.manual_seed(seed * 16 + 15)
    g1 = (gate_scale * (0.5 + torch.rand(H, generator=g))).to(device)
    g2 = (gate_scale * (0.5 + torch.rand(H, generator=g))).to(device)
    return BlockWeights(layers, g1, g2)


class Workspace:
    """Activation buffers for one block evaluation of m rows (reused by every block)."""

    def __init__(self, m: int, H: int, F: int, device, g_table: torch.Tensor):
        self.m, self.H, self.F = m, H, F
        e = dict(dtype=torch.bfloat16, device=device)
        self.qk = torch.empty(m, H, **e)         # Q and K outputs (unused by the stand-in attention)
        self.v = torch.empty(m, H, **e)
        self.x_mid = torch.empty(m, H, **e)
        self.f = torch.empty(m, F, **e)
        self.g_table = g_table                     # [n_blocks, 4] fp32 NVFP4 global scales
        self.acts = {}
        for slot, k in enumerate((H, H, H, F)):
            self.acts[(slot, D.FMT_INT8)] = D.QuantAct.empty(D.FMT_INT8, m, k, device)
            self.acts[(slot, D.FMT_NVFP4)] = D.QuantAct.empty(D.FMT_NVFP4, m, k, device, g=g_table[0, slot:slot + 1])
        self.tdc_ws = torch.zeros(D.tdc_workspace_bytes(m, H), dtype=torch.uint8, device=device)

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
                 force_fmt: int | None = None, group=None, hadamard: bool = False):
        self.nb, self.H, self.F, self.m = n_blocks, H, F, m_local
        self.device = torch.device(device)
        self.cfg = L.TdcConfig(*tdc_cfg)
        self.tau = tau_gamma if tau_gamma is not None else default_tau_gamma()
        self.tdc_enabled = tdc_enabled
        self.force_fmt = force_fmt
        self.group = group
        self.hadamard = hadamard      # online block-Hadamard smoothing (R14)
        if gate_scales is None:
            gate_scales = [0.004 * (1 + (b % 5)) for b in range(n_blocks)]
        self.blocks = [make_block_weights(H, F, seed * 1000 + b, self.device, gate_scales[b], hadamard)
                       for b in range(n_blocks)]
        self.g_table = torch.ones(n_blocks, N_SLOTS, dtype=torch.float32, device=self.device)
        self.amax = torch.zeros(n_blocks, N_SLOTS, dtype=torch.float32, device=self.device)
        self.ws = Workspace(m_local, H, F, self.device, self.g_table)
        self.delta = [torch.zeros(m_local, H, dtype=torch.bfloat16, device=self.device) for _ in range(n_blocks)]
        world = 1 if group is None else torch.distributed.get_world_size(group)
        self.world = world
        self.rank = 0 if group is None else torch.distributed.get_rank(group)
        self.stats_slots = torch.zeros(world, n_blocks, L.STATS_LEN, dtype=torch.float64, device=self.device)
        self.x_buf = [torch.empty(m_local, H, dtype=torch.bfloat16, device=self.device) for _ in range(2)]
        self.tdc = [D.tdc_new_state() for _ in range(n_blocks)]
        self.prev_stats = [None] * n_blocks     # global stats of the block's last step (None if skipped)
        self.prev_skipped = [False] * n_blocks
        self.records: list[StepRecord] = []
        self.launches = 0                       # libdmpq kernel launches issued (bench's gpu_launches)
        self.timing = False                     # record CUDA events around every GEMM (roofline)
        self.gemm_events = {D.FMT_INT8: [], D.FMT_NVFP4: []}
        self.gemm_flops = {D.FMT_INT8: 0.0, D.FMT_NVFP4: 0.0}
        self.capture = None                     # dict -> per-stage clones for the parity tests

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
    def _compute_block(self, b: int, x_in: torch.Tensor, x_out: torch.Tensor, fmts) -> float:
        W, ws, H, F, m = self.blocks[b], self.ws, self.H, self.F, self.m
        amax = self.amax[b]
        # attention input: LN fused into the quantizer, one pass for both formats if mixed
        need = set(fmts[0:3])
        a0_i8 = ws.act(0, D.FMT_INT8, b) if D.FMT_INT8 in need else None
        a0_f4 = ws.act(0, D.FMT_NVFP4, b) if D.FMT_NVFP4 in need else None
        cap = self.capture is not None
        h1 = torch.empty(m, H, dtype=torch.bfloat16, device=x_in.device) if cap else None
        hd = self.hadamard
        D.dmpq_quantize_act(x_in, out_i8=a0_i8, out_fp4=a0_f4, amax_out=amax[0:1], layernorm=True, h_out=h1, hadamard=hd)
        if cap:
            self._cap("x_in", x_in); self._cap("h1", h1)
            self._cap_act("a0_i8", a0_i8); self._cap_act("a0_f4", a0_f4)
        for j, out in ((0, ws.qk), (1, ws.qk), (2, ws.v)):
            a = a0_i8 if fmts[j] == D.FMT_INT8 else a0_f4
            self._gemm(a, W.layers[j], Y=out)
            self._cap(f"y{j}", out)
        # O projection on the attention stand-in a = v, gated residual in the epilogue
        a1 = ws.act(1, fmts[3], b)
        D.dmpq_quantize_act(ws.v, **{("out_i8" if fmts[3] == D.FMT_INT8 else "out_fp4"): a1}, amax_out=amax[1:2],
                            hadamard=hd)
        self._cap_act("a1", a1)
        self._gemm(a1, W.layers[3], Y=ws.x_mid, residual=x_in, gate=W.g1)
        self._cap("x_mid", ws.x_mid)
        # FFN
        a2 = ws.act(2, fmts[4], b)
        h2 = torch.empty(m, H, dtype=torch.bfloat16, device=x_in.device) if cap else None
        D.dmpq_quantize_act(ws.x_mid, **{("out_i8" if fmts[4] == D.FMT_INT8 else "out_fp4"): a2},
                            amax_out=amax[2:3], layernorm=True, h_out=h2, hadamard=hd)
        if cap:
            self._cap("h2", h2); self._cap_act("a2", a2)
        self._gemm(a2, W.layers[4], Y=ws.f, gelu=True)
        self._cap("f", ws.f)
        a3 = ws.act(3, fmts[5], b)
        D.dmpq_quantize_act(ws.f, **{("out_i8" if fmts[5] == D.FMT_INT8 else "out_fp4"): a3}, amax_out=amax[3:4],
                            hadamard=hd)
        self._cap_act("a3", a3)
        self._gemm(a3, W.layers[5], Y=x_out, residual=ws.x_mid, gate=W.g2)
        self._cap("x_out", x_out)
        self.launches += 4 + 6
        return 2.0 * m * (4 * H * H + 2 * H * F)

    def _gemm(self, a, w, **kw):
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
        self.gemm_events = {D.FMT_INT8: [], D.FMT_NVFP4: []}
        self.gemm_flops = {D.FMT_INT8: 0.0, D.FMT_NVFP4: 0.0}

    # ------------------------------------------------------------------ one timestep
    def step(self, x0: torch.Tensor, t: int) -> torch.Tensor:
        """Run all blocks at timestep t on this rank's rows; returns the last output
        (a view of an internal buffer). Call end_step(t) afterwards."""
        rec = StepRecord(t)
        self.amax.zero_()
        self.stats_slots.zero_()
        x_in = x0
        for b in range(self.nb):
            x_out = self.x_buf[b % 2]
            d = D.tdc_decide(self.tdc[b], self.cfg, t) if self.tdc_enabled else L.TDC_COMPUTE
            if d == L.TDC_DECIDE_SKIP:
                D.tdc_step(L.TDC_SKIP, x_in, x_out, self.delta[b])
                self.launches += 1
                rec.fmts.append(None)
                rec.gammas.append(float("nan"))
            else:
                if self.force_fmt is not None:
                    fmts, gamma = [self.force_fmt] * 6, float("nan")
                else:
                    fmts, gamma, _ = D.dmpq_predict(self.prev_stats[b], self.tau, t, self.prev_skipped[b])
                rec.linear_flops += self._compute_block(b, x_in, x_out, fmts)
                D.tdc_step(L.TDC_REFRESH, x_in, x_out, self.delta[b], self.stats_slots[self.rank, b],
                           self.ws.tdc_ws)
                self.launches += 1
                rec.fmts.append(fmts)
                rec.gammas.append(gamma)
            rec.decisions.append(d)
            x_in = x_out
        self.records.append(rec)
        return x_in

    def end_step(self, t: int):
        """Per-step exchange + host decisions: combine the statistics of all ranks
        (slot-packed SUM all-reduce = exact all-gather; MAX all-reduce for amax), copy
        them to the host once, update TDC (Eq. 10) and the NVFP4 global scales (R3)."""
        # one exchange per step; the D2H copy inside synchronises the stream
        stats = exchange(self.stats_slots, self.amax, self.group, self.world)
        D.dmpq_global_scale(self.amax.view(-1), 1344.0, self.g_table.view(-1))
        self.launches += 1
        rec = self.records[-1]
        for b in range(self.nb):
            d = rec.decisions[b]
            if d == L.TDC_DECIDE_SKIP:
                D.tdc_update(self.tdc[b], self.cfg, t, d, None)
                self.prev_stats[b] = None
                self.prev_skipped[b] = True
            else:
                st = L.BlockStats.from_seq(stats[b])
                D.tdc_update(self.tdc[b], self.cfg, t, d, st)
                self.prev_stats[b] = st
                self.prev_skipped[b] = False
        return stats

    def mix(self, records=None):
        """Realised NVFP4 / INT8 / skip mix over the given step records."""
        records = self.records if records is None else records
        n4 = n8 = sk = 0
        for r in records:
            for f in r.fmts:
                if f is None:
                    sk += 1
                else:
                    n4 += sum(1 for x in f if x == D.FMT_NVFP4)
                    n8 += sum(1 for x in f if x == D.FMT_INT8)
        tot_layers = max(1, n4 + n8)
        nblk = max(1, sum(len(r.fmts) for r in records))
        return {"nvfp4_layer_frac": n4 / tot_layers, "int8_layer_frac": n8 / tot_layers, "skip_block_frac": sk / nblk}
