"""Small invocations of every kernel for compute-sanitizer runs (memcheck / racecheck / synccheck)."""
import sys
import torch
sys.path.insert(0, '/root/repo')
from paper_2603_18742_b200 import build, dmpq as D, synth  # noqa: E402
build.build()
dev = "cuda"
for (m, k) in [(37, 1920), (130, 3072)]:
    x = synth.dit_activation(m, k, seed=m).to(dev)
    g = torch.tensor([0.01], device=dev)
    a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, dev, g=g)
    a8 = D.QuantAct.empty(D.FMT_INT8, m, k, dev)
    h = torch.empty(m, k, dtype=torch.bfloat16, device=dev)
    rs = torch.zeros(m, device=dev)
    ai = torch.zeros(1, device=dev)
    for had in (False, True):
        for ln in (False, True):
            D.dmpq_quantize_act(x, out_i8=a8, out_fp4=a4, layernorm=ln, h_out=h if ln else None, hadamard=had,
                                row_abs_sum=rs, amax_in=ai)
    w, b = synth.linear_weight(256, k, seed=1)
    for had in (False, True):
        pw = D.dmpq_pack_weights(w.to(dev), b.to(dev), hadamard=had, keep_bf16=True)
        y = torch.empty(m, 256, dtype=torch.bfloat16, device=dev)
        D.dmpq_gemm(a8, pw, Y=y)
        D.dmpq_gemm(a4, pw, Y=y, gelu=True)
        D.dmpq_gemm(D.QuantAct.bf16(x), pw, Y=y)
H = 128
m = 256
xi = synth.dit_activation(m, H, seed=1).to(dev)
xo = synth.dit_activation(m, H, seed=2).to(dev)
st = torch.zeros(7, dtype=torch.float64, device=dev)
ws = torch.zeros(D.tdc_workspace_bytes(m, H), dtype=torch.uint8, device=dev)
delta = torch.zeros(m, H, dtype=torch.bfloat16, device=dev)
D.tdc_step(1, xi, xo, delta, st, ws)
D.tdc_step(0, xi, xo, delta)
cache = D.DeltaCacheNvfp4(m, H, dev)
am = torch.zeros(1, device=dev)
D.tdc_delta_amax(xi, xo, am)
D.tdc_step_nvfp4(1, xi, xo, cache, g_new=torch.tensor([0.01], device=dev), amax_out=am, stats_out=st, workspace=ws)
D.tdc_step_nvfp4(0, xi, xo, cache)
# gated-residual epilogue (TMA-staged residual, chunks requested a tile ahead: several tiles per
# CTA at this size) and the fused TDC refresh epilogue, both formats
m2, n2, k2 = 1200, 3072, 128
x2 = synth.dit_activation(m2, k2, seed=5).to(dev)
w2, b2 = synth.linear_weight(n2, k2, seed=6)
pw2 = D.dmpq_pack_weights(w2.to(dev), b2.to(dev))
res = synth.dit_activation(m2, n2, seed=7).to(dev)
gate = torch.full((n2,), 0.01, device=dev)
y2 = torch.empty(m2, n2, dtype=torch.bfloat16, device=dev)
d2 = torch.zeros(m2, n2, dtype=torch.bfloat16, device=dev)
xin2 = synth.dit_activation(m2, n2, seed=8).to(dev)
wsg = torch.zeros(D.dmpq_gemm_tdc_workspace_bytes(), dtype=torch.uint8, device=dev)
for fmt in (D.FMT_INT8, D.FMT_NVFP4):
    a = D.QuantAct.empty(fmt, m2, k2, dev, g=torch.tensor([0.01], device=dev) if fmt == D.FMT_NVFP4 else None)
    D.dmpq_quantize_act(x2, out_fp4=a if fmt == D.FMT_NVFP4 else None, out_i8=a if fmt == D.FMT_INT8 else None,
                        hadamard=True)
    D.dmpq_gemm(a, pw2, Y=y2, residual=res, gate=gate)
    D.dmpq_gemm(a, pw2, Y=y2, residual=res, gate=gate, tdc_x_in=xin2, tdc_delta=d2, tdc_stats=st, tdc_workspace=wsg)
# round 2: on-the-fly INT8 weight cast, per-block INT8 (quantizer + promotion GEMM), device PDR gate with
# predicated GEMMs, producer-fused NVFP4 quantizer epilogue (both GEMM kinds)
m3, k3, n3 = 300, 1920, 384
x3 = synth.dit_activation(m3, k3, seed=9).to(dev)
w3, b3 = synth.linear_weight(n3, k3, seed=10)
lean = D.dmpq_pack_weights(w3.to(dev), b3.to(dev), hadamard=True, int8_resident=False, keep_bf16=True)
scratch = torch.empty(n3 * k3, dtype=torch.int8, device=dev)
cast = D.dmpq_cast_int8(lean, scratch)
ab = D.QuantAct.empty(D.FMT_INT8, m3, k3, dev, scale_block=128)
rs3 = torch.zeros(m3, device=dev)
ai3 = torch.zeros(1, device=dev)
D.dmpq_quantize_act(x3, out_i8=ab, hadamard=True, row_abs_sum=rs3, amax_in=ai3)
y3 = torch.empty(m3, n3, dtype=torch.bfloat16, device=dev)
res3 = synth.dit_activation(m3, n3, seed=11).to(dev)
gate3 = torch.full((n3,), 0.01, device=dev)
D.dmpq_gemm(ab, cast, Y=y3, gelu=True)
D.dmpq_gemm(ab, cast, Y=y3, residual=res3, gate=gate3)
flag = torch.zeros(1, dtype=torch.int32, device=dev)
D.dmpq_outlier_gate(rs3, ai3, m3 * k3, 25.0, flag)
a83 = D.QuantAct.empty(D.FMT_INT8, m3, k3, dev)
D.dmpq_quantize_act(x3, out_i8=a83, hadamard=True)
D.dmpq_gemm(a83, cast, Y=y3, run_if=flag, run_if_value=0)
D.dmpq_gemm(D.QuantAct.bf16(x3), cast, Y=y3, run_if=flag, run_if_value=1)
q = D.QuantAct.empty(D.FMT_NVFP4, m3, n3, dev, g=torch.tensor([0.01], device=dev))
qa = torch.zeros(1, device=dev)
for fmt in (D.FMT_INT8, D.FMT_NVFP4):
    a = D.QuantAct.empty(fmt, m3, k3, dev, g=torch.tensor([0.01], device=dev) if fmt == D.FMT_NVFP4 else None)
    D.dmpq_quantize_act(x3, out_fp4=a if fmt == D.FMT_NVFP4 else None, out_i8=a if fmt == D.FMT_INT8 else None,
                        hadamard=True)
    D.dmpq_gemm(a, cast, gelu=True, quant_out=q, quant_amax=qa)
torch.cuda.synchronize()
print("sanitize_small ok")
