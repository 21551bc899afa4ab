"""The four GEMM kinds of a CogVideoX-5B block step (QKV plain, O + gated residual, FFN1 + GELU,
FFN2 + gated residual; M = 35,552), both formats, CUDA-event timed. Development tool for
epilogue / pipeline variants (build with DMPQ_NVCC_EXTRA, select stages with DMPQ_GEMM_STAGES)."""
import json
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_18742_b200 import build, dmpq as D, synth  # noqa: E402
build.build()
m, H, F = 35552, 3072, 12288
res = {}
for name, n, k, kw in (("qkv", H, H, {}), ("o_res", H, H, {"res": True}), ("ffn1_gelu", F, H, {"gelu": True}),
                       ("ffn2_res", H, F, {"res": True})):
    x = synth.dit_activation(m, k, seed=1).cuda()
    w, b = synth.linear_weight_device(n, k, 2, "cuda")
    pw = D.dmpq_pack_weights(w, b)
    resid = torch.randn(m, n, device="cuda").to(torch.bfloat16) if kw.get("res") else None
    gate = torch.rand(n, device="cuda") if kw.get("res") else None
    for fmt in (D.FMT_NVFP4, D.FMT_INT8):
        g = torch.tensor([1e-3], device="cuda")
        a = D.QuantAct.empty(fmt, m, k, "cuda", g=g if fmt == D.FMT_NVFP4 else None)
        D.dmpq_quantize_act(x, **({"out_fp4": a} if fmt == D.FMT_NVFP4 else {"out_i8": a}))
        y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
        call = lambda: D.dmpq_gemm(a, pw, Y=y, gelu=kw.get("gelu", False), residual=resid, gate=gate)
        for _ in range(3):
            call()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(10):
            call()
        e.record(); torch.cuda.synchronize()
        t = s.elapsed_time(e) / 10 * 1e-3
        res[f"{name}_{'fp4' if fmt == D.FMT_NVFP4 else 'i8'}"] = round(t * 1e6, 1)
print(json.dumps({"extra": os.environ.get("DMPQ_NVCC_EXTRA", ""), "stages": os.environ.get("DMPQ_GEMM_STAGES", "5"),
                  "us": res, "sum_us": round(sum(res.values()), 1)}))
