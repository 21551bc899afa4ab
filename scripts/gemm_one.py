"""One GEMM configuration launched a few times (for ncu captures).
    python scripts/gemm_one.py M N K int8|nvfp4 [res]"""
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_2603_18742_b200 import build, dmpq as D, synth  # noqa: E402

build.build()
m, n, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
fmt = D.FMT_NVFP4 if sys.argv[4] == "nvfp4" else D.FMT_INT8
res_on = len(sys.argv) > 5 and sys.argv[5] == "res"
x = synth.dit_activation(m, k, seed=1).cuda()
w, b = synth.linear_weight_device(n, k, seed=2, device="cuda")
pw = D.dmpq_pack_weights(w, b)
g = torch.tensor([1e-3], device="cuda")
a = D.QuantAct.empty(fmt, m, k, "cuda", g=g if fmt == D.FMT_NVFP4 else None)
D.dmpq_quantize_act(x, out_fp4=a if fmt == D.FMT_NVFP4 else None, out_i8=a if fmt == D.FMT_INT8 else None)
y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
kw = {}
if res_on:
    kw = dict(residual=synth.dit_activation(m, n, seed=3).cuda(), gate=torch.full((n,), 0.01, device="cuda"))
for _ in range(4):
    D.dmpq_gemm(a, pw, Y=y, **kw)
torch.cuda.synchronize()
