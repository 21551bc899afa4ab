"""FFN2-shaped GEMM (M = 35,552, N = 3072, K = 12288, gated residual) with and without the
fused TDC refresh epilogue (development tool).   python scripts/fused_refresh_ab.py [int8|nvfp4] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_18742_b200 import build, dmpq as D, synth  # noqa: E402

build.build()
fmt = D.FMT_NVFP4 if (len(sys.argv) > 1 and sys.argv[1] == "nvfp4") else D.FMT_INT8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
m, n, k = 35552, 3072, int(os.environ.get("K", 12288))
x = synth.ffn2_activation(m, k, seed=1).cuda()
w, b = synth.linear_weight_device(n, k, seed=2, device="cuda")
pw = D.dmpq_pack_weights(w, b)
g = torch.tensor([1e-3], device="cuda")
a = D.QuantAct.empty(fmt, m, k, "cuda", g=g if fmt == D.FMT_NVFP4 else None)
D.dmpq_quantize_act(x, out_fp4=a if fmt == D.FMT_NVFP4 else None, out_i8=a if fmt == D.FMT_INT8 else None)
res = synth.dit_activation(m, n, seed=3).cuda()
xin = synth.dit_activation(m, n, seed=4).cuda()
delta = synth.dit_activation(m, n, seed=5).cuda()
gate = torch.full((n,), 0.01, device="cuda")
y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
st = torch.zeros(7, dtype=torch.float64, device="cuda")
ws = torch.zeros(D.dmpq_gemm_tdc_workspace_bytes(), dtype=torch.uint8, device="cuda")
tws = torch.zeros(D.tdc_workspace_bytes(m, n), dtype=torch.uint8, device="cuda")


def timeit(fn):
    for _ in range(2):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


tp = timeit(lambda: D.dmpq_gemm(a, pw, Y=y))
t0 = timeit(lambda: D.dmpq_gemm(a, pw, Y=y, residual=res, gate=gate))
t1 = timeit(lambda: D.dmpq_gemm(a, pw, Y=y, residual=res, gate=gate, tdc_x_in=xin, tdc_delta=delta, tdc_stats=st,
                                tdc_workspace=ws))
t2 = timeit(lambda: D.tdc_step(1, xin, y, delta, st, tws))
print(f"fmt={fmt} plain {tp:.1f} us, gated residual {t0:.1f} us, gemm+fused refresh {t1:.1f} us, separate refresh {t2:.1f} us")
