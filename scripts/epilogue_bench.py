import sys, json, torch
sys.path.insert(0, '/root/repo')
from paper_2603_18742_b200 import build, dmpq as D, synth
build.build()
m, n, k = 35552, 12288, 3072
x = synth.dit_activation(m, k, seed=1).cuda()
w, b = synth.linear_weight_device(n, k, 2, "cuda")
pw = D.dmpq_pack_weights(w, b)
for fmt in (D.FMT_NVFP4, D.FMT_INT8):
    g = torch.tensor([1e-3], device="cuda")
    a = D.QuantAct.empty(fmt, m, k, "cuda", g=g if fmt == D.FMT_NVFP4 else None)
    D.dmpq_quantize_act(x, **({"out_fp4": a} if fmt == D.FMT_NVFP4 else {"out_i8": a}))
    y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    for gelu in (False, True):
        for _ in range(3): D.dmpq_gemm(a, pw, Y=y, gelu=gelu)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(10): D.dmpq_gemm(a, pw, Y=y, gelu=gelu)
        e.record(); torch.cuda.synchronize()
        t = s.elapsed_time(e) / 10 * 1e-3
        print(json.dumps(dict(fmt=fmt, gelu=gelu, us=t * 1e6, tflops=2 * m * n * k / t / 1e12)))
