"""Writes the bf16 outputs of the INT8 and NVFP4 GEMMs (plain, GELU, gated residual; ragged M / N)
for one seeded problem to an .npz (used by tests/test_gpu_parity.py::test_gemm_cluster4_equals_pairs,
run once per DMPQ_GEMM_CLUSTER setting in its own process — the knob is read once per process)."""
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2603_18742_b200 import build, dmpq as D, synth  # noqa: E402

build.build()
out = {}
for (m, n, k) in [(300, 384, 512), (1029, 1920, 3072), (513, 96, 256)]:
    x = synth.dit_activation(m, k, seed=m + n).cuda()
    w, b = synth.linear_weight(n, k, seed=k)
    pw = D.dmpq_pack_weights(w.cuda(), b.cuda())
    res = synth.dit_activation(m, n, seed=n).cuda()
    gate = torch.rand(n, generator=torch.Generator().manual_seed(3)).cuda()
    a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=torch.tensor([0.004], device="cuda"))
    a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    D.dmpq_quantize_act(x, out_i8=a8, out_fp4=a4)
    for name, a in (("fp4", a4), ("i8", a8)):
        for ep in ("plain", "gelu", "res"):
            y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
            kw = {"gelu": True} if ep == "gelu" else ({"residual": res, "gate": gate} if ep == "res" else {})
            D.dmpq_gemm(a, pw, Y=y, **kw)
            out[f"{name}_{ep}_{m}_{n}_{k}"] = y.view(torch.int16).cpu().numpy()
torch.cuda.synchronize()
np.savez(sys.argv[1], **out)
