"""One quantizer configuration, launched a few times (for ncu captures).
    python scripts/quant_one.py K [nvfp4|int8|both] [had|plain] [ln]"""
import sys
import torch
sys.path.insert(0, '/root/repo')
from paper_2603_18742_b200 import build, dmpq as D, synth  # noqa: E402
build.build()
m, k = 35552, int(sys.argv[1])
fmt = sys.argv[2] if len(sys.argv) > 2 else "nvfp4"
had = (sys.argv[3] if len(sys.argv) > 3 else "had") == "had"
ln = len(sys.argv) > 4 and sys.argv[4] == "ln"
x = synth.dit_activation(m, k, seed=1).cuda()
g = torch.tensor([1e-3], device="cuda")
a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g) if fmt in ("nvfp4", "both") else None
a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda") if fmt in ("int8", "both") else None
for _ in range(4):
    D.dmpq_quantize_act(x, out_fp4=a4, out_i8=a8, hadamard=had, layernorm=ln)
torch.cuda.synchronize()
