"""Quantizer launch-shape sweep (development): CUDA-event time of the Hadamard / plain
quantizer for one (K, format) under the current DMPQ_QUANT_* environment."""
import json
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_18742_b200 import build, dmpq as D, synth  # noqa: E402
build.build()
m = 35552
res = {}
for k in (3072, 12288):
    xs = [synth.dit_activation(m, k, seed=i).cuda() for i in range(2)]
    g = torch.tensor([1e-3], device="cuda")
    for fmt in ("nvfp4", "int8", "both"):
        for had in (True, False):
            a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g) if fmt in ("nvfp4", "both") else None
            a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda") if fmt in ("int8", "both") else None
            for ln in ((False, True) if k == 3072 else (False,)):
                for i in range(3):
                    D.dmpq_quantize_act(xs[i % 2], out_fp4=a4, out_i8=a8, hadamard=had, layernorm=ln)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize(); s.record()
                for i in range(20):
                    D.dmpq_quantize_act(xs[i % 2], out_fp4=a4, out_i8=a8, hadamard=had, layernorm=ln)
                e.record(); torch.cuda.synchronize()
                res[f"{k}_{fmt}_{'had' if had else 'plain'}{'_ln' if ln else ''}"] = round(s.elapsed_time(e) / 20 * 1e3, 1)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("DMPQ_QUANT")}, "us": res}))
