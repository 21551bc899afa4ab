"""Hadamard quantizer timing at the CogVideoX-5B shapes (development tool): both formats,
with and without the LN prologue. Run with DMPQ_QUANT_HAD_CHUNK=1 for the chunk kernel.
    python scripts/had_ab.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_18742_b200 import build, dmpq as D, synth  # noqa: E402

build.build()
HBM = 6546.9
m = 35552
for k in (3072, 12288):
    xs = [synth.dit_activation(m, k, seed=i).cuda() for i in range(2)]
    g = torch.tensor([1e-3], device="cuda")
    a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g)
    a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    amax = torch.zeros(1, device="cuda")
    for fmt in ("nvfp4", "int8", "both"):
        for ln in ((False, True) if k == 3072 else (False,)):
            it = [0]

            def run():
                x = xs[it[0] % 2]
                it[0] += 1
                D.dmpq_quantize_act(x, out_fp4=a4 if fmt != "int8" else None, out_i8=a8 if fmt != "nvfp4" else None,
                                    amax_out=amax, hadamard=True, layernorm=ln)
            for _ in range(3):
                run()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            for _ in range(20):
                run()
            e.record()
            torch.cuda.synchronize()
            t = s.elapsed_time(e) / 20 * 1e-3
            bpe = 2 + (0.5 + 1 / 16 if fmt != "int8" else 0) + (1 + 4 / k if fmt != "nvfp4" else 0)
            print(json.dumps(dict(k=k, fmt=fmt, ln=ln, us=round(t * 1e6, 1), gbs=round(m * k * bpe / t / 1e9),
                                  frac=round(m * k * bpe / t / 1e9 / HBM, 3))))
