"""Diagnostic (development): where the Hadamard INT8 quantizer's codes differ from the oracle
(dense FFN2-input rows, K = 12288), with the properties of the differing elements' 128-blocks."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as orc  # noqa: E402
from paper_2603_18742_b200 import build, dmpq as D, synth  # noqa: E402
build.build()
m, k = 2053, 12288
x = synth.ffn2_activation(m, k, seed=k + 17)
for which in ("int8", "both"):
    a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=torch.tensor([0.004], device="cuda"))
    a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    D.dmpq_quantize_act(x.cuda(), out_i8=a8, out_fp4=a4 if which == "both" else None, hadamard=True)
    torch.cuda.synchronize()
    xf = orc.bf16_to_f32(synth.bits(x)).reshape(m, k)
    y = orc.fht128(xf)
    c8, s8 = orc.int8_quantize_f32(y)
    g8 = a8.codes.cpu().numpy()
    bad = np.argwhere(g8 != c8)
    print(which, "mismatches", len(bad), "scales equal", np.array_equal(a8.row_scale.cpu().numpy(), s8))
    for r, c in bad[:12]:
        blk = xf[r, (c // 128) * 128:(c // 128 + 1) * 128]
        sub = int(np.sum((np.abs(blk) < 1.1754944e-38) & (blk != 0)))
        v = np.float32(y[r, c]) * np.float32(127.0) / np.float32(s8[r] * 127.0) if False else None
        print(f"  row {r} col {c}: gpu {g8[r, c]} oracle {c8[r, c]} y {y[r, c]!r} scale {s8[r]!r} "
              f"subnormal inputs in block {sub} min|x|>0 {np.min(np.abs(blk[blk != 0])) if np.any(blk != 0) else 0!r}")
