"""The on-the-fly NVFP4 -> INT8 weight cast of the FFN1 layer (12288 x 3072), a few launches (ncu)."""
import sys
import torch
sys.path.insert(0, '/root/repo')
from paper_2603_18742_b200 import build, dmpq as D, synth  # noqa: E402
build.build()
w, b = synth.linear_weight_device(12288, 3072, seed=2, device="cuda")
pw = D.dmpq_pack_weights(w, b, hadamard=True, int8_resident=False)
scratch = torch.empty(12288 * 3072, dtype=torch.int8, device="cuda")
for _ in range(4):
    D.dmpq_cast_int8(pw, scratch)
torch.cuda.synchronize()
