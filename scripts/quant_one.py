import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2603_18742_b200 import build, dmpq as D, synth
build.build()
m, k = 35552, int(sys.argv[1])
x = synth.dit_activation(m, k, seed=1).cuda()
g = torch.tensor([1e-3], device="cuda")
a = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g)
for _ in range(4):
    D.dmpq_quantize_act(x, out_fp4=a, hadamard=True)
torch.cuda.synchronize()
