"""Print the per-step TDC / DMPQ decisions of the synthetic block stack (diagnostic)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_18742_b200 import build, synth  # noqa: E402
from paper_2603_18742_b200.block import DiTStack  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--blocks", type=int, default=4)
ap.add_argument("--H", type=int, default=3072)
ap.add_argument("--F", type=int, default=12288)
ap.add_argument("--M", type=int, default=8192)
ap.add_argument("--T", type=int, default=20)
ap.add_argument("--kappa", type=float, default=0.05)
ap.add_argument("--gate", type=float, nargs="*", default=None)
ap.add_argument("--pdr", action="store_true")
ap.add_argument("--hadamard", action="store_true")
a = ap.parse_args()
build.build()
dev = torch.device("cuda")
m = DiTStack(a.blocks, a.H, a.F, a.M, dev, seed=0, gate_scales=a.gate, pdr=a.pdr, hadamard=a.hadamard)
A, B = synth.trajectory_basis(a.M, a.H, 1000, dev)
for t in range(a.T):
    x = synth.trajectory_input(A, B, t, 50, a.kappa)
    m.step(x, t)
    m.end_step(t)
    r = m.records[-1]
    row = []
    for b in range(a.blocks):
        st = m.tdc[b]
        f = r.fmts[b]
        fs = "SKIP" if f is None else "".join({0: "8", 1: "4", 2: "B"}[v] for v in f)
        rr = "" if not a.pdr or m.ratio[b] is None else ":R=" + ",".join(f"{x:.0f}" for x in m.ratio[b])
        row.append(f"{fs}:g={r.gammas[b]:.4f}:e={st.e_tp:.2e}{rr}")
    print(t, " | ".join(row), flush=True)
