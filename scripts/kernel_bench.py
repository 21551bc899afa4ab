"""Per-kernel microbenchmarks (CUDA events on the launching stream, inputs larger
than L2 or rotated across buffers). Development tool; bench.py is the contract.

    python scripts/kernel_bench.py [--gemm] [--quant] [--tdc] [--shapes c2|c4]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_18742_b200 import build, dmpq as D, synth  # noqa: E402

PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))) \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else \
    {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def timeit(fn, iters=20, warmup=3):
    for _ in range(warmup):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def bench_gemm(m, n, k, fmt, nbuf=2, block=0, res=False):
    x = synth.dit_activation(m, k, seed=1).cuda()
    w, b = synth.linear_weight(n, k, seed=2)
    pw = D.dmpq_pack_weights(w.cuda(), b, hadamard=bool(block))
    g = torch.tensor([1e-3], device="cuda")
    acts = []
    for i in range(nbuf):
        a = D.QuantAct.empty(fmt, m, k, "cuda", g=g if fmt == D.FMT_NVFP4 else None, scale_block=block)
        if fmt == D.FMT_NVFP4:
            D.dmpq_quantize_act(x, out_fp4=a)
        else:
            D.dmpq_quantize_act(x, out_i8=a, hadamard=bool(block))
        acts.append(a)
    ys = [torch.empty(m, n, dtype=torch.bfloat16, device="cuda") for _ in range(nbuf)]
    kw = {}
    if res:   # gated residual epilogue (the O projection / FFN2 shape of the block)
        kw = dict(residual=synth.dit_activation(m, n, seed=3).cuda(), gate=torch.full((n,), 0.01, device="cuda"))
    it = [0]

    def run():
        i = it[0] % nbuf
        it[0] += 1
        D.dmpq_gemm(acts[i], pw, Y=ys[i], **kw)
    t = timeit(run)
    flops = 2.0 * m * n * k
    peak = PEAKS["bf16_tflops"] * (4 if fmt == D.FMT_NVFP4 else 2)
    return dict(kernel="gemm_" + ("nvfp4" if fmt == D.FMT_NVFP4 else "int8") + ("_block" if block else "") + ("_res" if res else ""),
                m=m, n=n, k=k,
                us=t * 1e6,
                tflops=flops / t / 1e12, frac=flops / t / 1e12 / peak)


def bench_quant(m, k, fmt, hadamard=False):
    xs = [synth.dit_activation(m, k, seed=i).cuda() for i in range(2)]
    g = torch.tensor([1e-3], device="cuda")
    a = D.QuantAct.empty(fmt, m, k, "cuda", g=g if fmt == D.FMT_NVFP4 else None)
    amax = torch.zeros(1, device="cuda")
    it = [0]

    def run():
        x = xs[it[0] % 2]
        it[0] += 1
        if fmt == D.FMT_NVFP4:
            D.dmpq_quantize_act(x, out_fp4=a, amax_out=amax, hadamard=hadamard)
        else:
            D.dmpq_quantize_act(x, out_i8=a, amax_out=amax, hadamard=hadamard)
    t = timeit(run)
    bpe = 2 + 0.5 + 1 / 16 if fmt == D.FMT_NVFP4 else 2 + 1 + 4 / k
    gbs = m * k * bpe / t / 1e9
    return dict(kernel="quant_" + ("nvfp4" if fmt == D.FMT_NVFP4 else "int8") + ("_had" if hadamard else ""), m=m, k=k,
                us=t * 1e6, gbs=gbs,
                frac=gbs / PEAKS["hbm_gbs"])


def bench_tdc(m, h):
    xi = synth.dit_activation(m, h, seed=1, outlier_frac=0, tail_frac=0).cuda()
    xo = synth.dit_activation(m, h, seed=2, outlier_frac=0, tail_frac=0).cuda()
    dl = synth.dit_activation(m, h, seed=3, outlier_frac=0, tail_frac=0).cuda()
    st = torch.zeros(7, dtype=torch.float64, device="cuda")
    ws = torch.zeros(D.tdc_workspace_bytes(m, h), dtype=torch.uint8, device="cuda")
    t = timeit(lambda: D.tdc_step(1, xi, xo, dl, st, ws))
    t2 = timeit(lambda: D.tdc_step(0, xi, xo, dl))
    cache = D.DeltaCacheNvfp4(m, h, "cuda")
    g = torch.tensor([1e-3], device="cuda")
    am = torch.zeros(1, device="cuda")
    t3 = timeit(lambda: D.tdc_step_nvfp4(1, xi, xo, cache, g_new=g, amax_out=am, stats_out=st, workspace=ws))
    t4 = timeit(lambda: D.tdc_step_nvfp4(0, xi, xo, cache))
    b3, b4 = 4 + 2 * 0.5625, 4 + 0.5625     # bytes per element: x_in + x_out + cache read (+ write)
    return [dict(kernel="tdc_refresh", m=m, h=h, us=t * 1e6, gbs=m * h * 8 / t / 1e9, frac=m * h * 8 / t / 1e9 / PEAKS["hbm_gbs"]),
            dict(kernel="tdc_skip", m=m, h=h, us=t2 * 1e6, gbs=m * h * 6 / t2 / 1e9, frac=m * h * 6 / t2 / 1e9 / PEAKS["hbm_gbs"]),
            dict(kernel="tdc_refresh_nvfp4", m=m, h=h, us=t3 * 1e6, gbs=m * h * b3 / t3 / 1e9,
                 frac=m * h * b3 / t3 / 1e9 / PEAKS["hbm_gbs"]),
            dict(kernel="tdc_skip_nvfp4", m=m, h=h, us=t4 * 1e6, gbs=m * h * b4 / t4 / 1e9,
                 frac=m * h * b4 / t4 / 1e9 / PEAKS["hbm_gbs"])]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gemm", action="store_true")
    ap.add_argument("--quant", action="store_true")
    ap.add_argument("--tdc", action="store_true")
    ap.add_argument("--shapes", default="c2,c4")
    ap.add_argument("--block", action="store_true", help="also the per-block INT8 GEMM (R17)")
    ap.add_argument("--res", action="store_true", help="also the gated-residual epilogue at the N = 3072 shapes")
    ap.add_argument("--one", default=None, help="fmt:m,n,k  e.g. nvfp4:35552,3072,3072 (one GEMM, 5 launches)")
    a = ap.parse_args()
    if a.one:
        build.build()
        f, dims = a.one.split(":")
        m, n, k = map(int, dims.split(","))
        print(json.dumps(bench_gemm(m, n, k, D.FMT_NVFP4 if f == "nvfp4" else D.FMT_INT8)))
        return
    if not (a.gemm or a.quant or a.tdc):
        a.gemm = a.quant = a.tdc = True
    build.build()
    res = []
    if a.gemm:
        shapes = []
        if "c2" in a.shapes:
            shapes += [(mm, 1920, 1920) for mm in (4096, 16384, 65536)]
        if "c4" in a.shapes:
            shapes += [(35552, 3072, 3072), (35552, 12288, 3072), (35552, 3072, 12288)]
        for (m, n, k) in shapes:
            for fmt, blk in ((D.FMT_NVFP4, 0), (D.FMT_INT8, 0), (D.FMT_INT8, 128)):
                if blk and not a.block:
                    continue
                r = bench_gemm(m, n, k, fmt, block=blk)
                print(json.dumps(r), flush=True)
                res.append(r)
                if a.res and m == 35552 and n == 3072 and not blk:
                    r = bench_gemm(m, n, k, fmt, res=True)
                    print(json.dumps(r), flush=True)
                    res.append(r)
    if a.quant:
        for (m, k) in [(35552, 3072), (35552, 12288), (65536, 1920)]:
            for fmt in (D.FMT_NVFP4, D.FMT_INT8):
                for had in (False, True):
                    r = bench_quant(m, k, fmt, had)
                    print(json.dumps(r), flush=True)
                    res.append(r)
    if a.tdc:
        for r in bench_tdc(35552, 3072):
            print(json.dumps(r), flush=True)
            res.append(r)


if __name__ == "__main__":
    main()
