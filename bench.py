"""bench.py — DMPQ + TDC hot path on B200: the driver's benchmark contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4|c2|c3|c5|c1]

Workload (default, BASELINE.json configs[3]): CogVideoX-5B-shaped block stack,
42 blocks, hidden 3072, FFN 12288, 49 frames at 480x720 -> 17,776 tokens per
sample, CFG batch 2 -> M = 35,552 token rows, token-sharded over N ranks (strong
scaling), 50-step synthetic PF-ODE-like trajectory with TDC skipping and DMPQ
routing live. One bench "step" = one denoising timestep through all 42 blocks:
TDC decisions, routing, LN+quantize, the six DMPQ GEMMs per computed block, the
TDC refresh/skip kernels, the per-step statistics exchange and host update.

metric/value: executed DMPQ linear TFLOP/s (2*m*N*K of every GEMM actually run,
all ranks) / max-over-ranks step time; block-step ms and the realised
NVFP4/INT8/skip mix are reported beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DMPQ linear TFLOPS (% FP4/INT8 peak) + block-step ms, CogVideoX-5B, 1/2/4/8 B200"

CONFIGS = {
    # name: (description, n_blocks, H, F, M_total, T)
    "c4": ("CogVideoX-5B 42-block step, hidden 3072, 49f 480x720 (17,776 tok) x CFG 2, 50-step TDC", 42, 3072, 12288,
           2 * 17776, 50),
    "c3": ("CogVideoX-2B 30-block step, hidden 1920, 49f 480x720 (17,776 tok) x CFG 2, 50-step TDC", 30, 1920, 7680,
           2 * 17776, 50),
    # HunyuanVideo: 20 dual-stream + 40 single-stream blocks; 129 frames at 720p -> 33 latent frames x 45 x 80 + 256 text
    "c5": ("HunyuanVideo-shaped 60-block step, hidden 3072, 720p x 129f (119,056 tok), 50-step TDC", 60, 3072, 12288,
           119056, 50),
    "c1": ("one DiT block, hidden 128, 256 tokens, 4 timesteps", 1, 128, 512, 256, 4),
    # single-layer sweep (BASELINE configs[1]): K = N = 1920, M = 4K..64K, NVFP4 and INT8 (run_sweep)
    "c2": ("single linear layer sweep M=4K-64K tokens, K=N=1920 (CogVideoX-2B QKV/FFN shapes), NVFP4 vs INT8", 1, 1920,
           1920, 65536, 1),
}
C2_MS = (4096, 8192, 16384, 32768, 65536)

# NVFP4 share of the executed GEMM FLOPs on each workload, as the GPU arm realises it (decisions are
# deterministic for the seeded input: the same at every world size). The GPU arm weights its own
# cpu_baseline with its live share; the reference arm (run first on the box, no GPU) uses this.
NVFP4_FLOP_SHARE = {"c4": 0.361, "c3": 0.36, "c5": 0.36, "c1": 0.5, "c2": 0.5}

PAPER_CONTEXT = {"e2e_speedup": 1.92, "e2e_speedup_dmpq_only": 1.36, "memory_reduction_vs_bf16": 3.32,
                 "gpu": "1x NVIDIA RTX 5090 (sm_120)", "model": "CogVideoX (DDIM 50 steps, CFG 6.0)",
                 "cite": "PAPER.md P:40, P:255, P:311, P:336", "comparable": False}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sms.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        # DMPQ_DEVICE_MAP=shared puts every rank on GPU 0 (functional test of the multi-rank
        # path on a 1-GPU box, with DMPQ_DIST_BACKEND=gloo); the contract run uses one GPU per rank.
        dev_index = 0 if os.environ.get("DMPQ_DEVICE_MAP") == "shared" else local
        torch.cuda.set_device(dev_index)
        backend = os.environ.get("DMPQ_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
        return dist.get_rank(), world, dev_index, dist.group.WORLD
    return 0, 1, 0, None


# ------------------------------------------------------------------------------------------ CPU oracle
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


_ORACLE_SAMPLES = {}


def cpu_oracle_sample(H: int, F: int, rows4: int, rows8: int, nvfp4_share: float, hadamard: bool = True,
                      col_frac: int = 4, threads: int = 0, seed: int = 7, shapes=None):
    """Time the CPU oracle (oracle/, plain C, as it stands) on a bounded sample of the workload's
    DMPQ linears: the six layers of one block restricted to 1/col_frac of each layer's output
    channels, `rows4` token rows per thread through the NVFP4 path and `rows8` per thread through
    the INT8 path (quantization incl. the block-Hadamard rotation when on, then the GEMM with its
    epilogue), `threads` (default: all host cores) threads over disjoint row ranges (the oracle is
    row-parallel; ctypes releases the GIL). The two per-format rates are combined with the GPU
    arm's NVFP4 share of the executed FLOPs (time per FLOP weighted by the share).
    Returns (TFLOP/s, seconds of timed CPU wall time, threads, description)."""
    import concurrent.futures as cf
    import numpy as np
    import oracle
    from paper_2603_18742_b200 import synth
    oracle.build()
    threads = threads or os.cpu_count() or 1
    shapes = shapes or [(H, H), (H, H), (H, H), (H, H), (F, H), (H, F)]
    layers = []

    def prep(j):
        n, k = shapes[j]
        w, b = synth.linear_weight(n, k, seed * 16 + j)
        w = w[: n // col_frac].contiguous()
        pk = oracle.pack_weights_hadamard(synth.bits(w)) if hadamard else oracle.pack_weights(synth.bits(w))
        x = synth.dit_activation(threads * max(rows4, rows8), k, seed + j) if j != 5 else \
            synth.ffn2_activation(threads * max(rows4, rows8), k, seed + j)
        xb = synth.bits(x)
        return dict(n=n // col_frac, k=k, pk=pk, b=b[: n // col_frac].numpy().copy(), xb=xb,
                    g=oracle.global_scale(oracle.amax_bf16(xb), 1344.0))

    key = (tuple(shapes), hadamard, col_frac, threads, max(rows4, rows8), seed)
    if key not in _ORACLE_SAMPLES:   # packed weights + inputs, reused by the reference arm's steps
        with cf.ThreadPoolExecutor(threads) as ex:
            _ORACLE_SAMPLES.clear()
            _ORACLE_SAMPLES[key] = list(ex.map(prep, range(len(shapes))))
    layers = _ORACLE_SAMPLES[key]

    def work(fmt, r0, r1):
        for L in layers:
            xb = L["xb"][r0:r1]
            if hadamard:
                y = oracle.fht128(oracle.bf16_to_f32(xb).reshape(r1 - r0, L["k"]))
            pk = L["pk"]
            if fmt == 4:
                c, s = oracle.nvfp4_quantize_f32(y, L["g"]) if hadamard else oracle.nvfp4_quantize(xb, L["g"])
                oracle.gemm_nvfp4(c, s, L["g"], pk["fp4_codes"], pk["fp4_sf"], pk["fp4_g"], L["b"])
            else:
                c, s = oracle.int8_quantize_f32(y) if hadamard else oracle.int8_quantize(xb)
                oracle.gemm_int8(c, s, pk["i8_codes"], pk["i8_scale"], L["b"])

    secs = {}
    flops_row = sum(2.0 * L["n"] * L["k"] for L in layers)
    with cf.ThreadPoolExecutor(threads) as ex:
        for fmt, rows in ((4, rows4), (8, rows8)):
            t0 = time.perf_counter()
            list(ex.map(lambda i: work(fmt, i * rows, (i + 1) * rows), range(threads)))
            secs[fmt] = time.perf_counter() - t0
    rate4 = flops_row * rows4 * threads / secs[4]
    rate8 = flops_row * rows8 * threads / secs[8]
    rate = 1.0 / (nvfp4_share / rate4 + (1.0 - nvfp4_share) / rate8)
    what = "the six linears of one block" if len(shapes) == 6 else f"{len(shapes)} linear layer(s)"
    desc = (f"oracle quantize{'+Hadamard' if hadamard else ''} + GEMM of {what} (H={H}, F={F}), "
            f"1/{col_frac} of each layer's output channels; NVFP4 {rows4 * threads} rows ({secs[4]:.1f} s, "
            f"{rate4 / 1e9:.3f} GFLOP/s), INT8 {rows8 * threads} rows ({secs[8]:.1f} s, {rate8 / 1e9:.2f} GFLOP/s), "
            f"{threads} threads on {cpu_model()}; combined with NVFP4 FLOP share {nvfp4_share:.3f}")
    return rate / 1e12, secs[4] + secs[8], threads, desc


def memory_report(model, args) -> dict:
    """Resident weight and delta-cache bytes of this rank against a BF16 model (P:336's 3.32x is a
    whole-model figure on another GPU: context only)."""
    params = sum(w.n * w.k for blk in model.blocks for w in blk.layers)
    w_bytes = sum(blk.nbytes() for blk in model.blocks)
    cache = sum(d.nbytes() if model.cache_nvfp4 else d.numel() * 2 for d in model.delta)
    return {"linear_params": params, "weights_bf16_bytes": 2 * params, "weights_resident_bytes": w_bytes,
            "weights_ratio_vs_bf16": 2 * params / w_bytes, "delta_cache_bytes": cache,
            "weights_forms": "NVFP4 only (INT8 cast per GEMM into a shared scratch)" if getattr(model, "int8_cast", False)
            else "NVFP4 + INT8 pre-packed"}


def run_sweep(args):
    """C2 (BASELINE configs[1]): one linear layer K = N = 1920 at M = 4K..64K token rows (each
    rank its row shard of every M), NVFP4 and INT8: a step is, for every M and both formats, the
    activation quantization (plain, g = amax/2688 of the tensor itself, R3) and the GEMM with its
    bias epilogue (bf16 output). L2 is flushed (a 512 MB write) before every quantize+GEMM pair;
    the step time is the sum of the pairs' CUDA-event intervals on the launching stream."""
    import torch
    from paper_2603_18742_b200 import build
    from paper_2603_18742_b200 import dmpq as D
    from paper_2603_18742_b200 import synth
    from paper_2603_18742_b200.shard import shard_rows
    build.build()
    rank, world, local, group = dist_setup(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    desc = CONFIGS["c2"][0]
    K = N = 1920
    peaks, peak_kind = load_peaks()
    w, b = synth.linear_weight_device(N, K, seed=args.seed * 16 + 1, device=dev)
    pw = D.dmpq_pack_weights(w, b)
    cases = []
    for M in C2_MS:
        r0, r1 = shard_rows(M, world, rank)
        m = r1 - r0
        X = synth.dit_activation_device(M, K, seed=args.seed + M, device=dev)[r0:r1].contiguous()
        amax = torch.zeros(1, device=dev)
        a8 = D.QuantAct.empty(D.FMT_INT8, m, K, dev)
        D.dmpq_quantize_act(X, out_i8=a8, amax_out=amax)
        if group is not None:   # the tensor's amax over all ranks (setup, not timed)
            torch.distributed.all_reduce(amax, op=torch.distributed.ReduceOp.MAX, group=group)
        g = torch.zeros(1, device=dev)
        D.dmpq_global_scale(amax, 2688.0, g)
        a4 = D.QuantAct.empty(D.FMT_NVFP4, m, K, dev, g=g)
        cases.append(dict(M=M, m=m, X=X, acts={D.FMT_NVFP4: a4, D.FMT_INT8: a8},
                          Y=torch.empty(m, N, dtype=torch.bfloat16, device=dev)))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    fmts = (D.FMT_NVFP4, D.FMT_INT8)

    def barrier():
        if group is not None:
            torch.distributed.barrier(group=group)

    def step(evs):
        for c in cases:
            for f in fmts:
                flush.zero_()
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                a = c["acts"][f]
                e[0].record()
                D.dmpq_quantize_act(c["X"], out_fp4=a if f == D.FMT_NVFP4 else None,
                                    out_i8=a if f == D.FMT_INT8 else None)
                e[1].record()
                D.dmpq_gemm(a, pw, Y=c["Y"])
                e[2].record()
                evs.append((c["M"], c["m"], f, e))

    for _ in range(args.warmup):
        step([])
    torch.cuda.synchronize()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    evs = []
    for _ in range(args.steps):
        step(evs)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    per = {}
    for M, m, f, e in evs:
        d = per.setdefault((M, f), dict(m=m, q=0.0, g=0.0, n=0))
        d["q"] += e[0].elapsed_time(e[1]) * 1e-3
        d["g"] += e[1].elapsed_time(e[2]) * 1e-3
        d["n"] += 1
    local_t = sum(d["q"] + d["g"] for d in per.values()) / args.steps
    local_flops = sum(2.0 * d["m"] * N * K for d in per.values())   # per step

    # e2e through the C ABI with host buffers: pinned H2D of X, quantize, GEMM, D2H of Y
    host = {c["M"]: (c["X"].cpu().pin_memory(), torch.empty(c["m"], N, dtype=torch.bfloat16).pin_memory())
            for c in cases}
    e2e_t = 0.0
    h2d = d2h = 0
    for _ in range(args.steps):
        for c in cases:
            hx, hy = host[c["M"]]
            for f in fmts:
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a = c["acts"][f]
                e0.record()
                c["X"].copy_(hx, non_blocking=True)
                D.dmpq_quantize_act(c["X"], out_fp4=a if f == D.FMT_NVFP4 else None,
                                    out_i8=a if f == D.FMT_INT8 else None)
                D.dmpq_gemm(a, pw, Y=c["Y"])
                hy.copy_(c["Y"], non_blocking=True)
                e1.record()
                torch.cuda.synchronize()
                e2e_t += e0.elapsed_time(e1) * 1e-3
        h2d = sum(c["X"].numel() * 2 for c in cases) * len(fmts)
        d2h = sum(c["Y"].numel() * 2 for c in cases) * len(fmts)
    e2e_t /= args.steps

    def maxsum(a, b_):
        t = torch.tensor([a, b_], dtype=torch.float64, device=dev)
        if group is None:
            return a, b_
        mx, sm = t.clone(), t.clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX, group=group)
        torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM, group=group)
        return float(mx[0]), float(sm[1])

    step_t, flops = maxsum(local_t, local_flops)
    e2e_step_t, _ = maxsum(e2e_t, 0.0)
    if rank != 0:
        if group is not None:
            torch.distributed.destroy_process_group()
        return
    burst = peaks["bf16_tflops"]
    ratio = {D.FMT_NVFP4: 4, D.FMT_INT8: 2}
    name = {D.FMT_NVFP4: "nvfp4", D.FMT_INT8: "int8"}
    sweep = []
    by_fmt = {}
    for (M, f), d in sorted(per.items()):
        n = d["n"]
        gf = 2.0 * d["m"] * N * K
        qb = d["m"] * K * (2 + 0.5 + 1 / 16) if f == D.FMT_NVFP4 else d["m"] * (K * 3 + 4)
        ach = gf / (d["g"] / n) / 1e12
        sweep.append({"M": M, "m_rank": d["m"], "fmt": name[f], "gemm_us": d["g"] / n * 1e6,
                      "quant_us": d["q"] / n * 1e6, "gemm_tflops": ach, "gemm_frac": ach / (burst * ratio[f]),
                      "quant_gbs": qb / (d["q"] / n) / 1e9, "quant_frac": qb / (d["q"] / n) / 1e9 / peaks["hbm_gbs"]})
        bf = by_fmt.setdefault(name[f], dict(flops=0.0, secs=0.0, launches=0))
        bf["flops"] += gf * n
        bf["secs"] += d["g"]
        bf["launches"] += n
    tot_secs = sum(d["q"] + d["g"] for d in per.values())
    for k_, bf in by_fmt.items():
        bf["achieved"] = bf["flops"] / bf["secs"] / 1e12
        bf["peak"] = burst * (4 if k_ == "nvfp4" else 2)
        bf["frac"] = bf["achieved"] / bf["peak"]
        bf["time_share_of_step"] = bf["secs"] / tot_secs
    dom = max(by_fmt, key=lambda k_: by_fmt[k_]["time_share_of_step"])
    d = by_fmt[dom]
    roofline = {"bound": "tensor", "kernel": f"dmpq_gemm ({dom})", "achieved": d["achieved"], "peak": d["peak"],
                "unit": "TFLOP/s", "frac": d["frac"], "traffic": None,
                "peak_source": f"{peak_kind} bf16 burst {burst} TF/s x {4 if dom == 'nvfp4' else 2} (nominal "
                               f"{dom}:bf16 ratio); kernels timed alone between L2 flushes",
                "by_format": {k_: {kk: vv for kk, vv in v.items() if kk not in ("flops", "secs")}
                              for k_, v in by_fmt.items()}}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, secs, threads, sample = cpu_oracle_sample(K, K, 64, 4096, 0.5, hadamard=False, col_frac=1,
                                                     shapes=[(N, K)])
        cpu = {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "oracle", "sample": sample, "seconds": secs}
    line = {
        "metric": METRIC, "value": flops / step_t / 1e12, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "nvfp4+int8 (fp32 accum)", "data": "synthetic (seeded; random-init weights)",
        "config": {"workload": desc, "K": K, "N": N, "M": list(C2_MS), "parallelism": f"token-shard x{world}",
                   "l2": "flushed (512 MB write) before every quantize+GEMM pair",
                   "quantizer": "plain (no Hadamard), g = amax/2688 of the tensor (R3)"},
        "sweep": sweep,
        "gpu_launches": len(evs) * 2,
        "clocks": clk,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": flops / e2e_step_t / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d * world,
                "d2h_bytes_per_step": d2h * world,
                "copies": "pinned host X -> device, quantize, GEMM, Y -> pinned host, serialised per pair"},
        "paper_context": PAPER_CONTEXT,
    }
    print(json.dumps(line))
    if group is not None:
        torch.distributed.destroy_process_group()


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on this workload's metric (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    desc, nb, H, F, M, T = CONFIGS[args.config][:6]
    share = NVFP4_FLOP_SHARE.get(args.config, 0.5)
    vals = []
    if args.config == "c2":   # one K = N = 1920 layer, plain quantizer (run_sweep)
        kw = dict(hadamard=False, col_frac=1, shapes=[(H, H)])
        big = (8, 512)
    else:
        kw = dict(hadamard=not args.no_hadamard)
        big = (1, 64)
    for _ in range(args.warmup):
        cpu_oracle_sample(H, F, *big, share, **kw)
    for _ in range(args.steps):
        v, t, threads, sample = cpu_oracle_sample(H, F, *big, share, **kw)
        vals.append((v, t))
    v = sum(x[0] for x in vals) / len(vals)
    step_s = sum(x[1] for x in vals) / len(vals)
    line = {
        "impl": "reference", "metric": METRIC,
        "value": v, "unit": "TFLOP/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64 (oracle accumulation of nvfp4/int8 codes)", "data": "synthetic",
        "config": {"workload": desc, "nvfp4_flop_share": share,
                   "nvfp4_flop_share_source": "the GPU arm's realised share on this workload (deterministic "
                                              "decisions; DESIGN.md §8)"},
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------------------------ ours
def run_ours(args):
    import torch
    from paper_2603_18742_b200 import build
    from paper_2603_18742_b200 import dmpq as D
    from paper_2603_18742_b200 import synth
    from paper_2603_18742_b200.block import DiTStack
    from paper_2603_18742_b200.shard import shard_rows
    from paper_2603_18742_b200._lib import TDC_METRIC_COS as L_TDC_COS, TDC_METRIC_REL_L2 as L_TDC_REL_L2

    build.build()
    rank, world, local, group = dist_setup(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    desc, nb, H, F, M, T = CONFIGS[args.config]
    if args.config == "c2":
        return run_sweep(args)
    if args.blocks:
        nb = args.blocks
    r0, r1 = shard_rows(M, world, rank)
    m = r1 - r0
    if args.rank_share:   # development: one rank's share of an N-GPU run, on one GPU (no exchange)
        r0, r1 = shard_rows(M, args.rank_share, 0)
        m = r1 - r0
    T = max(T, args.warmup + args.steps)
    peaks, peak_kind = load_peaks()

    tdc_cfg = (0.001, args.tdc_tau if args.tdc_tau is not None else 0.003, 2,
               {"cos": L_TDC_COS, "rel_l2": L_TDC_REL_L2}[args.tdc_metric])
    model = DiTStack(nb, H, F, m, dev, seed=args.seed, group=group, hadamard=not args.no_hadamard, tdc_cfg=tdc_cfg,
                     pdr={None: False, "delayed": True, "current": "current"}[args.pdr], m_total=M, cache_nvfp4=args.cache_nvfp4, fuse_refresh=args.fused_refresh,
                     int8_cast=args.int8_cast, int8_block=args.int8_block, fuse_quant=args.fuse_quant,
                     overlap_refresh=args.overlap_refresh, g_policy=args.g_policy)
    # block-0 input trajectory basis: ONE seeded global [M x H] input, of which this rank takes its
    # contiguous row shard -- every world size solves the same problem (same mix, same decisions)
    A, B = synth.trajectory_basis(M, H, seed=1000 + args.seed, device=dev)
    A, B = A[r0:r1].clone(), B[r0:r1].clone()
    torch.cuda.empty_cache()

    def x_at(t):
        return synth.trajectory_input(A, B, t, T)

    steps_inputs = {t: x_at(t) for t in range(args.warmup + args.steps)}
    torch.cuda.synchronize()

    def barrier():
        if group is not None:
            torch.distributed.barrier(group=group)

    def allmax_sum(vals):
        """(max over ranks of vals[0], sum over ranks of vals[1])"""
        tt = torch.tensor(vals, dtype=torch.float64, device=dev)
        if group is None:
            return float(tt[0]), float(tt[1])
        mx, sm = tt.clone(), tt.clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX, group=group)
        torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM, group=group)
        return float(mx[0]), float(sm[1])

    def warmup():
        """W untimed steps from a fresh state (TDC warm-up, graph capture, first launches)."""
        model.reset_state()
        for t in range(args.warmup):
            model.step(steps_inputs[t], t)
            model.end_step(t)
        torch.cuda.synchronize()
        barrier()

    # ---- pass A (headline): K timed steps, device-resident inputs, CUDA graphs per block pattern
    model.use_graphs = not args.no_graphs
    warmup()
    launches0 = model.launches
    rec0 = len(model.records)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.perf_counter()
    ev0.record()
    host_issue = 0.0
    for i in range(args.steps):
        t = args.warmup + i
        h0 = time.perf_counter()
        model.step(steps_inputs[t], t)      # enqueues the step (no synchronisation)
        host_issue += time.perf_counter() - h0
        model.end_step(t)
    ev1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    barrier()
    clk = clocks.stop()
    elapsed = ev0.elapsed_time(ev1) * 1e-3
    launches = model.launches - launches0
    recs = model.records[rec0:]
    local_flops = sum(r.linear_flops for r in recs)
    mix = model.mix(recs)

    # every rank must have taken identical TDC/routing decisions
    sig = float(sum((i + 1) * (2 + d + sum(f or [])) for r in recs for i, (d, f) in enumerate(zip(r.decisions, r.fmts))))
    if group is not None:
        s = torch.tensor([sig, -sig], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(s, op=torch.distributed.ReduceOp.MAX, group=group)
        assert float(s[0]) == sig and float(s[1]) == -sig, "ranks disagree on the per-step decisions"
    elapsed, total_flops = allmax_sum([elapsed, local_flops])
    value = total_flops / elapsed / 1e12
    dense_flops = 2.0 * M * (4 * H * H + 2 * H * F) * nb * args.steps

    # ---- pass B: the same timesteps again, launched eagerly with CUDA events around every
    # GEMM and every quantize / TDC kernel on the launching stream (roofline + breakdown)
    model.use_graphs = False
    warmup()
    model.timing = True
    model.reset_timing()
    eb0, eb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eb0.record()
    for i in range(args.steps):
        t = args.warmup + i
        model.step(steps_inputs[t], t)
        model.end_step(t)
    eb1.record()
    torch.cuda.synchronize()
    model.timing = False
    elapsed_b = eb0.elapsed_time(eb1) * 1e-3
    gemm_t = model.gemm_time_s()
    gemm_flops = dict(model.gemm_flops)
    brk = model.breakdown_s()
    breakdown = {"gemm": sum(v[0] for v in gemm_t.values()) / args.steps * 1e3,
                 "quantize": brk["quantize"] / args.steps * 1e3, "tdc": brk["tdc"] / args.steps * 1e3,
                 "exchange": brk["exchange"] / args.steps * 1e3, "int8_cast": brk["cast"] / args.steps * 1e3}
    breakdown["host_gaps_and_other"] = elapsed_b / args.steps * 1e3 - sum(breakdown.values())
    breakdown["pass"] = "eager replay of the timed steps with per-launch CUDA events"
    # in-step HBM-bound kernels: algorithmic bytes / their CUDA-event time, against the measured copy peak
    hbm_kernels = {}
    for kind in ("quantize", "tdc", "cast"):
        secs = brk[kind]
        if secs > 0:
            gbs = model.hbm_bytes[kind] / secs / 1e9
            hbm_kernels[kind] = {"bytes_per_step": model.hbm_bytes[kind] / args.steps, "ms_per_step": secs / args.steps * 1e3,
                                 "achieved_gbs": gbs, "peak_gbs": peaks["hbm_gbs"], "frac": gbs / peaks["hbm_gbs"]}

    # ---- pass C (e2e): the same steps through host buffers (pinned H2D of each step's input,
    # D2H of its output), graphs as in pass A. The copies run on a second stream, double-
    # buffered: step t+1's input uploads and step t's output downloads while step t computes.
    host_in = {t: steps_inputs[t].cpu().pin_memory() for t in steps_inputs}
    host_out = torch.empty(m, H, dtype=torch.bfloat16).pin_memory()
    model.use_graphs = not args.no_graphs
    warmup()
    flops2_0 = sum(r.linear_flops for r in model.records)
    main = torch.cuda.current_stream(dev)
    cs = torch.cuda.Stream(device=dev)
    dev_in = [torch.empty(m, H, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    out_stage = torch.empty(m, H, dtype=torch.bfloat16, device=dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    ev_out, ev_out_done = torch.cuda.Event(), torch.cuda.Event()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    cs.wait_event(e0)
    with torch.cuda.stream(cs):
        dev_in[0].copy_(host_in[args.warmup], non_blocking=True)
        ev_in[0].record(cs)
    for i in range(args.steps):
        t = args.warmup + i
        b = i % 2
        if i + 1 < args.steps:   # upload the next step's input into the other buffer
            with torch.cuda.stream(cs):
                if i >= 1:
                    cs.wait_event(ev_used[1 - b])
                dev_in[1 - b].copy_(host_in[t + 1], non_blocking=True)
                ev_in[1 - b].record(cs)
        main.wait_event(ev_in[b])
        out = model.step(dev_in[b], t)
        ev_used[b].record(main)
        if i >= 1:
            main.wait_event(ev_out_done)      # the previous download has read out_stage
        out_stage.copy_(out, non_blocking=True)
        ev_out.record(main)
        with torch.cuda.stream(cs):
            cs.wait_event(ev_out)
            host_out.copy_(out_stage, non_blocking=True)
            ev_out_done.record(cs)
        model.end_step(t)
    main.wait_stream(cs)
    e1.record(main)
    torch.cuda.synchronize()
    e2e_t = e0.elapsed_time(e1) * 1e-3
    e2e_flops = sum(r.linear_flops for r in model.records) - flops2_0
    e2e_t, e2e_flops = allmax_sum([e2e_t, e2e_flops])
    e2e_val = e2e_flops / e2e_t / 1e12

    if rank != 0:
        if group is not None:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (the GEMM format with the most time)
    sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    by_fmt = {}
    for f, name, ratio in ((D.FMT_NVFP4, "nvfp4", 4), (D.FMT_INT8, "int8", 2), (D.FMT_BF16, "bf16", 1)):
        secs, n = gemm_t[f]
        if n:
            ach = gemm_flops[f] / secs / 1e12
            by_fmt[name] = {"achieved": ach, "peak": sus * ratio, "frac": ach / (sus * ratio), "launches": n,
                            "avg_launch_us": secs / n * 1e6, "time_share_of_step": secs / elapsed_b,
                            "frac_vs_burst": ach / (peaks["bf16_tflops"] * ratio),
                            "frac_vs_nominal": ach / (2250.0 * ratio)}
    dom = max(by_fmt, key=lambda k: by_fmt[k]["time_share_of_step"]) if by_fmt else None
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if dom and os.path.exists(tr_path):
        traffic = json.load(open(tr_path)).get(f"{args.config}_{dom}")
    roofline = None
    if dom:
        d = by_fmt[dom]
        roofline = {"bound": "tensor", "kernel": f"dmpq_gemm ({dom})", "achieved": d["achieved"], "peak": d["peak"],
                    "unit": "TFLOP/s", "frac": d["frac"], "traffic": traffic,
                    "peak_source": f"{peak_kind} bf16 sustained {sus} TF/s x {dict(nvfp4=4, int8=2, bf16=1)[dom]} "
                                   f"(nominal {dom}:bf16 ratio); the sustained bf16 figure was measured with cuBLAS "
                                   f"power-capped at a median {peaks.get('clocks_under_load', {}).get('sm_mhz_median')} MHz, "
                                   f"so a kernel running at higher clocks can exceed it: see frac_vs_burst / frac_vs_nominal",
                    "by_format": by_fmt,
                    "timing": "CUDA events around every GEMM launch on its stream, eager replay of the timed steps"}

    # ---- optional bounds: all-NVFP4 and all-INT8 steps without TDC skips
    bounds = None
    if args.bounds:
        bounds = {}
        for name, fmt in (("all_nvfp4_no_skip", D.FMT_NVFP4), ("all_int8_no_skip", D.FMT_INT8)):
            model.force_fmt, model.tdc_enabled = fmt, False
            warmup()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record()
            fl0 = sum(r.linear_flops for r in model.records)
            for i in range(args.steps):
                t = args.warmup + i
                model.step(steps_inputs[t], t)
                model.end_step(t)
            b1.record()
            torch.cuda.synchronize()
            bt, bfl = allmax_sum([b0.elapsed_time(b1) * 1e-3, sum(r.linear_flops for r in model.records) - fl0])
            bounds[name] = {"ms_per_step": bt / args.steps * 1e3, "tflops": bfl / bt / 1e12}
        model.force_fmt, model.tdc_enabled = None, True

    cpu = None
    f4_share = gemm_flops[D.FMT_NVFP4] / max(1.0, sum(gemm_flops.values()))
    if world == 1 and not args.no_cpu_baseline:
        v, secs, threads, sample = cpu_oracle_sample(H, F, 8, 512, f4_share, hadamard=not args.no_hadamard)
        cpu = {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "oracle", "sample": sample, "seconds": secs}

    line = {
        "metric": METRIC,
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "nvfp4+int8 (fp32 accum)", "data": "synthetic (seeded; random-init weights)",
        "config": {"workload": desc, "blocks": nb, "hidden": H, "ffn": F, "tokens_total": M, "tokens_per_rank": m,
                   "timesteps": list(range(args.warmup, args.warmup + args.steps)), "T": T,
                   "parallelism": f"token-shard x{world}",
                   "device_map": os.environ.get("DMPQ_DEVICE_MAP", "one GPU per rank"),
                   "input": "one seeded global input; each rank takes its contiguous row shard", "l2": "inputs larger than L2 (multi-GB working set per step)",
                   "cuda_graphs": not args.no_graphs, "tdc_refresh": "fused in the FFN2 GEMM epilogue" if model.fuse_refresh else "own kernel",
                   "hadamard": not args.no_hadamard, "pdr_outlier_gate": args.pdr or False, "int8_weight_cast": args.int8_cast, "producer_fused_quant": model.fuse_quant, "nvfp4_g_policy": args.g_policy,
                   "tdc": {"rho": tdc_cfg[0], "tau": tdc_cfg[1], "n_max": tdc_cfg[2], "metric": args.tdc_metric},
                   "tdc_refresh_overlap": model.overlap_refresh,
                   "int8_granularity": "per 128-block (R17)" if args.int8_block else "per token (R2)",
                   "delta_cache": {"format": "nvfp4" if args.cache_nvfp4 else "bf16",
                                   "bytes_per_rank": sum(d.nbytes() if args.cache_nvfp4 else d.numel() * 2
                                                         for d in model.delta)},
                   "mix": dict(mix, nvfp4_flop_share=f4_share)},
        "block_step_ms": elapsed / args.steps / nb * 1e3,
        "memory": memory_report(model, args),
        "paper_context": PAPER_CONTEXT,
        "bounds": bounds,
        "breakdown_ms_per_step": breakdown,
        "hbm_kernels_in_step": hbm_kernels,
        "effective_tflops_dense_equiv": dense_flops / elapsed / 1e12,
        "wall_s_timed": wall,
        "host_issue_ms_per_step": host_issue / args.steps * 1e3,
        "gpu_launches": launches,
        "clocks": clk,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": m * H * 2 * world,
                "d2h_bytes_per_step": m * H * 2 * world + nb * 7 * 8 * world,
                "copies": "pinned host buffers on a second stream, double-buffered against the compute"},
    }
    print(json.dumps(line))
    if group is not None:
        torch.distributed.destroy_process_group()


def relaunch(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1. With fewer than N visible GPUs the ranks share GPU 0 over
    gloo (a functional run of the multi-rank path, flagged in config.device_map, not a scaling
    measurement)."""
    import socket
    import torch
    env = dict(os.environ)
    if torch.cuda.device_count() < n:
        env.setdefault("DMPQ_DEVICE_MAP", "shared")
        env.setdefault("DMPQ_DIST_BACKEND", "gloo")
    sck = socket.socket()
    sck.bind(("127.0.0.1", 0))
    port = sck.getsockname()[1]
    sck.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--blocks", type=int, default=0, help="override the block count (development only)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="launch every kernel eagerly (no CUDA graphs)")
    ap.add_argument("--no-hadamard", action="store_true", help="disable the online block-Hadamard smoothing (P:187)")
    ap.add_argument("--pdr", nargs="?", const="delayed", default=None, choices=["delayed", "current"],
                    help="enable the Purified Cache Refresh outlier gate (P:241, NEXT-3; off by default: the north_star "
                    "path is DMPQ + TDC): 'delayed' (R15, all-rank R of the last computed step, host decision) or "
                    "'current' (R18, this step's input, decided on the device, both GEMM kinds predicated)")
    ap.add_argument("--rank-share", type=int, default=0, help="development: time one rank's token share of an "
                    "N-GPU run on this GPU (host-overhead study; not a bench line)")
    ap.add_argument("--bounds", action="store_true", help="also time all-NVFP4 and all-INT8 steps without skips "
                    "(SURVEY 8(d) bounds)")
    ap.add_argument("--fused-refresh", action="store_true", help="run the TDC refresh in the FFN2 GEMM epilogue "
                    "instead of its own kernel (SURVEY NEXT-2; measured slower, DESIGN.md 5.7c)")
    ap.add_argument("--int8-block", action="store_true", help="per-block symmetric INT8 activations over the 128-element "
                    "Hadamard blocks (P:187, R17, NEXT-1) instead of per-token INT8")
    ap.add_argument("--overlap-refresh", action="store_true", help="run each block's TDC refresh on a side stream "
                    "overlapped with the next block (measured no faster; DESIGN.md 5.4)")
    ap.add_argument("--g-policy", default="delayed", choices=["delayed", "current"], help="NVFP4 per-tensor scale "
                    "(R3): delayed (previous step's amax / 1344, the default) or current (an amax pass over each "
                    "NVFP4-quantized input first, amax / 2688; single rank)")
    ap.add_argument("--tdc-metric", default="cos", choices=["cos", "rel_l2"], help="the distance D of Eq. 9 (P:215): "
                    "1 - CosSim (the paper's default) or the relative-L2 distance (R19)")
    ap.add_argument("--tdc-tau", type=float, default=None, help="TDC threshold tau (P:255: 0.003)")
    ap.add_argument("--fuse-quant", action="store_true", help="producer-fused NVFP4 quantization of the FFN2 input in "
                    "FFN1's epilogue (P:336, NEXT-2; plain quantizer only, i.e. with --no-hadamard)")
    ap.add_argument("--cache-nvfp4", action="store_true", help="NVFP4-compressed TDC delta cache (P:226, R16, NEXT-4)")
    ap.add_argument("--int8-cast", action="store_true",
                    help="NVFP4-only weight residency, INT8 codes cast on the fly per INT8 GEMM into an L2-resident "
                    "scratch (P:184, NEXT-4b): 3.5x less weight memory than BF16; same-box 0.5 %% slower at full size, "
                    "6 %% at one rank's share of 8 GPUs (DESIGN.md 5.7b). Default: both forms pre-packed (north_star)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: the contract needs --warmup >= 3", file=sys.stderr)
    world_env = os.environ.get("WORLD_SIZE")
    if args.impl == "ours" and args.gpus > 1 and world_env is None:
        sys.exit(relaunch(args.gpus))
    if args.impl == "ours" and world_env is not None and int(world_env) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
