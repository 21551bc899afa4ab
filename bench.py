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

CONFIGS = {
    # name: (description, n_blocks, H, F, M_total, T)
    "c4": ("CogVideoX-5B 42-block step, hidden 3072, 49f 480x720 (17,776 tok) x CFG 2, 50-step TDC", 42, 3072, 12288,
           2 * 17776, 50),
    "c3": ("CogVideoX-2B 30-block step, hidden 1920, 49f 480x720 (17,776 tok) x CFG 2", 30, 1920, 7680, 2 * 17776, 50),
    "c5": ("HunyuanVideo-shaped blocks, hidden 3072, 720p x 129f (119,056 tok)", 8, 3072, 12288, 119056, 50),
    "c1": ("one DiT block, hidden 128, 256 tokens, 4 timesteps", 1, 128, 512, 256, 4),
}


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
def cpu_oracle_sample(H: int, F: int, rows: int, nvfp4_frac: float, seed: int = 7):
    """Time the CPU oracle (oracle/, single-threaded C) on a bounded sample: the
    quantizers and the six DMPQ linears of one block for `rows` token rows, each
    layer in both formats, combined with the realised NVFP4 share. Returns
    (linear TFLOP/s, seconds, description)."""
    import numpy as np
    import oracle
    from paper_2603_18742_b200 import synth
    oracle.build()
    shapes = [(H, H), (H, H), (H, H), (H, H), (F, H), (H, F)]
    t4 = t8 = 0.0
    flops = 0.0
    for j, (n, k) in enumerate(shapes):
        w, b = synth.linear_weight(n, k, seed * 16 + j)
        pk = oracle.pack_weights(synth.bits(w))
        x = synth.dit_activation(rows, k, seed + j) if j != 5 else synth.ffn2_activation(rows, k, seed + j)
        xb = synth.bits(x)
        g = oracle.global_scale(oracle.amax_bf16(xb), 1344.0)
        t0 = time.perf_counter()
        c4, s4 = oracle.nvfp4_quantize(xb, g)
        oracle.gemm_nvfp4(c4, s4, g, pk["fp4_codes"], pk["fp4_sf"], pk["fp4_g"], b.numpy())
        t1 = time.perf_counter()
        c8, s8 = oracle.int8_quantize(xb)
        oracle.gemm_int8(c8, s8, pk["i8_codes"], pk["i8_scale"], b.numpy())
        t2 = time.perf_counter()
        t4 += t1 - t0
        t8 += t2 - t1
        flops += 2.0 * rows * n * k
    t = nvfp4_frac * t4 + (1 - nvfp4_frac) * t8
    return flops / t / 1e12, t, (f"quantize + six DMPQ linears of one block (H={H}, F={F}) on {rows} token rows, "
                                 f"NVFP4 {t4:.1f}s / INT8 {t8:.1f}s weighted by NVFP4 share {nvfp4_frac:.2f}")


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on this workload's metric."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    desc, nb, H, F, M, T = CONFIGS[args.config]
    rows = 4
    vals = []
    for _ in range(args.warmup):
        cpu_oracle_sample(H, F, rows, 0.5)
    for _ in range(args.steps):
        v, t, sample = cpu_oracle_sample(H, F, rows, 0.5)
        vals.append((v, t))
    v = sum(x[0] for x in vals) / len(vals)
    step_s = sum(x[1] for x in vals) / len(vals)
    line = {
        "impl": "reference", "metric": "DMPQ linear TFLOPS (% FP4/INT8 peak) + block-step ms, CogVideoX-5B, 1/2/4/8 B200",
        "value": v, "unit": "TFLOP/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64 (oracle accumulation of nvfp4/int8 codes)", "data": "synthetic",
        "config": {"workload": desc, "sample_rows": rows, "nvfp4_share_assumed": 0.5},
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": 1, "kind": "oracle", "sample": sample},
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

    build.build()
    rank, world, local, group = dist_setup(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    desc, nb, H, F, M, T = CONFIGS[args.config]
    if args.blocks:
        nb = args.blocks
    r0, r1 = shard_rows(M, world, rank)
    m = r1 - r0
    if args.rank_share:   # development: one rank's share of an N-GPU run, on one GPU (no exchange)
        r0, r1 = shard_rows(M, args.rank_share, 0)
        m = r1 - r0
    T = max(T, args.warmup + args.steps)
    peaks, peak_kind = load_peaks()

    model = DiTStack(nb, H, F, m, dev, seed=args.seed, group=group, hadamard=not args.no_hadamard,
                     pdr=args.pdr, m_total=M, cache_nvfp4=args.cache_nvfp4, fuse_refresh=args.fused_refresh)
    # block-0 input trajectory basis (this rank's rows)
    A, B = synth.trajectory_basis(m, H, seed=1000 + rank, device=dev)

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
                 "exchange": brk["exchange"] / args.steps * 1e3}
    breakdown["host_gaps_and_other"] = elapsed_b / args.steps * 1e3 - sum(breakdown.values())
    breakdown["pass"] = "eager replay of the timed steps with per-launch CUDA events"

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
    if world == 1 and not args.no_cpu_baseline:
        v, secs, sample = cpu_oracle_sample(H, F, 4, mix["nvfp4_layer_frac"])
        cpu = {"value": v, "unit": "TFLOP/s", "cores": 1, "kind": "oracle", "sample": sample, "seconds": secs}

    line = {
        "metric": "DMPQ linear TFLOPS (% FP4/INT8 peak) + block-step ms, CogVideoX-5B, 1/2/4/8 B200",
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "nvfp4+int8 (fp32 accum)", "data": "synthetic (seeded; random-init weights)",
        "config": {"workload": desc, "blocks": nb, "hidden": H, "ffn": F, "tokens_total": M, "tokens_per_rank": m,
                   "timesteps": list(range(args.warmup, args.warmup + args.steps)), "T": T,
                   "parallelism": f"token-shard x{world}", "l2": "inputs larger than L2 (multi-GB working set per step)",
                   "cuda_graphs": not args.no_graphs, "tdc_refresh": "fused in the FFN2 GEMM epilogue" if model.fuse_refresh else "own kernel",
                   "hadamard": not args.no_hadamard, "pdr_outlier_gate": args.pdr,
                   "delta_cache": {"format": "nvfp4" if args.cache_nvfp4 else "bf16",
                                   "bytes_per_rank": sum(d.nbytes() if args.cache_nvfp4 else d.numel() * 2
                                                         for d in model.delta)},
                   "mix": mix},
        "block_step_ms": elapsed / args.steps / nb * 1e3,
        "bounds": bounds,
        "breakdown_ms_per_step": breakdown,
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
    ap.add_argument("--pdr", action="store_true", help="enable the Purified Cache Refresh outlier gate (P:241, "
                    "NEXT-3; off by default: the north_star path is DMPQ + TDC)")
    ap.add_argument("--rank-share", type=int, default=0, help="development: time one rank's token share of an "
                    "N-GPU run on this GPU (host-overhead study; not a bench line)")
    ap.add_argument("--bounds", action="store_true", help="also time all-NVFP4 and all-INT8 steps without skips "
                    "(SURVEY 8(d) bounds)")
    ap.add_argument("--fused-refresh", action="store_true", help="run the TDC refresh in the FFN2 GEMM epilogue "
                    "instead of its own kernel (SURVEY NEXT-2; measured slower, DESIGN.md 5.7c)")
    ap.add_argument("--cache-nvfp4", action="store_true", help="NVFP4-compressed TDC delta cache (P:226, R16, NEXT-4)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: the contract needs --warmup >= 3", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
