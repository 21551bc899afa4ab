"""Multi-rank tests of the token-sharded path on one GPU (every rank on cuda:0, gloo):

- bench.py --gpus 2 launches its own two ranks (no external launcher), every rank takes
  identical decisions (bench asserts it) and rank 0 prints one JSON line;
- SURVEY §4 T3: a W = 2 token-sharded DiTStack run equals the W = 1 run -- concatenated
  shard outputs of every step and delta caches bit for bit, NVFP4 global scales bit for bit
  (the maxima travel exactly through the single SUM collective), routing / TDC decisions
  identical, FP64 statistics equal up to the re-association of the per-shard sums (R12)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_launches_two_ranks():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--config", "c1"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["tokens_per_rank"] == 128 and d["value"] > 0


M, H, F, NB, T = 1030, 128, 512, 2, 7


def _run_stack(world, rank, q, port):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2603_18742_b200 import build, synth
    from paper_2603_18742_b200.block import DiTStack
    from paper_2603_18742_b200.shard import shard_rows
    build.build()
    group = None
    if world > 1:
        os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        group = dist.group.WORLD
    torch.cuda.set_device(0)
    r0, r1 = shard_rows(M, world, rank)
    stack = DiTStack(NB, H, F, r1 - r0, "cuda", seed=6, gate_scales=[0.008, 0.012], hadamard=True, group=group,
                     m_total=M, tdc_cfg=(0.001, 0.02, 2))
    stack.use_graphs = True
    A, B = synth.trajectory_basis(M, H, seed=9)
    outs, stats, gs = [], [], []
    for t in range(T):
        x = synth.trajectory_input(A[r0:r1], B[r0:r1], t, 50).cuda()
        outs.append(stack.step(x, t).cpu().clone())
        stats.append(stack.end_step(t).copy())
        gs.append(stack.g_table.cpu().clone())
    # numpy payloads (pickled by value: torch tensors would travel as shared-memory handles that
    # die with this process)
    res = dict(rank=rank, outs=[synth.bits(o) for o in outs], stats=stats, g=[x.numpy() for x in gs],
               delta=[synth.bits(d.cpu()) for d in stack.delta],
               dec=[r.decisions for r in stack.records], fmts=[r.fmts for r in stack.records])
    q.put(res)
    if world > 1:
        dist.destroy_process_group()


def _spawn(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_run_stack, args=(world, r, q, port)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_token_shard_w2_equals_w1():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    one, = _spawn(1)
    two = _spawn(2)
    assert two[0]["dec"] == two[1]["dec"] == one["dec"]
    assert two[0]["fmts"] == two[1]["fmts"] == one["fmts"]
    assert any(d == 1 for ds in one["dec"] for d in ds), "the trajectory should skip"
    assert {f for fs in one["fmts"] for ff in fs if ff for f in ff} >= {0, 1}, "both formats should run"
    for t in range(T):
        assert np.array_equal(np.concatenate([two[0]["outs"][t], two[1]["outs"][t]]), one["outs"][t]), t
        assert np.array_equal(two[0]["g"][t], one["g"][t]) and np.array_equal(two[1]["g"][t], one["g"][t]), t
        assert np.array_equal(two[0]["stats"][t], two[1]["stats"][t])          # identical on every rank
        np.testing.assert_allclose(two[0]["stats"][t], one["stats"][t], rtol=1e-12, atol=1e-300)
    for b in range(NB):
        assert np.array_equal(np.concatenate([two[0]["delta"][b], two[1]["delta"][b]]), one["delta"][b])
