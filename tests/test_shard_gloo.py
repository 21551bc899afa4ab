"""Token sharding + the per-step statistics exchange on CPU (gloo, world size 2).

Each rank computes the oracle's block statistics on its own contiguous row shard,
fills its slot, and the exchange (SUM all-reduce of zero-padded slots + MAX
all-reduce of amax, rank-ordered combine) must give every rank bit-identical
global statistics equal to the unsharded statistics, hence identical routing and
TDC decisions."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_18742_b200.shard import SlotBuffer, exchange, shard_rows


def test_shard_rows_partition():
    for M in (1, 7, 256, 17776, 35552, 119056):
        for W in (1, 2, 3, 4, 8):
            rows = [shard_rows(M, W, r) for r in range(W)]
            assert rows[0][0] == 0 and rows[-1][1] == M
            assert all(rows[i][1] == rows[i + 1][0] for i in range(W - 1))
            sizes = [b - a for a, b in rows]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(M, H, nb):
    from paper_2603_18742_b200 import synth
    out = []
    for b in range(nb):
        xi = synth.dit_activation(M, H, seed=10 + b, outlier_frac=0, tail_frac=0)
        xo = (xi.float() + (0.004 * (b + 1)) * synth.dit_activation(M, H, seed=20 + b, outlier_frac=0,
                                                                    tail_frac=0).float()).to(torch.bfloat16)
        dp = ((0.004 * (b + 1)) * synth.dit_activation(M, H, seed=30 + b, outlier_frac=0, tail_frac=0).float()).to(torch.bfloat16)
        out.append((xi, xo, dp))
    return out


def _worker(rank, world, port, M, H, nb, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2603_18742_b200 import dmpq as D, synth
    r0, r1 = shard_rows(M, world, rank)
    slots = SlotBuffer(world, rank, nb * 7, nb * 4, "cpu")
    stats_view = slots.stats.view(world, nb, 7)
    amax = torch.zeros(nb, 4, dtype=torch.float32)
    for b, (xi, xo, dp) in enumerate(_inputs(M, H, nb)):
        _, st = oracle.block_stats(synth.bits(xi[r0:r1]), synth.bits(xo[r0:r1]), synth.bits(dp[r0:r1]))
        stats_view[rank, b] = torch.from_numpy(st)
        amax[b, 0] = oracle.amax_bf16(synth.bits(xi[r0:r1]))
        amax[b, 1] = oracle.amax_bf16(synth.bits(xo[r0:r1]))
    stats = exchange(slots, amax, dist.group.WORLD).reshape(nb, 7)
    taus = [D.dmpq_derive_tau(0.1 * (1 + j / 2), 0.001, 0.0025) for j in range(6)]
    fmts = [D.dmpq_predict(stats[b], taus, 3, False)[0] for b in range(nb)]
    q.put((rank, stats, amax.numpy().copy(), fmts))
    dist.destroy_process_group()


def test_exchange_gloo_world2(orc):
    M, H, nb, world = 301, 64, 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, H, nb, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # bit-identical on every rank
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][2], res[1][2])
    assert res[0][3] == res[1][3]
    # equal to the unsharded statistics (FP64 sums, re-associated across the shard boundary)
    from paper_2603_18742_b200 import dmpq as D, synth
    taus = [D.dmpq_derive_tau(0.1 * (1 + j / 2), 0.001, 0.0025) for j in range(6)]
    for b, (xi, xo, dp) in enumerate(_inputs(M, H, nb)):
        _, st = orc.block_stats(synth.bits(xi), synth.bits(xo), synth.bits(dp))
        np.testing.assert_allclose(res[0][1][b], st, rtol=1e-12)
        assert res[0][2][b, 0] == orc.amax_bf16(synth.bits(xi))
        assert res[0][2][b, 1] == orc.amax_bf16(synth.bits(xo))
        assert res[0][3][b] == orc.route_block(orc.gamma_from_stats(st), taus, 3, False)
