"""Seeded synthetic inputs shaped like the paper's workloads.

Shared by the tests, bench.py and the oracle-side checks. Holds NO arithmetic of
the method (no quantization, no statistics): only random tensors. All tensors
are generated on the CPU with torch.Generator so both sides see identical bytes.
"""
from __future__ import annotations

import math

import torch


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def dit_activation(m: int, k: int, seed: int, outlier_frac: float = 0.005, tail_frac: float = 0.01) -> torch.Tensor:
    """Video-DiT-like linear-layer input (bf16 [m, k]): N(0,1) base, a per-token
    LogNormal(0, 0.5) magnitude (so per-token INT8 scales vary), 0.5% outlier
    channels scaled by U(10, 50) (DiT channel outliers) and
    Student-t(4) tails on 1% of entries."""
    g = _gen(seed)
    x = torch.randn(m, k, generator=g)
    x *= torch.exp(0.5 * torch.randn(m, 1, generator=g))
    n_out = max(1, int(round(outlier_frac * k)))
    ch = torch.randperm(k, generator=g)[:n_out]
    x[:, ch] *= 10 + 40 * torch.rand(n_out, generator=g)
    if tail_frac > 0:
        mask = torch.rand(m, k, generator=g) < tail_frac
        # Student-t(4): normal / sqrt(chi2_4 / 4)
        z = torch.randn(m, k, generator=g)
        chi = (torch.randn(m, k, 4, generator=g) ** 2).sum(-1)
        x = torch.where(mask, z / torch.sqrt(chi / 4), x)
    return x.to(torch.bfloat16)


def ffn2_activation(m: int, k: int, seed: int) -> torch.Tensor:
    """FFN2 input: GELU-tanh of an FFN1-like tensor (skewed, mostly >= -0.17)."""
    x = dit_activation(m, k, seed).float()
    return torch.nn.functional.gelu(x, approximate="tanh").to(torch.bfloat16)


def linear_weight(n: int, k: int, seed: int):
    """nn.Linear-like weights W ~ N(0, 1/k) (bf16 [n, k]) and bias ~ N(0, 0.02) (fp32 [n])."""
    g = _gen(seed)
    w = (torch.randn(n, k, generator=g) / math.sqrt(k)).to(torch.bfloat16)
    b = 0.02 * torch.randn(n, generator=g)
    return w, b


def adversarial_rows(k: int) -> torch.Tensor:
    """Edge-case rows for the quantizers: zero rows, +-0, constant rows, tiny and
    huge magnitudes, blocks whose E4M3 scale is subnormal, a reciprocal near-tie."""
    rows = []
    rows.append(torch.zeros(k))
    r = torch.zeros(k); r[1::2] = -0.0; rows.append(r)
    rows.append(torch.full((k,), 3.0))
    rows.append(torch.full((k,), -1e-30))
    r = torch.full((k,), 1e30); r[::3] = -2e29; rows.append(r)
    r = torch.randn(k, generator=_gen(7)) * 1e-3; r[0] = 300.0; rows.append(r)   # subnormal-scale blocks
    r = torch.zeros(k); r[0::16] = 0.17578125; r[1::16] = 0.03662109375; rows.append(r)  # R4 tie vector
    r = torch.arange(k, dtype=torch.float32) - k / 2; rows.append(r)
    # bf16 subnormals (|x| < 2^-126) next to a few small normals that keep the INT8 row scale's
    # reciprocal finite: sums of subnormals survive into the codes (no flush-to-zero anywhere)
    r = torch.randn(k, generator=_gen(8)) * 3e-39; r[0::128] = 4e-37; rows.append(r)
    r = torch.rand(k, generator=_gen(9)) * 1.1e-38; r[5] = -1e-36; rows.append(r)
    # INT8 exact ties: row max 127 -> x * 127/amax = x; k + 0.5 values must round half to even
    r = torch.tensor([127.0, 2.5, 3.5, 0.5, 1.5, -4.5, 126.5, -0.5, -1.5, 5.5, -126.5, 0.0, 64.5, -63.5, 7.5, 8.5])
    rows.append(r.repeat(k // 16))
    return torch.stack(rows).to(torch.bfloat16)


def bits(t: torch.Tensor):
    """bf16 tensor -> numpy uint16 bit patterns (for the oracle)."""
    return t.contiguous().view(torch.int16).cpu().numpy().view("uint16")


def linear_weight_device(n: int, k: int, seed: int, device):
    """Device-side variant of linear_weight (same distribution; different stream of
    random numbers) for the large bench models, where CPU generation is too slow."""
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    w = (torch.randn(n, k, generator=g, device=device) / math.sqrt(k)).to(torch.bfloat16)
    b = 0.02 * torch.randn(n, generator=g, device=device)
    return w, b


def dit_activation_device(m: int, k: int, seed: int, device, outlier_frac: float = 0.005,
                          tail_frac: float = 0.01) -> torch.Tensor:
    """Device-side variant of dit_activation (same recipe, different random stream) for the large
    bench inputs (the C2 sweep's 64K x 1920 rows), where CPU generation is slow."""
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    x = torch.randn(m, k, generator=g, device=device)
    x *= torch.exp(0.5 * torch.randn(m, 1, generator=g, device=device))
    n_out = max(1, int(round(outlier_frac * k)))
    ch = torch.randperm(k, generator=g, device=device)[:n_out]
    x[:, ch] *= 10 + 40 * torch.rand(n_out, generator=g, device=device)
    if tail_frac > 0:
        mask = torch.rand(m, k, generator=g, device=device) < tail_frac
        z = torch.randn(m, k, generator=g, device=device)
        chi = sum(torch.randn(m, k, generator=g, device=device) ** 2 for _ in range(4))
        x = torch.where(mask, z / torch.sqrt(chi / 4), x)
    return x.to(torch.bfloat16)


def trajectory_basis(m: int, h: int, seed: int, device=None):
    """Two bf16-valued basis tensors A, B [m, h] for the synthetic PF-ODE-like
    block-0 input X_t = cos(theta_t) A + sin(theta_t) B (a smooth, locally
    linear trajectory), with per-token magnitudes and a few outlier channels."""
    if device is None or str(device) == "cpu":
        a = dit_activation(m, h, seed, tail_frac=0.0).float()
        b = dit_activation(m, h, seed + 1, tail_frac=0.0).float()
        return a, b
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    out = []
    for _ in range(2):
        x = torch.randn(m, h, generator=g, device=device)
        x *= torch.exp(0.5 * torch.randn(m, 1, generator=g, device=device))
        ch = torch.randperm(h, generator=g, device=device)[: max(1, h // 200)]
        x[:, ch] *= 10 + 40 * torch.rand(ch.numel(), generator=g, device=device)
        out.append(x)
    return out[0], out[1]


def trajectory_input(A: torch.Tensor, B: torch.Tensor, t: int, T: int, kappa: float = 0.05) -> torch.Tensor:
    """X_t = cos(theta_t) A + sin(theta_t) B with theta_t = kappa * t / T (bf16)."""
    th = kappa * t / T
    return (math.cos(th) * A + math.sin(th) * B).to(torch.bfloat16)
