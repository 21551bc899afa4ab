"""Scalar decision logic of DMPQ and TDC, written out from the paper.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Pure Python, fp64 scalars.

- Eq. 3: Gamma_{t-1} = ||Y_{t-1} - X_{t-1}||_1 / ||X_{t-1}||_1
- Eq. 6: tau_Gamma = (tau_rel - beta) / alpha
- Eq. 7: INT8 if Gamma_{t-1} > tau_Gamma else NVFP4
- P:241 (PDR): after a Skip, Gamma_{t-1} is missing -> all layers INT8
- Eq. 9: E = 1 - CosSim(Delta_{t-1}, Delta_{t-2})
- Eq. 10: E_acc <- E_tp after Compute, E_acc + E_tp + rho after Skip
- Eq. 11: Skip iff E_acc <= tau and t - t_p <= N_max
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

FMT_INT8 = 0
FMT_NVFP4 = 1
FMT_BF16 = 2

COMPUTE = 0
SKIP = 1


def derive_tau_gamma(alpha: float, beta: float, tau_rel: float, eps_slope: float = 1e-8) -> float:
    """Eq. 6. A slope alpha <= eps_slope has no usable inversion; the
    threshold is then -inf, which routes every Gamma >= 0 to INT8."""
    if alpha <= eps_slope:
        return -math.inf
    return (tau_rel - beta) / alpha


def gamma_from_stats(st, metric: str = "l1") -> float | None:
    """Eq. 3 from the block statistics (sum|d|, sum|x|, sum d^2, sum x^2, ...).
    Returns None when the reference norm is zero (Eq. 3 undefined)."""
    if metric == "l1":
        num, den = st[0], st[1]
        if den == 0.0:
            return None
        return num / den
    num, den = st[2], st[3]
    if den == 0.0:
        return None
    return math.sqrt(num) / math.sqrt(den)


def route_block(gamma: float | None, tau_gamma, t: int, prev_skipped: bool):
    """Eq. 7 for every linear layer j of one block, plus the two fallbacks:
    t = 0 has no Gamma_{t-1} and a block computed right after a Skip has
    none either -> INT8. An undefined Gamma (zero-norm input) -> INT8.
    Equality Gamma == tau routes NVFP4 (Eq. 7's "<=")."""
    out = []
    for tau in tau_gamma:
        if t == 0 or prev_skipped or gamma is None or gamma > tau:
            out.append(FMT_INT8)
        else:
            out.append(FMT_NVFP4)
    return out


def purify_route(base, ratio: float | None, prev_skipped: bool, tau_outlier: float = 25.0):
    """Purified Cache Refresh, per layer: an outlier ratio strictly
    above tau_outlier routes the layer to full precision (BF16); otherwise the first
    compute after a Skip routes INT8; otherwise the DMPQ decision stands.
    Precedence outlier > post-skip > base."""
    if ratio is not None and ratio > tau_outlier:
        return FMT_BF16
    if prev_skipped:
        return FMT_INT8
    return base


def cosine_error_from_stats(dot: float, n_new: float, n_prev: float) -> float:
    """Eq. 9 with D = 1 - CosSim. Zero-norm delta -> +inf (maximal
    error, forces Compute)."""
    if n_new == 0.0 or n_prev == 0.0:
        return math.inf
    return 1.0 - dot / math.sqrt(n_new * n_prev)


def rel_l2_error_from_stats(dot: float, n_new: float, n_prev: float) -> float:
    """Eq. 9 with D = relative-L2 distance ("other metrics such as relative-L2 distance";
    reading R19): ||Delta_t - Delta_prev||_2 / ||Delta_prev||_2, with ||a - b||^2 expanded as
    ||a||^2 - 2 a.b + ||b||^2 (the three sums the refresh produces). A zero reference norm is
    maximal error (+inf), as for the cosine."""
    if n_prev == 0.0:
        return math.inf
    return math.sqrt(max(n_new - 2.0 * dot + n_prev, 0.0)) / math.sqrt(n_prev)


def prediction_error_from_stats(st, metric: str = "cos") -> float:
    """E_{t_p} of Eq. 9 from a block's statistics (dot, ||Delta_t||^2, ||Delta_prev||^2 at [4:7])."""
    if metric == "rel_l2":
        return rel_l2_error_from_stats(st[4], st[5], st[6])
    return cosine_error_from_stats(st[4], st[5], st[6])


@dataclass
class TdcConfig:
    """rho = 0.001, N_max = 2, tau = 0.003; D of Eq. 9: "cos" (default) or "rel_l2"."""
    rho: float = 0.001
    tau: float = 0.003
    n_max: int = 2
    metric: str = "cos"


@dataclass
class TdcState:
    t_p: int = -1            # last fully-computed timestep
    e_tp: float = math.inf   # E_{t_p}: prediction error measured at t_p
    e_acc: float = math.inf  # E_acc
    last: int | None = None  # S_{t-1}
    n_computed: int = 0      # computed deltas so far (warm-up needs two)
    history: list = field(default_factory=list)


def tdc_decide(st: TdcState, cfg: TdcConfig, t: int) -> int:
    """Eq. 11. Warm-up: the first two computes are forced (two deltas are
    needed by Eq. 9)."""
    if st.n_computed < 2:
        return COMPUTE
    if st.e_acc <= cfg.tau and (t - st.t_p) <= cfg.n_max:
        return SKIP
    return COMPUTE


def tdc_update(st: TdcState, cfg: TdcConfig, t: int, decision: int, e_new: float | None = None) -> None:
    """Eq. 10, applied at the end of step t.

    After a Compute, ``e_new`` is E_{t_p} = D(Delta_t, Delta_{previous compute})
    (+inf when there is no previous delta). After a Skip, E_acc grows by
    E_{t_p} + rho, evaluated left to right in fp64."""
    if decision == COMPUTE:
        st.e_tp = math.inf if (e_new is None or st.n_computed == 0) else e_new
        st.e_acc = st.e_tp
        st.t_p = t
        st.n_computed += 1
    else:
        st.e_acc = (st.e_acc + st.e_tp) + cfg.rho
    st.last = decision
    st.history.append(decision)
