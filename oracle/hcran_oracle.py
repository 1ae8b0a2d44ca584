"""CPU ORACLE (test infrastructure only) -- numpy float64 restatement of the
reference's batched-instance hot path: Dinkelbach -> SCALE rounds -> power
sweeps (budget bisection + projected subgradient duals) -> repair/selection.

    *** Not part of the product. ***  Only tests/, __graft_entry__.smoke() and
    bench.py's cpu_baseline / --impl reference legs may import this module, and
    only as the checker or as the timed CPU baseline.  The product path
    (paper_1803_07772_b200) never calls it and fails loudly without its CUDA
    extension.

Parity pinning: this restatement is checked against golden fixtures produced
by running the unmodified reference (/root/reference/pkg/src/hcran_noma) in
the build container (tests/golden/make_golden.py, tests/test_oracle_golden.py):
EE and total power within 1e-4 relative and identical rho/a outside the
reference's own near-tie set.

Every function cites the reference lines it restates.  The numeric forms that
decide floor-scale outcomes are kept: cross interference as
`full - own` (model.py:268-274), psi_cross as `sum(g*u_tot) - sum(g*u)`
(scale.py:756-759), the per-RRH budget multiplier by exact bisection with the
reference's bracket (scale.py:444-475).  Decode-order sums use prefix/suffix
scans over a per-(m, n) rank (O(MKN) instead of the reference's O(MK^2N)
boolean einsum), which only reorders float additions.

Scope: exclusive seatings (one head per user, <= l_max users per (m, n)).  The
non-exclusive "products-active" multiplier families (scale.py:761-775,
835-840, 861-895) are out of scope for this round; `ProductsActive` is raised
when a seating would need them (never at any BASELINE configuration: the
multistart that opens every cell only runs when M*K*N <= 16).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

LN2 = math.log(2.0)
Z_FLOOR = 1e-300


class ProductsActive(NotImplementedError):
    """The seating is not exclusive: theta/theta' families would be live."""


class Infeasible(RuntimeError):
    """First inner solve infeasible (dinkelbach.py:81-86)."""


# ---------------------------------------------------------------------------
# problem data
# ---------------------------------------------------------------------------

@dataclass
class Prob:
    gamma: np.ndarray       # (M, K, N)
    sigma: np.ndarray       # (M, K, N)
    p_max: np.ndarray       # (M,)
    p_mask: np.ndarray      # (M, K, N)
    eta: np.ndarray         # (M,)
    w: np.ndarray           # (M, K)
    elastic: np.ndarray     # (K,) bool
    min_rates: np.ndarray   # (K,)
    static_power: float
    l_max: int
    tol: object             # Tolerances-like (xi, varpi1_rel, ..., box_rel_tol)
    rho1: float
    rho2: float
    order: np.ndarray = field(init=False)   # (M, K, N) users strong -> weak
    rank: np.ndarray = field(init=False)    # (M, K, N) decode rank of each user

    def __post_init__(self):
        self.order, self.rank = decode_order(self.gamma)

    @property
    def shape(self):
        return self.gamma.shape

    @property
    def max_mask(self) -> float:
        return float(self.p_mask.max())

    @property
    def streaming(self) -> list[int]:
        return [int(k) for k in np.nonzero(~self.elastic)[0]]

    @classmethod
    def from_config(cls, cfg, ch) -> "Prob":
        """Any reference-compatible (cfg, ch) pair (model.py:83-201)."""
        return cls(gamma=np.asarray(ch.gamma, float), sigma=np.asarray(ch.sigma, float),
                   p_max=np.asarray(cfg.p_max, float), p_mask=np.asarray(cfg.p_mask, float),
                   eta=np.asarray(cfg.eta, float), w=np.asarray(cfg.weights, float),
                   elastic=np.asarray(cfg.elastic_mask(), bool),
                   min_rates=np.asarray(cfg.min_rates(), float),
                   static_power=float(cfg.static_power()), l_max=int(cfg.l_max),
                   tol=cfg.tolerances, rho1=float(cfg.rho1), rho2=float(cfg.rho2))


def decode_order(gamma: np.ndarray):
    """SIC decode order per (m, n): user i is stronger than k iff
    gamma_i > gamma_k, ties toward the lower index (model.py:235-244)."""
    order = np.argsort(-gamma, axis=1, kind="stable")
    rank = np.empty_like(order)
    np.put_along_axis(rank, order, np.arange(gamma.shape[1])[None, :, None], axis=1)
    return order, rank


def _exclusive_prefix(x_sorted: np.ndarray) -> np.ndarray:
    c = np.cumsum(x_sorted, axis=1)
    out = np.zeros_like(c)
    out[:, 1:] = c[:, :-1]
    return out


def stronger_sum(P: Prob, x: np.ndarray) -> np.ndarray:
    """sum over users stronger than k on (m, n) of x[m, ., n]."""
    xs = np.take_along_axis(x, P.order, axis=1)
    return np.take_along_axis(_exclusive_prefix(xs), P.rank, axis=1)


def weaker_sum(P: Prob, x: np.ndarray) -> np.ndarray:
    """sum over users weaker than k on (m, n) of x[m, ., n]."""
    xs = np.take_along_axis(x, P.order, axis=1)[:, ::-1, :]
    return np.take_along_axis(_exclusive_prefix(xs)[:, ::-1, :], P.rank, axis=1)


# ---------------------------------------------------------------------------
# rates (model.py:268-341)
# ---------------------------------------------------------------------------

def cross_of(P: Prob, p: np.ndarray) -> np.ndarray:
    """Other-RRH power received at user k through RRH m's channel index:
    full - own (model.py:268-274)."""
    totals = p.sum(axis=1)
    full = np.einsum("jn,jkn->kn", totals, P.gamma)
    return full[None, :, :] - totals[:, None, :] * P.gamma


def noise_floor(P: Prob, p: np.ndarray, cross: np.ndarray | None = None) -> np.ndarray:
    if cross is None:
        cross = cross_of(P, p)
    return P.sigma + P.gamma * stronger_sum(P, p) + cross


def sinr(P: Prob, p: np.ndarray) -> np.ndarray:
    return p * P.gamma / noise_floor(P, p)          # model.py:287-290


def user_rates(P: Prob, p: np.ndarray) -> np.ndarray:
    """(K,) weighted rate per user (model.py:320-323)."""
    return np.einsum("mk,mkn->k", P.w, np.log2(1.0 + sinr(P, p)))


def elastic_power(P: Prob, p: np.ndarray) -> float:
    """Static floor + eta-weighted elastic transmit power (model.py:332-335)."""
    return P.static_power + float(np.dot(P.eta, p[:, P.elastic, :].sum(axis=(1, 2))))


def report(P: Prob, p: np.ndarray) -> tuple[float, float, float]:
    """(sum_rate, total_power, ee) -- model.py:326-341."""
    r = float(user_rates(P, p)[P.elastic].sum())
    pw = elastic_power(P, p)
    return r, pw, r / pw


def true_objective(P: Prob, p: np.ndarray, e: float) -> float:
    """scale.py:908-911."""
    rates = np.log2(1.0 + sinr(P, p))
    r = float(np.sum(rates[:, P.elastic, :] * P.w[:, P.elastic, None]))
    return r - e * elastic_power(P, p)


# ---------------------------------------------------------------------------
# SCALE bound (scale.py:68-115)
# ---------------------------------------------------------------------------

def bound_coeffs(P: Prob, p: np.ndarray):
    """alpha = z/(1+z), beta = log2(1+z) - alpha log2 z at the SINR of p;
    z <= 0 takes (1, 0) (scale.py:88-96)."""
    z = sinr(P, p)
    ok = z > 0
    zz = np.where(ok, z, 1.0)
    a = zz / (1.0 + zz)
    b = np.log2(1.0 + zz) - a * np.log2(zz)
    return np.where(ok, a, 1.0), np.where(ok, b, 0.0)


def surrogate_rates(P: Prob, p: np.ndarray, alpha, beta) -> np.ndarray:
    """beta + alpha log2 z, zero (instead of -inf) where z <= 0
    (scale.py:109-115 with the finite mask of scale.py:904)."""
    z = sinr(P, p)
    with np.errstate(divide="ignore"):
        lz = np.log2(np.maximum(z, Z_FLOOR))
    return np.where(z > 0, beta + alpha * lz, 0.0)


# ---------------------------------------------------------------------------
# per-(instance, e) solve context (scale.py:651-711)
# ---------------------------------------------------------------------------

class Ctx:
    GAINS = (0.6, 0.8, 0.6, 0.6, 0.6)   # scale.py:495 (budget, rate, pair, tuple, sic)
    RATE_SCALE = 10.0                    # scale.py:689

    def __init__(self, P: Prob, e: float, sic: str = "dense"):
        """sic="dense": the reference's SIC family over every oriented pair.
        sic="seated": the device's default model, multipliers only on pairs
        whose members are both seated (the family is re-created per seating);
        `floor_tie` records a seat whose numerator vanishes exactly while its
        denominator is not positive -- the reference then decides the seat from
        the floor-level multipliers of unseated pairs."""
        self.P, self.e = P, float(e)
        self.sic = sic
        self.floor_tie = False
        M, K, N = P.shape
        self.p_floor = 1e-30 * P.max_mask
        iu, ju = np.triu_indices(K, 1)
        ri = P.rank[:, iu, :]                      # (M, Q, N)
        rj = P.rank[:, ju, :]
        a = np.broadcast_to(iu[None, :, None], ri.shape)
        b = np.broadcast_to(ju[None, :, None], rj.shape)
        self.s_idx = np.where(ri < rj, a, b)       # strong member  (model.py:247-265)
        self.w_idx = np.where(ri < rj, b, a)       # weak member
        self.n_pairs = iu.size
        take = lambda arr, idx: np.take_along_axis(arr, idx, axis=1)
        self.take = take
        self.g_s, self.g_w = take(P.gamma, self.s_idx), take(P.gamma, self.w_idx)
        self.s_s, self.s_w = take(P.sigma, self.s_idx), take(P.sigma, self.w_idx)
        cm = cross_of(P, P.p_mask)
        self.sic_scale = (self.g_w * self.s_s + self.g_s * self.s_w
                          + self.g_w * take(cm, self.s_idx) + self.g_s * take(cm, self.w_idx)
                          + 1e-300)
        self.mask_s, self.mask_w = take(P.p_mask, self.s_idx), take(P.p_mask, self.w_idx)
        p_ref = 0.5 * float(P.p_max.mean()) / (K * N)
        self.den_scale = max(self.e * float(P.eta.max()), 1.0 / (LN2 * p_ref))
        g_rate, g_sic = self.GAINS[1], self.GAINS[4]
        cap = P.tol.dual_cap
        self.zeta_step = g_rate / self.RATE_SCALE
        self.zeta_cap = cap
        self.sic_step = g_sic * self.den_scale / (
            p_ref * self.sic_scale ** 2 * self.mask_s * self.mask_w + 1e-300)
        self.sic_cap = cap * self.den_scale / p_ref

    # pair scatter helpers ---------------------------------------------------
    def scatter(self, idx: np.ndarray, vals: np.ndarray) -> np.ndarray:
        out = np.zeros(self.P.shape)
        M, Q, N = idx.shape
        mm = np.broadcast_to(np.arange(M)[:, None, None], idx.shape)
        nn = np.broadcast_to(np.arange(N)[None, None, :], idx.shape)
        np.add.at(out, (mm, idx, nn), vals)
        return out

    def linearize(self, p_lin: np.ndarray) -> dict:
        """Tangent constants of the subtracted SIC product at the round's
        point (scale.py:726-735)."""
        c_lin = cross_of(self.P, p_lin)
        gconst = self.g_s * self.take(p_lin, self.s_idx) * self.take(p_lin, self.w_idx)
        return {"p_lin": p_lin, "log_p_lin": np.log(np.maximum(p_lin, Z_FLOOR)),
                "gconst": gconst, "g_val": gconst * self.take(c_lin, self.w_idx)}

    def analyze(self, p, zeta, zt, alpha, beta, lin):
        """One Jacobi snapshot: numerators, denominators (budget multiplier
        excluded) and the rate / SIC residuals (scale.py:738-858)."""
        P, e = self.P, self.e
        cross = cross_of(P, p)
        floor = P.sigma + P.gamma * stronger_sum(P, p) + cross
        inv_floor = 1.0 / floor
        z = p * P.gamma * inv_floor
        r_hat = beta + alpha * np.log2(np.maximum(z, Z_FLOOR))
        zeta_of = np.where(P.elastic, 1.0, zeta)
        c_rate = (P.w * zeta_of[None, :])[:, :, None] * alpha
        t_same = c_rate * P.gamma * inv_floor / LN2
        psi_same = weaker_sum(P, t_same)
        u = c_rate * inv_floor / LN2
        u_tot = u.sum(axis=0)
        psi_cross = (np.einsum("mln,ln->mn", P.gamma, u_tot)
                     - np.einsum("mln,mln->mn", P.gamma, u))[:, None, :]

        num_sic = 0.0
        den_sic = 0.0
        p_s, p_w = self.take(p, self.s_idx), self.take(p, self.w_idx)
        bracket = self.g_w * self.s_s - self.g_s * self.s_w + self.g_w * self.take(cross, self.s_idx)
        if zt.any():
            den_sic = self.scatter(self.s_idx, zt * p_w * bracket) + \
                self.scatter(self.w_idx, zt * p_s * bracket)
            d_agg = self.scatter(self.s_idx, zt * p_s * p_w * self.g_w)
            d_tot = d_agg.sum(axis=0)
            den_sic = den_sic + (np.einsum("an,man->mn", d_tot, P.gamma)
                                 - np.einsum("man,man->mn", d_agg, P.gamma))[:, None, :]
            own = zt * lin["g_val"]
            num_sic = self.scatter(self.s_idx, own) + self.scatter(self.w_idx, own)
            a_agg = self.scatter(self.w_idx, zt * lin["gconst"])
            a_tot = a_agg.sum(axis=0)
            b_term = (np.einsum("bn,mbn->mn", a_tot, P.gamma)
                      - np.einsum("mbn,mbn->mn", a_agg, P.gamma))[:, None, :]
            num_sic = num_sic + lin["p_lin"] * b_term
        dlog = np.log(np.maximum(p, Z_FLOOR)) - lin["log_p_lin"]
        f_term = (lin["p_lin"] * dlog).sum(axis=1)
        h_full = np.einsum("jn,jbn->bn", f_term, P.gamma)
        h_cross = h_full[None, :, :] - f_term[:, None, :] * P.gamma
        g_lin = (lin["g_val"] * (1.0 + self.take(dlog, self.s_idx) + self.take(dlog, self.w_idx))
                 + lin["gconst"] * self.take(h_cross, self.w_idx))
        sic_slack = p_s * p_w * bracket - g_lin

        num = c_rate / LN2 + num_sic
        den = ((e * P.eta)[:, None, None] * P.elastic[None, :, None]
               + psi_same + psi_cross + den_sic)
        r_user = np.einsum("mk,mkn->k", P.w, r_hat)
        rate_slack = np.clip(np.where(P.elastic, 0.0, P.min_rates - r_user),
                             -2.0 * self.RATE_SCALE, 2.0 * self.RATE_SCALE)
        return num, den, rate_slack, sic_slack

    def surrogate(self, p, alpha, beta) -> float:
        """scale.py:902-906."""
        P = self.P
        r = surrogate_rates(P, p, alpha, beta)
        return float(np.sum(r[:, P.elastic, :] * P.w[:, P.elastic, None])) - \
            self.e * elastic_power(P, p)

    def streaming_stuck(self, zeta, p, alpha, beta) -> bool:
        """scale.py:913-924."""
        P = self.P
        if not P.streaming:
            return False
        r_user = np.einsum("mk,mkn->k", P.w, surrogate_rates(P, p, alpha, beta))
        at_cap = zeta >= self.zeta_cap * (1 - 1e-9)
        return bool(np.any(at_cap & (r_user < P.min_rates - P.tol.c13_rate_tol)))


def clamp_update(num, den, mask, floor):
    """num/den clamped to [0, mask]; mask when den <= 0, 0 when num <= 0,
    then lifted to the log-domain floor (scale.py:433-441)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        raw = np.where(den > 0, num / np.where(den > 0, den, 1.0), mask)
    raw = np.where(num <= 0, 0.0, raw)
    return np.maximum(np.clip(raw, 0.0, mask), floor)


def budget_multiplier(num, den, mask, budget, warm=None, iters: int = 42):
    """Smallest xi >= 0 per RRH with sum clip(num/(den+xi), 0, mask) <= budget:
    0 when slack; else bracket from max(4 warm, 1e-6) growing x8 (<= 80 times)
    and 42 bisection halvings, returning the feasible end (scale.py:444-475)."""

    def load(xi):
        d = den + xi[:, None, None]
        with np.errstate(divide="ignore", invalid="ignore"):
            q = np.where(d > 0, num / np.where(d > 0, d, 1.0), mask)
        q = np.where(num <= 0, 0.0, np.clip(q, 0.0, mask))
        return q.sum(axis=(1, 2))

    M = den.shape[0]
    lo = np.zeros(M)
    tight = load(lo) > budget
    if not tight.any():
        return lo
    hi = np.ones(M) if warm is None else np.maximum(4.0 * warm, 1e-6)
    for _ in range(80):
        over = load(hi) > budget
        if not over.any():
            break
        hi[over] *= 8.0
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        over = load(mid) > budget
        lo = np.where(over, mid, lo)
        hi = np.where(over, hi, mid)
    return np.where(tight, hi, 0.0)


# ---------------------------------------------------------------------------
# starting seatings (scale.py:1017-1071)
# ---------------------------------------------------------------------------

def service_scores(P: Prob) -> np.ndarray:
    """(M, K) mean full-load rate per head (scale.py:1017-1026)."""
    load = (P.p_max / P.shape[2])[:, None, None] * P.gamma
    cross = load.sum(axis=0)[None] - load
    return np.log2(1.0 + P.p_mask * P.gamma / (P.sigma + cross)).mean(axis=2)


def greedy_start(P: Prob) -> np.ndarray:
    """Best-score head per user; streaming users get their best subcarrier;
    elastic users fill the remaining <= l_max seats per (m, n) by gain;
    budget-scaled mask powers on seats, floor elsewhere (scale.py:1029-1060)."""
    M, K, N = P.shape
    floor = 1e-30 * P.max_mask
    head = np.argmax(service_scores(P), axis=0)
    seat = np.zeros((M, K, N), bool)
    for k in P.streaming:
        m = int(head[k])
        seat[m, k, int(np.argmax(P.gamma[m, k, :]))] = True
    for m in range(M):
        mine = np.nonzero((head == m) & P.elastic)[0]
        if mine.size == 0:
            continue
        by_gain = np.argsort(P.gamma[m, mine, :], axis=0)[::-1]
        for n in range(N):
            free = P.l_max - int(seat[m, :, n].sum())
            if free > 0:
                seat[m, mine[by_gain[:free, n]], n] = True
    p = np.where(seat, P.p_mask, floor)
    s = np.minimum(1.0, P.p_max / np.maximum(p.sum(axis=(1, 2)), 1e-300))
    return np.maximum(p * s[:, None, None], floor)


def seating_exclusive(seat: np.ndarray, l_max: int) -> bool:
    """scale.py:1007-1014."""
    if np.any(seat.any(axis=2).sum(axis=0) > 1):
        return False
    return bool(np.all(seat.sum(axis=1) <= l_max))


# ---------------------------------------------------------------------------
# SCA rounds over one seating (scale.py:553-615)
# ---------------------------------------------------------------------------

@dataclass
class InnerStats:
    rounds: int = 0
    total_sweeps: int = 0
    round_objectives: list = field(default_factory=list)
    status: str = "ok"
    infeasible_reason: str | None = None
    true_objective: float = float("nan")
    floor_tie: bool = False


def sca_rounds(ctx: Ctx, p0: np.ndarray, stats: InnerStats):
    P = ctx.P
    tol = P.tol
    seat = p0 > ctx.p_floor
    if not seating_exclusive(seat, P.l_max):
        raise ProductsActive("non-exclusive seating")
    pair_mask = None
    if ctx.sic == "seated":
        pair_mask = ctx.take(seat, ctx.s_idx) & ctx.take(seat, ctx.w_idx)
    mask_eff = np.where(seat, P.p_mask, ctx.p_floor)
    zeta = np.where(P.elastic, 0.0, 1.0)
    zt = np.zeros_like(ctx.g_s)
    p = p0
    xi = np.zeros(P.shape[0])
    eps1 = tol.varpi1_rel * P.p_max
    eps2 = tol.varpi2_rel * P.p_max
    objs = []
    for s in range(tol.s_max):
        alpha, beta = bound_coeffs(P, p)
        lin = ctx.linearize(p)
        p_round = p
        for v in range(1, tol.v_max + 1):
            num, den, rate_slack, sic_slack = ctx.analyze(p, zeta, zt, alpha, beta, lin)
            if pair_mask is not None and np.any(seat & (num == 0.0) & ~(den > 0.0)):
                ctx.floor_tie = True
            xi = budget_multiplier(num, den, mask_eff, P.p_max, xi)
            p_next = clamp_update(num, den + xi[:, None, None], mask_eff, ctx.p_floor)
            damp = 1.0 / math.sqrt(max(v, 1))
            zeta = np.clip(zeta + damp * ctx.zeta_step * rate_slack, 0.0, ctx.zeta_cap)
            zt = np.clip(zt + damp * ctx.sic_step * sic_slack, 0.0, ctx.sic_cap)
            if pair_mask is not None:
                zt = np.where(pair_mask, zt, 0.0)
            delta = np.abs(p_next - p).max(axis=(1, 2))
            p = p_next
            stats.total_sweeps += 1
            if v >= 8 and np.all(delta < eps1):
                break
        rejected = ctx.surrogate(p, alpha, beta) < ctx.surrogate(p_round, alpha, beta)
        if rejected:
            p = p_round
        objs.append(ctx.surrogate(p, alpha, beta))
        if rejected:
            break
        if ctx.streaming_stuck(zeta, p, alpha, beta):
            stats.infeasible_reason = "rate multiplier at cap with unmet demand"
            break
        if s > 0 and np.all(np.abs(p - p_round).max(axis=(1, 2)) < eps2):
            break
    return p, objs


# ---------------------------------------------------------------------------
# repair (scale.py:927-1004, 1086-1203)
# ---------------------------------------------------------------------------

def sic_cleanup(ctx: Ctx, q: np.ndarray) -> np.ndarray:
    """Zero one member of every powered pair whose cancellation margin is
    positive (the weak one unless only the strong one is elastic); repeat
    while removals change the cross terms (scale.py:974-1004)."""
    P = ctx.P
    gone = np.zeros(q.shape, bool)
    if not ctx.n_pairs:
        return gone
    drop = np.where(~P.elastic[ctx.w_idx] & P.elastic[ctx.s_idx], ctx.s_idx, ctx.w_idx)
    M, Q, N = drop.shape
    for _ in range(P.shape[1] + 1):
        cross = cross_of(P, q)
        omega = (ctx.g_w * ctx.s_s - ctx.g_s * ctx.s_w
                 + ctx.g_w * ctx.take(cross, ctx.s_idx) - ctx.g_s * ctx.take(cross, ctx.w_idx))
        bad = ((ctx.take(q, ctx.s_idx) > 0) & (ctx.take(q, ctx.w_idx) > 0)
               & (omega > 0.5 * P.tol.c14_rel_tol * ctx.sic_scale))
        if not bad.any():
            return gone
        mi, qi, ni = np.nonzero(bad)
        ki = drop[mi, qi, ni]
        q[mi, ki, ni] = 0.0
        gone[mi, ki, ni] = True
    return gone


def trim_streaming(P: Prob, q: np.ndarray, margin: float = 0.05, passes: int = 2) -> None:
    """Scale each streaming user down (30-step bisection on a common factor)
    until its rate sits just above min_rate + margin (scale.py:1086-1114)."""
    for _ in range(passes):
        touched = False
        for k in P.streaming:
            base = q[:, k, :].copy()
            if base.max() <= 0:
                continue
            target = P.min_rates[k] + margin
            if float(user_rates(P, q)[k]) <= target:
                continue
            lo, hi = 0.0, 1.0
            for _ in range(30):
                mid = 0.5 * (lo + hi)
                q[:, k, :] = mid * base
                if user_rates(P, q)[k] >= target:
                    hi = mid
                else:
                    lo = mid
            q[:, k, :] = hi * base
            touched = True
        if not touched:
            break


def boost_streaming(P: Prob, q: np.ndarray, banned: np.ndarray):
    """Water-fill deficient streaming users on their serving head, strongest
    subcarriers first (evicting the weakest elastic occupant of a full
    subcarrier, shrinking the head's elastic powers by 0.85 when the budget is
    exhausted); move a user wholesale to its next-best untried head when its
    head yields crumbs (scale.py:1117-1203).  Returns (q, ok)."""
    streaming = P.streaming
    if not streaming:
        return q, True
    M, K, N = P.shape
    tol = P.tol.c13_rate_tol
    scores = service_scores(P)
    tried = {k: set() for k in streaming}

    def fill(k: int, m: int) -> bool:
        progressed = False
        for n in np.argsort(P.gamma[m, k, :])[::-1]:
            if banned[m, k, n]:
                continue
            occ = np.nonzero(q[m, :, n] > 0)[0]
            if q[m, k, n] <= 0 and len(occ) >= P.l_max:
                movable = [u for u in occ if P.elastic[u]]
                if not movable:
                    continue
                out = min(movable, key=lambda u: q[m, u, n])
                q[m, out, n] = 0.0
            room = P.p_max[m] - q[m].sum()
            if room <= 1e-15 * P.p_max[m]:
                shrink = P.elastic & (np.arange(K) != k)
                q[m, shrink, :] *= 0.85
                room = P.p_max[m] - q[m].sum()
            add = min(P.p_mask[m, k, n] - q[m, k, n], room)
            if add <= 1e-12 * P.p_mask[m, k, n]:
                continue
            q[m, k, n] += add
            progressed = True
            if float(user_rates(P, q)[k]) >= P.min_rates[k] - tol * 0.5:
                break
        return progressed

    for _ in range(4 * len(streaming) + 4):
        rates = user_rates(P, q)
        deficit = np.where(P.elastic, 0.0, P.min_rates - rates)
        needy = [k for k in streaming if deficit[k] > tol * 0.5]
        if not needy:
            return q, True
        progress = False
        for k in sorted(needy, key=lambda k: -deficit[k]):
            r0 = float(user_rates(P, q)[k])
            tot = q.sum(axis=2)
            m = int(np.argmax(tot[:, k])) if tot[:, k].max() > 0 else int(np.argmax(scores[:, k]))
            tried[k].add(m)
            fill(k, m)
            r1 = float(user_rates(P, q)[k])
            if r1 >= P.min_rates[k] - tol * 0.5 or r1 > r0 + 0.05:
                progress = True
                continue
            alts = [mm for mm in np.argsort(scores[:, k])[::-1] if mm not in tried[k]]
            if alts:
                q[:, k, :] = 0.0
                tried[k].add(int(alts[0]))
                fill(k, int(alts[0]))
                r2 = float(user_rates(P, q)[k])
                if r2 >= P.min_rates[k] - tol * 0.5 or r2 > r0 + 0.05:
                    progress = True
        if not progress:
            return q, False
    rates = user_rates(P, q)
    return q, bool(np.all(rates[streaming] >= P.min_rates[streaming] - tol))


def repair(ctx: Ctx, p: np.ndarray):
    """Threshold, one head per user, top-l_max per (m, n), SIC cleanup, budget
    rescale, SIC cleanup, then streaming trim/boost rounds (scale.py:927-972)."""
    P = ctx.P
    M, K, N = P.shape
    q = p.copy()
    q[q <= 1e-6 * P.max_mask] = 0.0
    if M > 1:
        head = np.argmax(q.sum(axis=2), axis=0)
        keep = np.zeros(q.shape, bool)
        keep[head, np.arange(K), :] = True
        q[~keep] = 0.0
    if K > P.l_max:
        by_power = np.argsort(q, axis=1)[:, ::-1, :]
        ranked = np.take_along_axis(q, by_power, axis=1)
        np.put_along_axis(q, by_power,
                          np.where(np.arange(K)[None, :, None] < P.l_max, ranked, 0.0), axis=1)
    sic_cleanup(ctx, q)
    s = np.minimum(1.0, P.p_max / np.maximum(q.sum(axis=(1, 2)), 1e-300))
    q *= s[:, None, None]
    sic_cleanup(ctx, q)
    ok = True
    if P.streaming:
        banned = np.zeros(q.shape, bool)
        for _ in range(4):
            trim_streaming(P, q)
            q, ok = boost_streaming(P, q, banned)
            gone = sic_cleanup(ctx, q)
            banned |= gone
            if ok and not gone.any():
                break
        trim_streaming(P, q)
        rates = user_rates(P, q)
        st = P.streaming
        ok = bool(np.all(rates[st] >= P.min_rates[st] - P.tol.c13_rate_tol))
    return q, ok


# ---------------------------------------------------------------------------
# feasibility and indicators (model.py:404-521)
# ---------------------------------------------------------------------------

def feasible(P: Prob, p: np.ndarray) -> bool:
    """C4 box, C10 one head per user, C11 <= l_max per (m, n), C12 budgets,
    C13 streaming rates, C14 cancellation order on powered pairs."""
    tol = P.tol
    M, K, N = P.shape
    if np.any(p - P.p_mask * (1 + tol.box_rel_tol) > 0) or np.any(p < 0):
        return False
    if M > 1:
        peak = p.max(axis=2)                       # (M, K): largest power per head
        top2 = np.sort(peak, axis=0)[-2:, :]
        if np.any(top2[0] * top2[1] > P.rho1):
            return False
    ell = P.l_max + 1
    if K >= ell:
        if np.any(np.sort(p, axis=1)[:, -ell:, :].prod(axis=1) > P.rho2):
            return False
    if np.any(p.sum(axis=(1, 2)) > P.p_max * (1 + tol.box_rel_tol)):
        return False
    rates = user_rates(P, p)
    st = P.streaming
    if st and np.any(P.min_rates[st] - rates[st] > tol.c13_rate_tol):
        return False
    cross = cross_of(P, p)
    g_i, g_j = P.gamma[:, :, None, :], P.gamma[:, None, :, :]
    s_i, s_j = P.sigma[:, :, None, :], P.sigma[:, None, :, :]
    c_i, c_j = cross[:, :, None, :], cross[:, None, :, :]
    omega = g_j * s_i - g_i * s_j + g_j * c_i - g_i * c_j
    scale = g_j * s_i + g_i * s_j + g_j * c_i + g_i * c_j
    pp = p[:, :, None, :] * p[:, None, :, :]
    stronger = P.rank[:, :, None, :] < P.rank[:, None, :, :]
    return not np.any(stronger & (pp * omega > tol.c14_rel_tol * pp * scale) & (pp > 0))


def indicators(P: Prob, p: np.ndarray):
    """rho: top-l_max powers above 1e-6*max_mask per (m, n); a: head with the
    largest total power per user, if above the threshold (model.py:497-521)."""
    M, K, N = P.shape
    eps = 1e-6 * P.max_mask
    per = p.sum(axis=2)
    head = np.argmax(per, axis=0)
    on = per[head, np.arange(K)] > eps
    a = np.zeros((M, K), np.uint8)
    a[head[on], np.nonzero(on)[0]] = 1
    by_power = np.argsort(p, axis=1)[:, ::-1, :]
    ranked = np.take_along_axis(p, by_power, axis=1)
    keep = (ranked > eps) & (np.arange(K)[None, :, None] < P.l_max)
    rho = np.zeros(p.shape, np.uint8)
    np.put_along_axis(rho, by_power, keep.astype(np.uint8), axis=1)
    return rho, a


# ---------------------------------------------------------------------------
# inner solve (scale.py:506-551) and Dinkelbach (dinkelbach.py:65-112)
# ---------------------------------------------------------------------------

@dataclass
class InnerResult:
    p: np.ndarray
    rho: np.ndarray | None
    a: np.ndarray | None
    status: str
    stats: InnerStats


def solve_fixed_e(P: Prob, e: float, warm_p: np.ndarray | None = None,
                  sic: str = "dense") -> InnerResult:
    """sic="device": the B200 default -- the seated-pair SIC model, with the
    inner solve redone from its start with the dense family when it met a
    floor tie (a seat with num == 0 and den <= 0)."""
    if sic == "device":
        res = solve_fixed_e(P, e, warm_p, "seated")
        if res.stats.floor_tie:
            res = solve_fixed_e(P, e, warm_p, "dense")
            res.stats.floor_tie = True
        return res
    ctx = Ctx(P, e, sic)
    stats = InnerStats()
    if warm_p is not None:
        p0 = np.clip(warm_p, ctx.p_floor, P.p_mask)
    else:
        if P.gamma.size <= 16:
            raise ProductsActive("multistart seatings on <= 16 cells")
        p0 = greedy_start(P)
    p, objs = sca_rounds(ctx, p0, stats)
    stats.round_objectives = objs
    stats.rounds = len(objs)
    q, ok = repair(ctx, p)
    if ok:
        ok = feasible(P, q)
    if warm_p is not None:
        if not ok or true_objective(P, q, e) < true_objective(P, warm_p, e):
            q, ok = warm_p.copy(), True
    if not ok:
        stats.status = "infeasible"
        stats.infeasible_reason = stats.infeasible_reason or \
            "repair could not meet the streaming rates"
        return InnerResult(q, None, None, "infeasible", stats)
    rho, a = indicators(P, q)
    stats.true_objective = true_objective(P, q, e)
    stats.floor_tie = ctx.floor_tie
    return InnerResult(q, rho, a, "ok", stats)


@dataclass
class Trace:
    e_values: list = field(default_factory=list)
    surplus: list = field(default_factory=list)
    inner: list = field(default_factory=list)
    final_e: float = 0.0
    p: np.ndarray | None = None
    rho: np.ndarray | None = None
    a: np.ndarray | None = None
    status: str = "converged"
    floor_tie: bool = False


def dinkelbach(P: Prob, e0: float = 0.0, sic: str = "dense") -> Trace:
    """sic="dense": the reference.  sic="device": the B200 default path
    (see solve_fixed_e)."""
    tol = P.tol
    tr = Trace()
    e = e0
    warm = None
    for _ in range(tol.outer_max):
        res = solve_fixed_e(P, e, warm.p if warm is not None else None, sic)
        if getattr(res.stats, "floor_tie", False):
            tr.floor_tie = True
        if res.status != "ok":
            if warm is None:
                raise Infeasible(res.stats.infeasible_reason)
            tr.status = "stalled"
            break
        warm = res
        r, pw, ee = report(P, res.p)
        s = r - e * pw
        tr.e_values.append(e)
        tr.surplus.append(s)
        tr.inner.append(res.stats)
        if s <= tol.xi:
            tr.final_e, tr.p, tr.rho, tr.a, tr.status = ee, res.p, res.rho, res.a, "converged"
            return tr
        if ee <= e:
            tr.status = "stalled"
            break
        e = ee
    else:
        tr.status = "cap"
    tr.final_e = report(P, warm.p)[2]
    tr.p, tr.rho, tr.a = warm.p, warm.rho, warm.a
    return tr
