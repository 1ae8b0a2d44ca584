"""M/G/1 delay bound -> minimum physical-layer rate (one host scalar per
streaming user).

Mirrors /root/reference/pkg/src/hcran_noma/traffic.py: `TrafficSpec`
(traffic.py:17-56), `max_delay_from_queue` (traffic.py:59-63), `delay_roots`
(traffic.py:66-81) and `min_rate_for_delay` (traffic.py:84-100), evaluated in
the cancellation-free conjugate form.
"""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class TrafficSpec:
    lam: float          # packets/s
    t_max: float        # s, mean delay bound
    packet_bits: float  # bits
    q_len: float | None = None

    def __post_init__(self) -> None:
        if self.lam <= 0 or self.t_max <= 0 or self.packet_bits <= 0:
            raise ValueError("arrival rate, delay bound and packet size must be positive")
        if self.q_len is not None and not math.isclose(self.q_len / self.lam, self.t_max,
                                                       rel_tol=1e-9):
            raise ValueError("queue length inconsistent with t_max = q/lam")

    @classmethod
    def from_queue(cls, q_len: float, lam: float, packet_bits: float) -> "TrafficSpec":
        return cls(lam=lam, t_max=max_delay_from_queue(q_len, lam),
                   packet_bits=packet_bits, q_len=q_len)


def max_delay_from_queue(q_len: float, lam: float) -> float:
    if lam <= 0:
        raise ValueError(f"arrival rate must be positive, got {lam}")
    return q_len / lam


def delay_roots(lam: float, t_max: float) -> tuple[float, float]:
    """Roots of lam*x^2 - (2+2*lam*T)*x + 2*T; the small one in conjugate form."""
    if lam <= 0 or t_max <= 0:
        raise ValueError("lam and t_max must be positive")
    lt = lam * t_max
    s = math.sqrt(1.0 + lt * lt)
    return 2.0 * t_max / (1.0 + lt + s), (1.0 + lt + s) / lam


def min_rate_for_delay(spec: TrafficSpec, subcarrier_bandwidth: float) -> float:
    """Psi = z*(1 + lam*T + sqrt(1 + (lam*T)^2)) / (2T) / b_n  (bits/s/Hz)."""
    if subcarrier_bandwidth <= 0:
        raise ValueError("subcarrier bandwidth must be positive")
    lt = spec.lam * spec.t_max
    rate_hz = spec.packet_bits * (1.0 + lt + math.sqrt(1.0 + lt * lt)) / (2.0 * spec.t_max)
    return rate_hz / subcarrier_bandwidth
