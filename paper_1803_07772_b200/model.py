"""Host-side problem description: the reference's data types, same field names.

These mirror `hcran_noma.model` (/root/reference/pkg/src/hcran_noma/model.py)
so that a caller of the reference can hand either the reference's objects or
these to the B200 solver (attribute-compatible, duck-typed):

* `Tolerances`      model.py:59-80   (same defaults; v_max=120 as in the code)
* `UserSpec`        model.py:42-56
* `NetworkConfig`   model.py:83-185  (p_max, p_mask, eta, weights, users, l_max, ...)
* `ChannelState`    model.py:188-201 (gamma, sigma: (M, K, N))
* `PowerAllocation` model.py:204-217 (p, rho, a)
* `EnergyReport`    model.py:220-224

Nothing here computes rates or powers: that is device work (csrc/).  The only
arithmetic is the per-config constants the device needs (static power,
minimum rates), which are scalars per config.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .traffic import TrafficSpec, min_rate_for_delay

LN2 = float(np.log(2.0))


def dbm_to_watts(dbm: float) -> float:
    return 10.0 ** ((dbm - 30.0) / 10.0)


class ConfigError(ValueError):
    """Structural invariant violated (reference: model.py:38-39)."""


@dataclass(frozen=True)
class UserSpec:
    kind: str                       # "elastic" | "streaming"
    position: tuple[float, float]   # metres
    traffic: TrafficSpec | None = None

    def __post_init__(self) -> None:
        if self.kind not in ("elastic", "streaming"):
            raise ConfigError(f"unknown user kind {self.kind!r}")
        if (self.kind == "streaming") != (self.traffic is not None):
            raise ConfigError("streaming users (and only they) carry a TrafficSpec")


@dataclass(frozen=True)
class Tolerances:
    xi: float = 0.01
    varpi1_rel: float = 1e-4
    varpi2_rel: float = 1e-3
    s_max: int = 20
    v_max: int = 120
    outer_max: int = 30
    rho1: float | None = None
    rho2: float | None = None
    dual_cap: float = 1e8
    c13_rate_tol: float = 1e-6
    c14_rel_tol: float = 1e-9
    box_rel_tol: float = 1e-9


@dataclass(frozen=True)
class NetworkConfig:
    m_f: int
    n_subcarriers: int
    subcarrier_bandwidth: float
    users: tuple[UserSpec, ...]
    l_max: int
    p_max: np.ndarray
    p_mask: np.ndarray
    eta: np.ndarray
    p_fiber_lpn: float
    p_fiber_hpn: float
    p_circuit_lpn: float
    p_circuit_hpn: float
    weights: np.ndarray
    rrh_positions: np.ndarray
    noise_density: float = dbm_to_watts(-174.0)
    tolerances: Tolerances = field(default_factory=Tolerances)

    def __post_init__(self) -> None:
        m, k, n = self.n_rrh, self.n_users, self.n_subcarriers
        if self.m_f < 0 or n <= 0 or k <= 0:
            raise ConfigError("need at least one RRH, user and subcarrier")
        if self.l_max < 1:
            raise ConfigError("l_max must be >= 1")
        if self.subcarrier_bandwidth <= 0 or self.noise_density <= 0:
            raise ConfigError("bandwidth and noise density must be positive")
        for name, shape in (("p_max", (m,)), ("p_mask", (m, k, n)), ("eta", (m,)),
                            ("weights", (m, k)), ("rrh_positions", (m, 2))):
            if np.shape(getattr(self, name)) != shape:
                raise ConfigError(f"{name} has shape {np.shape(getattr(self, name))}, "
                                  f"expected {shape}")
        if np.any(self.p_max <= 0) or np.any(self.p_mask <= 0) or np.any(self.eta <= 0):
            raise ConfigError("powers and efficiencies must be strictly positive")
        if np.any(self.p_mask > self.p_max[:, None, None] * (1 + 1e-12)):
            raise ConfigError("p_mask must not exceed the per-RRH budget")
        if np.any(self.weights < 0) or np.any(self.weights > 1):
            raise ConfigError("weights must lie in [0, 1]")

    @property
    def n_rrh(self) -> int:
        return self.m_f + 1

    @property
    def n_users(self) -> int:
        return len(self.users)

    def streaming_users(self) -> list[int]:
        return [i for i, u in enumerate(self.users) if u.kind == "streaming"]

    def elastic_users(self) -> list[int]:
        return [i for i, u in enumerate(self.users) if u.kind == "elastic"]

    def elastic_mask(self) -> np.ndarray:
        return np.array([u.kind == "elastic" for u in self.users], dtype=bool)

    @property
    def max_mask(self) -> float:
        return float(np.max(self.p_mask))

    @property
    def rho1(self) -> float:
        r = self.tolerances.rho1
        return r if r is not None else 1e-6 * self.max_mask ** 2

    @property
    def rho2(self) -> float:
        r = self.tolerances.rho2
        return r if r is not None else 1e-6 * self.max_mask ** (self.l_max + 1)

    @property
    def binarization_threshold(self) -> float:
        return 1e-6 * self.max_mask

    def static_power(self) -> float:
        return (self.p_fiber_hpn + self.m_f * self.p_fiber_lpn
                + self.m_f * self.p_circuit_lpn + self.p_circuit_hpn)

    def min_rates(self) -> np.ndarray:
        out = np.zeros(self.n_users)
        for k in self.streaming_users():
            out[k] = min_rate_for_delay(self.users[k].traffic, self.subcarrier_bandwidth)
        return out


@dataclass(frozen=True)
class ChannelState:
    gamma: np.ndarray   # (M, K, N) linear power gains
    sigma: np.ndarray   # (M, K, N) noise powers, W

    def __post_init__(self) -> None:
        if np.shape(self.gamma) != np.shape(self.sigma) or np.ndim(self.gamma) != 3:
            raise ConfigError("gamma and sigma must share an (M, K, N) shape")


@dataclass
class PowerAllocation:
    p: np.ndarray
    rho: np.ndarray | None = None
    a: np.ndarray | None = None

    def copy(self) -> "PowerAllocation":
        return PowerAllocation(p=self.p.copy(),
                               rho=None if self.rho is None else self.rho.copy(),
                               a=None if self.a is None else self.a.copy())


@dataclass(frozen=True)
class EnergyReport:
    sum_rate: float
    total_power: float
    ee: float
