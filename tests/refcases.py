"""The reference's hand-built unit-test networks, restated with this package's
types (mirror of /root/reference/pkg/tests/conftest.py:8-44: users on a line,
flat mask p_max/N, static 3+1 / 3+0.1 W), and the list of reference test
cases (test_scale.py:343-383, test_dinkelbach.py:62-110) that
tests/golden/make_tiny_golden.py pins with reference outputs."""

from __future__ import annotations

import numpy as np

from paper_1803_07772_b200.model import ChannelState, NetworkConfig, Tolerances, UserSpec
from paper_1803_07772_b200.traffic import TrafficSpec


def make_config(m=2, k=3, n=2, streaming=(), l_max=3, p_max=None, eta=None, bandwidth=31250.0,
                arrival=125.0, queue=25.0, bits=1024.0, weights=None, tolerances=None):
    traffic = TrafficSpec.from_queue(queue, arrival, bits)
    users = tuple(UserSpec(kind="streaming" if i in streaming else "elastic",
                           position=(100.0 * (i + 1), 50.0),
                           traffic=traffic if i in streaming else None) for i in range(k))
    p_max = np.asarray(p_max if p_max is not None else [2.0] * m, dtype=float)
    mask = np.broadcast_to((p_max / n)[:, None, None], (m, k, n)).copy()
    return NetworkConfig(
        m_f=m - 1, n_subcarriers=n, subcarrier_bandwidth=bandwidth, users=users, l_max=l_max,
        p_max=p_max, p_mask=mask,
        eta=np.asarray(eta if eta is not None else [2.0] * m, dtype=float),
        p_fiber_hpn=3.0, p_fiber_lpn=1.0, p_circuit_hpn=3.0, p_circuit_lpn=0.1,
        weights=np.ones((m, k)) if weights is None else np.asarray(weights, dtype=float),
        rrh_positions=np.stack([np.array([300.0 * j, 0.0]) for j in range(m)]),
        tolerances=tolerances or Tolerances())


def make_channel(cfg, seed=0, gamma_scale=1e-7):
    rng = np.random.default_rng(seed)
    shape = (cfg.n_rrh, cfg.n_users, cfg.n_subcarriers)
    gamma = rng.exponential(gamma_scale, size=shape)
    sigma = np.full(shape, cfg.noise_density * cfg.subcarrier_bandwidth)
    return ChannelState(gamma=gamma, sigma=sigma)


# (name, make_config kwargs, channel seed, gamma_scale, mode, e)
#   mode "fixed": ScaleSolver().solve_fixed_e(ch, cfg, e); "warm": a second
#   solve at e warm-started from the e=0 result; "dinkel": dinkelbach.solve
UNIT_CASES = (
    [(f"rounds_nondecreasing_{s}", dict(m=2, k=4, n=3, streaming=(0,)), 30 + s, 1e-7, "fixed", 0.5 * s)
     for s in range(6)]                                                     # test_scale.py:343-350
    + [(f"output_feasible_{s}", dict(m=2, k=4, n=3, streaming=(0, 1)), 40 + s, 1e-7, "fixed", 0.3)
       for s in range(5)]                                                   # test_scale.py:352-358
    + [("fixed_point_residual", dict(m=1, k=2, n=2), 50, 1e-7, "fixed", 0.5),         # :360-364
       ("infeasible_detection", dict(m=1, k=2, n=1, streaming=(0,), bandwidth=1e-3), 51, 1e-7,
        "fixed", 0.0),                                                                # :366-370
       ("never_worse_than_warm", dict(m=2, k=4, n=3, streaming=(0,)), 52, 1e-7, "warm", 1.0),
       ("small_default", dict(), 0, 1e-7, "fixed", 0.4),                               # conftest small
       ("monotone_e", dict(m=2, k=4, n=3, streaming=(0,)), 5, 1e-7, "dinkel", 0.0),    # test_dinkelbach.py:72-79
       ("infeasible_raises", dict(m=1, k=2, n=1, streaming=(0,), bandwidth=1e-3), 6, 1e-7,
        "dinkel", 0.0),                                                                 # :81-86
       ("grid_oracle", dict(m=1, k=2, n=2, p_max=[1.0]), 9, 1e-8, "dinkel", 0.0),      # :112-132
       ("small_streaming", dict(streaming=(0,)), 7, 1e-7, "dinkel", 0.0)]
)

TINY_SEED = 11  # tiny_instance(default_rng([TINY_SEED, d])) (scenarios.py:310-327)
