"""Instance loader (scenarios.py restatement) reproduces the reference's draws
bit-for-bit: gamma digests recorded from the reference in tests/golden."""

import hashlib

import numpy as np
import pytest

from paper_1803_07772_b200 import min_rate_for_delay, TrafficSpec
from paper_1803_07772_b200.scenarios import workload_batch, workload_instance


def digest(g):
    return hashlib.sha256(np.ascontiguousarray(g, np.float64).tobytes()).hexdigest()[:16]


@pytest.mark.parametrize("name,count", [("c0", 128), ("c1", 24), ("c2", 7), ("c4", 256)])
def test_gamma_digests(golden, name, count):
    g = golden(name)
    for i in range(count):
        _, ch, _ = workload_instance(name, int(g["draw"][i]))
        assert digest(ch.gamma) == g["gamma_digest"][i]


def test_batch_matches_single():
    b = workload_batch("c4", range(8))
    for i in range(8):
        cfg, ch, e = workload_instance("c4", i)
        assert np.array_equal(b.gamma[i], ch.gamma)
        assert b.e_fixed[i] == e
        assert np.array_equal(b.elastic[i], cfg.elastic_mask())
        assert np.array_equal(b.min_rates[i], cfg.min_rates())


def test_min_rate_kat():
    # traffic.py KAT (test_traffic.py:40-48): Psi = 4.18 at lam=125, T=0.2, z=1024, b_n=31.25 kHz
    spec = TrafficSpec.from_queue(25.0, 125.0, 1024.0)
    assert abs(min_rate_for_delay(spec, 31250.0) - 4.18) < 0.01
