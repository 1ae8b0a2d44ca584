"""Desk-scale parity: the reference's own unit-test networks
and tiny_instance draws, where it runs the <= 16-cell multistart (greedy by
score, greedy by peak gain, fully open seating; scale.py:512-518, 1063-1071)
and the products-active theta family (scale.py:696-703, 761-763, 835-840).
Reference outputs: tests/golden/tiny_cases.npz (make_tiny_golden.py).
CPU: host build of the device solver; GPU: the sm_100a library (C ABI)."""

import numpy as np
import pytest

from tiny_common import check, load_cases, run_case

CASES = load_cases()


def _emu(cfg, g, sigma, mode, e, warm):
    from emu import runner
    return runner.run(cfg, g, sigma, mode=mode, e_fixed=e, warm_p=warm)


def _gpu(cfg, g, sigma, mode, e, warm):
    from paper_1803_07772_b200 import solve_batch
    o = solve_batch(cfg, g, sigma, mode="dinkelbach" if mode == 0 else "fixed_e", e_fixed=e,
                    warm_p=warm)
    return {k: v.cpu().numpy() for k, v in o.items() if hasattr(v, "cpu")}


def _run_all(solve):
    bad, n = [], 0
    for name, ref in CASES.items():
        if bool(ref["near_tie"]):
            continue
        n += 1
        bad += check(name, ref, run_case(name, ref, solve))
    return bad, n


def test_tiny_cases_host_build():
    bad, n = _run_all(_emu)
    assert n >= 100
    assert bad == []


@pytest.mark.gpu
def test_tiny_cases_b200():
    bad, n = _run_all(_gpu)
    assert n >= 100
    assert bad == []
