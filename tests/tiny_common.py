"""Shared driver of the desk-scale parity cases (tests/golden/tiny_cases.npz,
make_tiny_golden.py): rebuild each case's network with this package's types and
solve it through a backend (the sm_100a library, or the host build of the same
solver source for the CPU suite)."""

from __future__ import annotations

import os

import numpy as np

from conftest import GOLDEN, rel
from refcases import UNIT_CASES, make_config
from paper_1803_07772_b200.scenarios import tiny_instance


def load_cases():
    z = np.load(os.path.join(GOLDEN, "tiny_cases.npz"))
    cases = {}
    for key in z.files:
        name, field = key.split("/")
        cases.setdefault(name, {})[field] = z[key]
    return cases


def network(name):
    if name.startswith("tiny_"):
        _, seed, d = name.split("_")
        inst = tiny_instance(np.random.default_rng([int(seed), int(d)]))
        return inst.cfg
    kw = next(c[1] for c in UNIT_CASES if c[0] == name)
    return make_config(**kw)


def check(name, ref, out, counts=True):
    """[] when the backend output `out` (dict of arrays, batch of 1) matches the
    reference case `ref`; else a list of mismatch descriptions."""
    bad = []
    if int(out["status"][0]) != int(ref["status"]):
        return [f"{name}: status {int(out['status'][0])} vs {int(ref['status'])}"]
    if "p" not in ref:
        return bad
    key = "objective" if "objective" in ref else "ee"
    if rel(float(out[key][0]), float(ref[key])) > 1e-4:
        bad.append(f"{name}: {key} {float(out[key][0])} vs {float(ref[key])}")
    if "rho" in ref and not (np.array_equal(out["rho"][0], ref["rho"]) and
                             np.array_equal(out["a"][0], ref["a"])):
        bad.append(f"{name}: rho/a differ")
    if counts and "rounds" in ref and (int(out["rounds"][0]) != int(ref["rounds"]) or
                                       int(out["sweeps"][0]) != int(ref["sweeps"])):
        bad.append(f"{name}: rounds/sweeps {int(out['rounds'][0])}/{int(out['sweeps'][0])} vs "
                   f"{int(ref['rounds'])}/{int(ref['sweeps'])}")
    return bad


def run_case(name, ref, solve):
    """solve(cfg, gamma[1], sigma, mode, e_fixed, warm_p) -> dict of arrays."""
    cfg = network(name)
    mode = str(ref["mode"])
    g = ref["gamma"][None]
    if mode == "dinkel":
        return solve(cfg, g, ref["sigma"], 0, None, None)
    warm = ref["warm_p"][None] if mode == "warm" else None
    return solve(cfg, g, ref["sigma"], 1, np.array([float(ref["e"])]), warm)
