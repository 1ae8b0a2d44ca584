"""Reference rows of the acceptance campaigns (test_acceptance.py:34-96:
criteria 1-3, seed 11, 50 draws, K = 12, N = 32) from the UNMODIFIED
reference's run_sweep, for tests/test_acceptance_gpu.py:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_acceptance_golden.py
"""

import json
import os

from hcran_noma.scenarios import Scenario, run_sweep

CAMPAIGNS = {
    "noma": dict(architecture="hcran", sweep="none", values=(12,), l_max=3),
    "oma": dict(architecture="hcran", sweep="none", values=(12,), l_max=1),
    "streaming": dict(architecture="hcran", sweep="streaming", values=(2, 4, 6), l_max=3),
    "arrival": dict(architecture="hcran", sweep="arrival", values=(75.0, 100.0, 125.0), l_max=3),
}
for arch in ("hcran", "cran", "hcn", "hpn1"):
    CAMPAIGNS[f"users_{arch}"] = dict(architecture=arch, sweep="users", values=(10, 12, 16), l_max=3)


def scenario(kw, workers):
    return Scenario(architecture=kw["architecture"], sweep=kw["sweep"], values=kw["values"],
                    k_total=12, k_streaming=6, arrival_rate=125.0, l_max=kw["l_max"],
                    n_subcarriers=32, draws=50, seed=11, workers=workers)


def main():
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "acceptance_rows.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name, kw in CAMPAIGNS.items():
        if name in out:
            continue
        rows = run_sweep(scenario(kw, max(1, (os.cpu_count() or 2) - 1)))
        out[name] = {"scenario": {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()},
                     "rows": [r.__dict__ for r in rows]}
        json.dump(out, open(path, "w"), indent=1)
        print(name, [(r.value, r.mean_ee, r.n_feasible) for r in rows], flush=True)


if __name__ == "__main__":
    main()
