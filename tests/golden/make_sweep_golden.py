"""Golden rows of the reference's `run_sweep` (scenarios.py:266-296) for the
batcher parity test.  Runs the unmodified reference in this container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_sweep_golden.py
"""

import json
import os

from hcran_noma.scenarios import Scenario, run_sweep

SCENARIOS = {
    "users": dict(architecture="hcran", sweep="users", values=(5, 7), k_total=6, k_streaming=2,
                  n_subcarriers=8, draws=6, seed=3, workers=6),
    "streaming": dict(architecture="hcran", sweep="streaming", values=(0, 3), k_total=6,
                      k_streaming=2, n_subcarriers=8, draws=6, seed=5, workers=6),
    "lpn": dict(architecture="hcran", sweep="lpn", values=(1, 3), k_total=6, k_streaming=2,
                n_subcarriers=8, draws=6, seed=7, workers=6),
    "cran": dict(architecture="cran", sweep="none", values=(0,), k_total=6, k_streaming=2,
                 n_subcarriers=8, draws=6, seed=9, workers=6),
}


def main():
    out = {}
    for name, kw in SCENARIOS.items():
        rows = run_sweep(Scenario(**kw))
        out[name] = {"scenario": {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()},
                     "rows": [r.__dict__ for r in rows]}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "sweep_rows.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, default=float)
    print("wrote", path)


if __name__ == "__main__":
    main()
