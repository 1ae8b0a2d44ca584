"""Dump per-instance device outcomes of a workload range to gpurun_out/ (npz):
status, flags, outer iterations, EE, total power -- used to pick the draws
whose reference outcome is pinned by fixtures (tests/golden/make_golden.py)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_07772_b200 import solve_batch  # noqa: E402
from paper_1803_07772_b200.scenarios import workload_batch  # noqa: E402

name, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
chunk = int(sys.argv[4]) if len(sys.argv) > 4 else hi - lo
acc = {}
for a in range(lo, hi, chunk):
    b = workload_batch(name, range(a, min(hi, a + chunk)))
    o = solve_batch(b.cfg, b.gamma, b.sigma,
                    outputs=["status", "flags", "outer_iters", "ee", "total_power", "sweeps"])
    for k in ("status", "flags", "outer_iters", "ee", "total_power", "sweeps"):
        acc.setdefault(k, []).append(o[k].cpu().numpy())
out = {k: np.concatenate(v) for k, v in acc.items()}
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/status_{name}_{lo}_{hi}.npz", draws=np.arange(lo, hi), **out)
u, c = np.unique(out["status"], return_counts=True)
print(name, lo, hi, dict(zip(u.tolist(), c.tolist())))
