"""config[3] parity proxy (the reference cannot run c3: MemoryError,
SURVEY.md 6): the default SIC model (seated pairs, floor ties re-run dense)
against the exact dense pair family on device-synthesised c3 instances."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_07772_b200 import solve_batch, synth_gamma  # noqa: E402
from paper_1803_07772_b200.scenarios import gen_sigma, workload_instance  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg, _, _ = workload_instance("c3", 0)
g = synth_gamma(cfg, 0, B)
sig = gen_sigma(cfg)
out = {}
for mode, exact in (("default", False), ("dense", True)):
    t = time.time()
    o = solve_batch(cfg, g, sig, exact=exact, outputs=["ee", "total_power", "status", "rho", "a",
                                                       "flags", "sweeps"])
    out[mode] = {k: v.cpu().numpy() for k, v in o.items() if hasattr(v, "cpu")}
    print(mode, "s", round(time.time() - t, 1), "status", np.bincount(out[mode]["status"], minlength=5),
          "flags", np.bincount(out[mode]["flags"], minlength=4), flush=True)
a, b = out["default"], out["dense"]
rel_ee = np.abs(a["ee"] - b["ee"]) / np.abs(b["ee"])
rel_p = np.abs(a["total_power"] - b["total_power"]) / np.abs(b["total_power"])
same = [bool(np.array_equal(a["rho"][i], b["rho"][i]) and np.array_equal(a["a"][i], b["a"][i]))
        for i in range(B)]
print("max rel EE", rel_ee.max(), "max rel P", rel_p.max(), "rho/a equal", sum(same), "/", B)
np.savez("gpurun_out/c3_proxy.npz", **{f"{m}_{k}": v for m, d in out.items() for k, v in d.items()})
