"""Timing probe at config[3] (device-synthesised inputs): one wave per SIC mode."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_07772_b200 import solve_batch, synth_gamma
from paper_1803_07772_b200.scenarios import gen_sigma, workload_instance
mode, B = sys.argv[1], int(sys.argv[2])
cfg, _, _ = workload_instance("c3", 0)
g = synth_gamma(cfg, 0, B)
t = time.time()
o = solve_batch(cfg, g, gen_sigma(cfg), exact={"default": False, "fast": "fast", "dense": True}[mode],
                outputs=["ee", "status", "flags", "sweeps", "outer_iters"])
dt = time.time() - t
st = o["status"].cpu().numpy(); fl = o["flags"].cpu().numpy()
print(mode, B, "s", round(dt, 1), "inst/s", round(B / dt, 2), "status", np.bincount(st, minlength=5).tolist(),
      "flags", np.bincount(fl, minlength=4).tolist(), "sweeps", float(o["sweeps"].double().mean()), flush=True)
