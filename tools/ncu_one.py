import sys, os
sys.path.insert(0, os.getcwd())
from paper_1803_07772_b200 import solve_batch
from paper_1803_07772_b200.scenarios import workload_batch
name = sys.argv[1]; nb = int(sys.argv[2])
b = workload_batch(name, range(nb))
o = solve_batch(b.cfg, b.gamma, b.sigma)
print("ok", float(o["ee"].mean()))
