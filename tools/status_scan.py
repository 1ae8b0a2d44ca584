import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_07772_b200 import solve_batch
from paper_1803_07772_b200.scenarios import workload_batch
name, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
b = workload_batch(name, range(lo, hi))
o = solve_batch(b.cfg, b.gamma, b.sigma)
st = o['status'].cpu().numpy(); it = o['outer_iters'].cpu().numpy(); ee = o['ee'].cpu().numpy()
fl = o['flags'].cpu().numpy(); sw = o['sweeps'].cpu().numpy()
for i in range(hi - lo):
    print(lo + i, int(st[i]), int(it[i]), int(sw[i]), int(fl[i]), repr(float(ee[i])))
