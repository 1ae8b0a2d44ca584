import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1803_07772_b200 import solve_batch
from paper_1803_07772_b200.scenarios import workload_batch
name = sys.argv[1]; n = int(sys.argv[2])
b = workload_batch(name, range(n))
try:
    o = solve_batch(b.cfg, b.gamma, b.sigma)
    print('ok', o['ee'].cpu().numpy()[:4], o['status'].cpu().numpy()[:8], o['sweeps'].cpu().numpy()[:4])
except Exception as e:
    print('ERR', repr(e))
