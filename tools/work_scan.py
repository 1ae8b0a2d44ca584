"""Per-instance work distribution of a batch (device run): top instances and
gpurun_out/work_{name}.npz for tools/sched_sim.py."""
import sys, os, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1803_07772_b200 import solve_batch
from paper_1803_07772_b200.scenarios import workload_batch
name, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
b = workload_batch(name, range(lo, hi))
o = {k: v.cpu().numpy() for k, v in solve_batch(b.cfg, b.gamma, b.sigma).items() if hasattr(v, 'cpu')}
w = o['work']; idx = np.argsort(-w)[:12]
print('work mean', w.mean(), 'max', w.max(), 'p99', np.percentile(w, 99))
for i in idx: print(lo + i, 'work %.3g' % w[i], 'st', o['status'][i], 'it', o['outer_iters'][i], 'sweeps', o['sweeps'][i], 'flags', o['flags'][i], 'evals', o['bisect_evals'][i])
os.makedirs(os.path.join(ROOT, 'gpurun_out'), exist_ok=True)
np.savez(os.path.join(ROOT, 'gpurun_out', f'work_{name}.npz'), work=w, flags=o['flags'], sweeps=o['sweeps'],
         iters=o['outer_iters'], status=o['status'])
