"""config[3] on one B200: a small batch through the device path (SIC mode from argv),
device time and full-size invariants.  python tools/c3_probe.py B [exact|fast|default]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1803_07772_b200 import solve_batch
from paper_1803_07772_b200.scenarios import workload_batch
B = int(sys.argv[1]); mode = sys.argv[2] if len(sys.argv) > 2 else 'fast'
exact = {'fast': 'fast', 'exact': True, 'default': False}[mode]
t0 = time.time(); b = workload_batch('c3', range(B)); print('gen %.1f s' % (time.time() - t0), flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g = torch.from_numpy(b.gamma).cuda()
e0.record(); o = solve_batch(b.cfg, g, b.sigma, b.elastic, b.min_rates, exact=exact); e1.record(); torch.cuda.synchronize()
o = {k: v.cpu().numpy() for k, v in o.items() if hasattr(v, 'cpu')}
print('c3 B', B, mode, 'device s %.2f' % (e0.elapsed_time(e1) / 1e3), 'inst/s %.3f' % (B / e0.elapsed_time(e1) * 1e3))
print('status', np.bincount(o['status'], minlength=5), 'flags', np.bincount(o['flags'], minlength=4), 'feasible', o['feasible'].mean())
print('ee', np.round(o['ee'], 4).tolist(), 'iters', o['outer_iters'].tolist(), 'sweeps', o['sweeps'].tolist())
ok = o['status'] <= 2
print('EE=R/P', np.allclose(o['ee'][ok], o['sum_rate'][ok] / o['total_power'][ok], rtol=1e-12))
