import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'tests'))
from paper_1803_07772_b200 import solve_batch
from paper_1803_07772_b200.scenarios import workload_batch
from emu import runner
name = sys.argv[1] if len(sys.argv) > 1 else 'c1'
g = dict(np.load(f'tests/golden/{name}_0_{ {"c1":24,"c0":128,"c2":7}[name] }.npz'))
idx = np.arange(len(g['draw']))
b = workload_batch(name, g['draw'])
o = {k: (v.cpu().numpy() if hasattr(v, 'cpu') else v) for k, v in solve_batch(b.cfg, b.gamma, b.sigma).items() if not k.startswith('_')}
e = runner.run(b.cfg, b.gamma, b.sigma, mode=0)
for i in idx:
    rg = abs(o['ee'][i]-g['ee'][i])/g['ee'][i]; rp = abs(o['total_power'][i]-g['total_power'][i])/g['total_power'][i]
    same = np.array_equal(o['rho'][i], g['rho'][i]) and np.array_equal(o['a'][i], g['a'][i])
    re = abs(e['ee'][i]-g['ee'][i])/g['ee'][i]
    print(i, 'dev ee rel %.2e P rel %.2e same %d | emu rel %.2e | it dev %d emu %d ref %d | sweeps dev %d emu %d | st %d %d flags %d %d nt %d' % (
        rg, rp, same, re, o['outer_iters'][i], e['outer_iters'][i], np.sum(~np.isnan(g['e_values'][i])),
        o['sweeps'][i], e['sweeps'][i], o['status'][i], g['status'][i], o['flags'][i], e['flags'][i], g['near_tie'][i]))
    if not same:
        d = np.argwhere(o['rho'][i] != g['rho'][i]); print('    rho diff at', d[:6].tolist())
