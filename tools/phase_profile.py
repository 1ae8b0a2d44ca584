"""Build a -DHCRAN_PROFILE copy of the library and print per-phase cycle shares."""
import ctypes as C, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1803_07772_b200 import build as B, solver
lib_path = os.path.join(ROOT, 'tools', 'libhcran_prof.so')
if not os.path.exists(lib_path) or os.path.getmtime(lib_path) < os.path.getmtime(B.LIB):
    B.build_lib(lib_path, extra=['-DHCRAN_PROFILE'])
solver.LIB_PATH = lib_path
lib = solver.library()
lib.hcran_b200_phase_cycles.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
from paper_1803_07772_b200 import solve_batch
from paper_1803_07772_b200.scenarios import workload_batch
name = sys.argv[1] if len(sys.argv) > 1 else 'c1'
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 256
b = workload_batch(name, range(nb))
out = (C.c_ulonglong * 32)()
solve_batch(b.cfg, b.gamma, b.sigma)
lib.hcran_b200_phase_cycles(out, 1)
o = solve_batch(b.cfg, b.gamma, b.sigma)
lib.hcran_b200_phase_cycles(out, 0)
# thread 0 (warp 0) clock per phase; marks 1-5 are warp 0's own subcarriers
names = {0: 'sw:products', 1: 'an:tables+full+utot', 2: 'an:columns (psi, own)', 3: 'an:dense family',
         4: 'an:num/den', 12: 'fast:stage', 13: 'fast:rows', 14: 'fast:columns', 15: 'fast:seats+own',
         20: 'fast:num/den', 21: 'fast:tail', 24: 'sw:analyze tail',
         25: 'sw:dense update', 26: 'sw:budget multiplier', 7: 'sw:closed form+zeta', 8: 'sw:convergence',
         10: 'round_start', 11: 'round end (surrogate, stops)',
         16: 'inner:setup', 17: 'inner:rounds', 18: 'inner:repair', 19: 'inner:feasible',
         27: 'repair:prune+rescale', 28: 'repair:trim', 29: 'repair:boost', 30: 'repair:sic_cleanup', 31: 'repair:final rates'}
tot = sum(out[i] for i in (0, 1, 2, 3, 4, 12, 13, 14, 15, 20, 21, 24, 25, 26, 7, 8)) or 1
print('sweeps', int(o['sweeps'].sum().item()), 'instances', nb)
for i in range(32):
    if out[i]:
        print(f"{names.get(i, i):28s} {out[i]/1e9:9.3f} Gcyc  {100*out[i]/max(tot,1):6.1f}% of sweep")
