import sys, os, ctypes as C, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1803_07772_b200 import solver, pack, _abi
from paper_1803_07772_b200.scenarios import workload_batch
lib = solver.library()
for name in sys.argv[1:]:
    b = workload_batch(name, range(1))
    prob = solver._DeviceProblem(b.cfg, b.sigma, torch.device('cuda'))
    eng, cs, sm = C.c_int32(), C.c_int32(), C.c_size_t()
    lib.hcran_b200_engine(C.byref(prob.struct), 1024, 0, C.byref(eng), C.byref(cs), C.byref(sm))
    g, w = C.c_int32(), C.c_size_t()
    lib.hcran_b200_plan(C.byref(prob.struct), 1024, 0, C.byref(g), C.byref(w))
    print(name, 'engine', eng.value, 'cluster', cs.value, 'smem', sm.value, 'grid', g.value, 'ws MB', w.value / 2**20)
