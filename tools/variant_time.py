"""Device time of one solve for the library in HCRAN_LIB: config, batch sizes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1803_07772_b200 import DeviceProblem, solve_batch
from paper_1803_07772_b200.scenarios import workload_batch
name = sys.argv[1]
for B in [int(x) for x in sys.argv[2:]]:
    b = workload_batch(name, range(B))
    prob = DeviceProblem(b.cfg, b.sigma)
    g = torch.from_numpy(b.gamma).cuda()
    solve_batch(b.cfg, g, None, b.elastic, b.min_rates, problem=prob)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); solve_batch(b.cfg, g, None, b.elastic, b.min_rates, problem=prob, sync=False); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(os.path.basename(os.environ.get('HCRAN_LIB', 'default')), name, B, 'ms %.1f' % min(ts), 'inst/s %.0f' % (B / min(ts) * 1e3), flush=True)
