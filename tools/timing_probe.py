"""Why does the e2e loop beat the device-timed loop?  Time variants of the step."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_1803_07772_b200 import solve_batch
from paper_1803_07772_b200.scenarios import workload_batch
b = workload_batch('c1', range(1024))
dev = torch.device('cuda')
g = torch.from_numpy(b.gamma).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
want = ["p", "rho", "a", "ee", "sum_rate", "total_power", "status", "outer_iters"]
def run(tag, n=4, do_flush=True, outputs=None, sync_each=False):
    for _ in range(2): solve_batch(b.cfg, g, b.sigma, b.elastic, b.min_rates, sync=True, outputs=outputs)
    ts = []
    for s in range(n):
        if do_flush: flush.random_(0, 255)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record()
        o = solve_batch(b.cfg, g, b.sigma, b.elastic, b.min_rates, sync=False, outputs=outputs)
        e1.record()
        h1 = time.perf_counter()
        if sync_each: torch.cuda.synchronize()
        ts.append((e0, e1, h1 - h0))
    torch.cuda.synchronize()
    print(tag, ['%.1f ms (host %.1f)' % (a.elapsed_time(c), 1e3 * h) for a, c, h in ts], flush=True)
run('flush,all')
run('noflush,all', do_flush=False)
run('flush,want', outputs=want)
run('flush,all,sync', sync_each=True)
run('flush,all', n=6)
