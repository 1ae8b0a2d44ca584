"""Makespan of the persistent-CTA queue for a per-instance cost vector:
    python tools/sched_sim.py gpurun_out/work_c1.npz [slots]"""
import heapq, sys, numpy as np
d = np.load(sys.argv[1]); w = d['work'].astype(float)
slots = int(sys.argv[2]) if len(sys.argv) > 2 else 148
def makespan(order, S):
    h = [0.0] * S
    for i in order:
        t = heapq.heappop(h); heapq.heappush(h, t + w[i])
    return max(h)
ideal = w.sum() / slots
for tag, order in [('fifo', range(len(w))), ('lpt', np.argsort(-w))]:
    m = makespan(order, slots)
    print(f'{tag}: makespan/ideal {m / ideal:.3f}  (max single {w.max() / ideal:.3f})')
