"""Expected outputs of the B200 default path (HCRAN_SIC_SEATED) computed by the
ORACLE's independent restatement of that model (`oracle.dinkelbach(...,
sic="device")`: seated-pair SIC multipliers + dense re-solve of floor ties),
for every golden instance.  Instances where this model and the reference
disagree are the "floor-sensitive" set: the reference decides a
seat there from floor-level multipliers of unseated pairs.

    python tests/golden/make_device_model.py c0_0_128 c1_0_24 ...
"""

import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def one(args):
    name, draw = args
    from oracle import hcran_oracle as O
    from paper_1803_07772_b200.scenarios import workload_instance
    cfg, ch, e = workload_instance(name, int(draw))
    P = O.Prob.from_config(cfg, ch)
    if name == "c4":
        r = O.solve_fixed_e(P, e, sic="seated")
        if r.stats.floor_tie:
            r = O.solve_fixed_e(P, e, sic="dense")
        if r.status != "ok":
            return dict(status=3, p=r.p, rho=np.zeros(r.p.shape, np.uint8),
                        a=np.zeros(r.p.shape[:2], np.uint8), ee=np.nan, tp=np.nan, obj=np.nan)
        rr, pw, ee = O.report(P, r.p)
        return dict(status=0, p=r.p, rho=r.rho, a=r.a, ee=ee, tp=pw, obj=rr - e * pw)
    try:
        tr = O.dinkelbach(P, sic="device")
    except O.Infeasible:
        z = np.zeros(P.shape)
        return dict(status=3, p=z, rho=z.astype(np.uint8), a=np.zeros(P.shape[:2], np.uint8),
                    ee=np.nan, tp=np.nan, obj=np.nan)
    rr, pw, ee = O.report(P, tr.p)
    st = {"converged": 0, "cap": 1, "stalled": 2}[tr.status]
    return dict(status=st, p=tr.p, rho=tr.rho, a=tr.a, ee=ee, tp=pw, obj=np.nan)


def main(names):
    for fn in names:
        g = np.load(os.path.join(HERE, fn + ".npz"))
        name = str(g["config"])
        with ProcessPoolExecutor(max_workers=max(1, (os.cpu_count() or 2) - 1)) as pool:
            res = list(pool.map(one, [(name, d) for d in g["draw"]], chunksize=1))
        dm = {"draw": g["draw"],
              "status": np.array([r["status"] for r in res], np.int8),
              "ee": np.array([r["ee"] for r in res]),
              "total_power": np.array([r["tp"] for r in res]),
              "objective": np.array([r["obj"] for r in res]),
              "rho": np.stack([r["rho"] for r in res]).astype(np.uint8),
              "a": np.stack([r["a"] for r in res]).astype(np.uint8)}

        def rel(a, b):
            return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
        key = "objective" if name == "c4" else "ee"
        same = (rel(dm[key], g[key]) <= 1e-4) & (dm["status"] == g["status"])
        same &= np.array([np.array_equal(dm["rho"][i], g["rho"][i]) and
                          np.array_equal(dm["a"][i], g["a"][i]) for i in range(len(res))])
        if name != "c4":
            same &= rel(dm["total_power"], g["total_power"]) <= 1e-4
        dm["floor_sensitive"] = ~same
        out = os.path.join(HERE, fn + "_devmodel.npz")
        np.savez_compressed(out, **dm)
        print(fn, "floor-sensitive:", np.nonzero(~same)[0].tolist(), "of", len(res), file=sys.stderr)


if __name__ == "__main__":
    main(sys.argv[1:])
