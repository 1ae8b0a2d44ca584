"""Benchmark: solved instances/s of the batched Dinkelbach/SCA-Lagrangian EE
solver (BASELINE.json metric) on N B200s, one process per GPU.

    python bench.py [--gpus N --steps K --warmup W] [--config c1] [--impl b200|reference]

A step = one full solve (Dinkelbach outer loop, SCA rounds, sweeps, repair,
feasibility, binaries) of one batch of independent channel realisations.
Weak scaling: every rank solves its own batch of distinct draws (draw index
rank*B + i), no collective on the data path; timing is max over ranks.

`value` is device-timed with inputs resident in HBM; `e2e` goes through the
public API (`solve_batch`) from host numpy gamma with the H2D copy of inputs
and the D2H copy of the allocation + scalars inside the timed region.  The
CPU baseline is the oracle port (oracle/hcran_oracle.py, the numpy
restatement of the reference) on the host cores, bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1803_07772_b200.scenarios import WORKLOADS, workload_batch  # noqa: E402
from paper_1803_07772_b200.shard import max_over_ranks, weak_range  # noqa: E402

METRIC = "solved instances/sec (RxNxK, batch)"
UNIT = "instances/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c0", "c1", "c2", "c3", "c4"])
    ap.add_argument("--batch", type=int, default=None, help="instances per GPU (default: config's)")
    ap.add_argument("--cpu-sample", type=int, default=None,
                    help="instances in the bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-only", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2,
                    help="steps of the end-to-end leg (at most --steps; c2 steps take ~1 min)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_desc(name, batch):
    m_f, k, ks, n, bw, _ = WORKLOADS[name]
    desc = {"workload": f"{name}: BASELINE.json configs[{name[1]}]",
            "rrh": m_f + 1, "users": k, "subcarriers": n, "batch_per_gpu": batch,
            "seed": 1, "draws": "rank*batch + i",
            "builder_pinned": {"bandwidth_hz": bw, "streaming_users": ks},
            "l2": "flushed between timed steps (256 MiB write)"}
    if name == "c4":
        desc["builder_pinned"]["streaming_users"] = "0/1 (30%)"
        desc["mode"] = "fixed-e inner solve"
    if name == "c3":
        desc["workload"] = "c3: BASELINE.json configs[3], one wave per GPU"
        desc["inputs"] = ("device-synthesised (hcran_b200_synth_gamma: Philox4x32-10 per draw, "
                          "the reference's distributions); draws rank*batch + i")
        desc["full_config_batch"] = 131072
    return desc


# ---------------------------------------------------------------- CPU side
def _oracle_one(args):
    name, draw = args
    from oracle import hcran_oracle as O
    from paper_1803_07772_b200.scenarios import workload_instance
    cfg, ch, e = workload_instance(name, draw)
    P = O.Prob.from_config(cfg, ch)
    try:
        if e is not None:
            O.solve_fixed_e(P, e)
        else:
            O.dinkelbach(P)
    except (O.Infeasible, O.ProductsActive):
        pass
    return draw


def cpu_rate(name, sample, first_draw=0):
    """Oracle port over `sample` draws on all host cores; returns (inst/s, cores, wall)."""
    from concurrent.futures import ProcessPoolExecutor
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("MKL_NUM_THREADS", "1")
    cores = os.cpu_count() or 1
    tasks = [(name, first_draw + i) for i in range(sample)]
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=min(cores, sample)) as pool:
        list(pool.map(_oracle_one, tasks, chunksize=1))
    wall = time.perf_counter() - t0
    return sample / wall, min(cores, sample), wall


DEFAULT_CPU_SAMPLE = {"c0": 256, "c1": 64, "c2": 16, "c3": 0, "c4": 1024}
# config[3] (131,072 instances over 2/4/8 GPUs, ~4 MiB of gains each) is
# benchmarked on a per-GPU wave of device-synthesised instances (hcran_b200_synth_gamma)
C3_BATCH = 296


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank, world):
    if rank != 0:
        return
    name = args.config
    if name == "c3":
        print(json.dumps({"impl": "reference", "metric": METRIC, "unit": UNIT,
                          "unavailable": "config[3] does not run on the CPU path: the reference "
                                         "allocates dense (M,M,K,N,N) float64 arrays of 16 GiB per "
                                         "instance (scale.py:696) -- MemoryError (SURVEY.md 6)"}),
              flush=True)
        return
    sample = args.cpu_sample or DEFAULT_CPU_SAMPLE[name]
    # a config[2] draw takes ~1 min on one core: one pass over a fixed sample
    # bounds the arm to a few minutes; lighter configs time `steps` samples
    passes = 1 if name == "c2" else args.steps
    if name != "c2":
        for _ in range(args.warmup if args.warmup < 1 else 1):
            cpu_rate(name, min(sample, os.cpu_count() or 1), first_draw=10_000)
    rates, walls = [], []
    for s in range(passes):
        r, cores, w = cpu_rate(name, sample, first_draw=s * sample)
        rates.append(r)
        walls.append(w)
    total = sum(walls)
    value = passes * sample / total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": passes, "warmup": 0 if name == "c2" else args.warmup,
            "ms_per_step": 1e3 * total / passes,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference instance generator, seed 1)",
            "config": workload_desc(name, args.batch or WORKLOADS[name][5]), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{sample} draws of {name} x {passes} pass(es), oracle/hcran_oracle.py "
                                       f"(numpy restatement of the reference) in a "
                                       f"{cores}-process pool on {cpu_model()}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU side
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) < 8:
                continue
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_peaks():
    """Pipe peaks: MEASURED_PEAKS.json has HBM/bf16 only, so the FP64 peak is our
    own microbenchmark (tools/peaks.cu, committed under profiles/) when present."""
    for path in (os.path.join(ROOT, "profiles", "peaks_b200.json"),):
        if os.path.exists(path):
            with open(path) as f:
                d = json.load(f)
            return float(d["fp64_fma_tflops"]), f"measured (tools/peaks.cu, {os.path.relpath(path, ROOT)})"
    return 37.2, "fallback: nominal 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz"


def load_fp32_peak():
    path = os.path.join(ROOT, "profiles", "peaks_b200.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f)["fp32_fma_tflops"])
    return 74.4


def load_traffic(name, batch):
    """DRAM bytes (read + write) of the solve kernel for this workload and batch
    from one `ncu --set full` capture (profiles/ncu_traffic.json), else None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f).get(f"{name}:{batch}")
    return None if d is None else float(d["dram_bytes_per_launch"])


def run_b200(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_1803_07772_b200 import DeviceProblem, solve_batch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    name = args.config
    B = args.batch or (C3_BATCH if name == "c3" else WORKLOADS[name][5])
    fixed = name == "c4"
    if name == "c3":  # gains synthesised on the device; one host copy for the e2e leg
        from paper_1803_07772_b200 import synth_gamma
        from paper_1803_07772_b200.scenarios import gen_sigma, workload_instance
        cfg, _, _ = workload_instance("c3", 0)
        g = synth_gamma(cfg, rank * B, B, seed=1, device=dev)
        K = cfg.n_users
        h_in = {"gamma": g.cpu().pin_memory(),
                "elastic": torch.from_numpy(np.ascontiguousarray(
                    np.broadcast_to(cfg.elastic_mask(), (B, K)), np.uint8)).pin_memory(),
                "min_rates": torch.from_numpy(np.ascontiguousarray(
                    np.broadcast_to(cfg.min_rates(), (B, K)))).pin_memory()}
        sigma = gen_sigma(cfg)
    else:
        batch = workload_batch(name, weak_range(rank, B))
        cfg = batch.cfg
        sigma = batch.sigma
        # per-instance inputs, pinned on the host (the e2e leg copies them every step)
        h_in = {"gamma": torch.from_numpy(batch.gamma).pin_memory(),
                "elastic": torch.from_numpy(np.ascontiguousarray(batch.elastic, np.uint8)).pin_memory(),
                "min_rates": torch.from_numpy(np.ascontiguousarray(batch.min_rates)).pin_memory()}
        if fixed:
            h_in["e_fixed"] = torch.from_numpy(np.ascontiguousarray(batch.e_fixed)).pin_memory()
    d_in = {k: v.to(dev) for k, v in h_in.items()}
    # config[3]: the seated SIC family without floor-tie re-solves (HCRAN_SIC_SEATED_FAST):
    # the exact dense pair family costs 8,128 pairs per (RRH, subcarrier) there
    # (minutes per flagged instance); flagged instances are counted in the line
    exact = "fast" if name == "c3" else False
    problem = DeviceProblem(cfg, sigma, dev, exact=exact)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    cpu_proc = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and name != "c3":
        cmd = [sys.executable, os.path.abspath(__file__), "--cpu-only", "--config", name]
        if args.cpu_sample:
            cmd += ["--cpu-sample", str(args.cpu_sample)]
        cpu_proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

    def step(x, outputs=None):
        kw = dict(mode="fixed_e", e_fixed=x["e_fixed"]) if fixed else {}
        return solve_batch(cfg, x["gamma"], None, x["elastic"], x["min_rates"], problem=problem,
                           sync=False, outputs=outputs, **kw)

    for _ in range(args.warmup):
        out = step(d_in)
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches = 0
    work = 0.0
    works = []  # per-step work counters only: a step's full outputs (~7 GB at c2 / 16,384)
    out = None  # are released when the next step replaces them (stream-ordered reuse)
    for s in range(args.steps):
        flush.random_(0, 255)  # L2 flush between timed steps (outside the events)
        ev[s][0].record(stream)
        out = step(d_in)
        ev[s][1].record(stream)
        launches += out["launches"]
        works.append(out["work"])
    barrier()
    clocks = sampler.stop()
    ms = [a.elapsed_time(b) for a, b in ev]
    t_dev = sum(ms) / 1e3
    for w in works:
        work += float(w.sum().item())
    sweeps = float(out["sweeps"].double().mean().item())
    st = out["status"].cpu().numpy()
    t_all = max_over_ranks(t_dev, dev)
    solved = B - int((st == 4).sum())  # HCRAN_ST_UNSUPPORTED instances do not count as solved
    value = world * solved * args.steps / t_all

    # end-to-end through the public API: host gamma (pinned) in, allocation +
    # per-instance scalars out (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        want = ["p", "rho", "a", "ee", "sum_rate", "total_power", "status", "outer_iters"]
        o = step(d_in, outputs=want)  # shapes for the pinned result buffers (untimed)
        host_out = {k: torch.empty(o[k].shape, dtype=o[k].dtype, pin_memory=True) for k in want}
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        e2e_steps = max(1, min(args.e2e_steps, args.steps))
        t0.record(stream)
        d2h = 0
        for s in range(e2e_steps):
            o = step(h_in, outputs=want)
            d2h = 0
            for k in want:
                v = o[k]
                host_out[k].copy_(v, non_blocking=True)
                d2h += v.numel() * v.element_size()
        t1.record(stream)
        barrier()
        h2d = sum(v.numel() * v.element_size() for v in h_in.values())
        te = max_over_ranks(t0.elapsed_time(t1) / 1e3, dev)
        e2e = {"value": world * solved * e2e_steps / te, "unit": UNIT, "steps": e2e_steps,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    if rank == 0:
        peak, peak_src = load_peaks()
        fp32_peak = load_fp32_peak()
        achieved = work / t_dev / 1e12  # rank 0's own launches and time
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (reference instance generator: users in a 500 m disc, "
                        "Rayleigh x d^-3 gains, seed 1)",
                "config": workload_desc(name, B),
                "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak,
                             "unit": "TFLOP/s", "frac": achieved / peak,
                             "traffic": load_traffic(name, B), "traffic_unit": "DRAM bytes per launch",
                             "peak_source": peak_src,
                             "note": "algorithmic FP64 flop-equivalents counted by the kernel "
                                     "(DESIGN.md work model) / device time of the solve"},
                "roofline_fp32_sfu": {"achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                                      "frac": achieved / fp32_peak,
                                      "note": "north_star framing: the same work as if it ran on "
                                              "the FP32 pipe (measured FFMA peak); the parity-"
                                              "critical core is FP64 (DESIGN.md)"},
                "sic_mode": ("seated, floor ties flagged not re-solved (HCRAN_SIC_SEATED_FAST)"
                             if name == "c3" else
                             "seated+dense-retry (HCRAN_SIC_SEATED, exact on all golden draws)"),
                "gpu_launches": launches, "clocks": clocks, "e2e": e2e,
                "solver": {"mean_sweeps_per_instance": sweeps,
                           "status_counts": {str(k): int(v) for k, v in
                                             zip(*np.unique(st, return_counts=True))},
                           "unsupported": int((st == 4).sum()),
                           "floor_tie_flagged": int((out["flags"].cpu().numpy() & 1).sum()),
                           "note": "status 0 converged, 1 outer-iteration cap, 2 stalled, 3 "
                                   "infeasible (the reference raises): all solved outcomes; "
                                   "4 = device capacity exceeded (counted in value only if "
                                   "'unsupported' > 0)"}}
        if name == "c3":
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                                    "sample": "not runnable: the reference allocates dense "
                                              "(M,M,K,N,N) float64 arrays of 16 GiB per instance "
                                              "(scale.py:696, SURVEY.md 6) -- MemoryError"}
        elif cpu_proc is not None:
            out, _ = cpu_proc.communicate()
            line["cpu_baseline"] = json.loads(out.strip().splitlines()[-1])
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_only(args):
    """The cpu_baseline leg as its own process, started by the GPU arm before
    its warm-up so the host sample overlaps the device timing."""
    name = args.config
    sample = args.cpu_sample or DEFAULT_CPU_SAMPLE[name]
    r, cores, wall = cpu_rate(name, sample)
    print(json.dumps({"value": r, "unit": UNIT, "cores": cores, "kind": "port",
                      "sample": f"{sample} draws of {name} ({wall:.1f} s), oracle/hcran_oracle.py "
                                f"in a {cores}-process pool on {cpu_model()}, run concurrently "
                                f"with the device timing"}), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.cpu_only:
        cpu_only(args)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_b200(args, rank, world, local)


if __name__ == "__main__":
    main()
