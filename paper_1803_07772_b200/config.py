"""Config and CSV plumbing of the reference front end, with a backend switch
(reference `cli.py:35-151, 199-240`).

* `load_config(path)` -- YAML key-value file -> (NetworkConfig, Scenario):
  every key optional with the experiment defaults, unknown keys (and unknown
  `tolerances` keys) rejected by name (cli.py:35-97).
* `header_lines(tag, payload)` -- the CSV comment block: config hash (sha256
  of the sorted-key JSON, first 16 hex digits), git revision, config
  (cli.py:108-112).  Identical (config, seed) runs give identical bytes.
* `sweep_lines(scenario, rows)` -- the `sweep` CSV body (cli.py:222-236).
* `python -m paper_1803_07772_b200.config sweep --config X --backend b200`
  -- the `sweep` subcommand on the B200 path (`sweep.run_sweep`: one device
  launch per sweep value); `--backend reference` runs the reference
  package's own `run_sweep` when it is importable.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import subprocess
from dataclasses import asdict, replace
from pathlib import Path

import numpy as np

from .model import ConfigError, NetworkConfig, Tolerances
from .scenarios import build_config
from .sweep import Scenario, SweepRow, run_sweep

NETWORK_KEYS = {"architecture", "m_f", "n_subcarriers", "bandwidth_hz", "noise_dbm_hz",
                "l_max", "mask_dbm"}
TRAFFIC_KEYS = {"arrival_rate", "queue_packets", "packet_bits"}
SCENARIO_KEYS = {"sweep", "values", "users", "streaming_users", "draws", "seed", "solver",
                 "workers", "oma"}
TOLERANCE_KEYS = {"xi", "varpi1_rel", "varpi2_rel", "s_max", "v_max", "outer_max", "rho1",
                  "rho2"}


def parse_config(raw) -> tuple[NetworkConfig, Scenario]:
    """A parsed YAML mapping -> (network with defaults applied, scenario)."""
    raw = raw or {}
    if not isinstance(raw, dict):
        raise ConfigError("config root must be a mapping")
    known = NETWORK_KEYS | TRAFFIC_KEYS | SCENARIO_KEYS | {"tolerances"}
    bad = [k for k in raw if k not in known]
    if bad:
        raise ConfigError(f"unknown config key {bad[0]!r}")
    tol_raw = raw.get("tolerances") or {}
    bad = [k for k in tol_raw if k not in TOLERANCE_KEYS]
    if bad:
        raise ConfigError(f"unknown tolerances key {bad[0]!r}")
    l_max = 1 if raw.get("oma") else int(raw.get("l_max", 3))
    users = raw.get("users", 12)
    scenario = Scenario(
        architecture=raw.get("architecture", "hcran"), sweep=raw.get("sweep", "none"),
        values=tuple(raw.get("values", (users,))), k_total=int(users),
        k_streaming=int(raw.get("streaming_users", 6)),
        arrival_rate=float(raw.get("arrival_rate", 125.0)), l_max=l_max,
        n_subcarriers=int(raw.get("n_subcarriers", 32)),
        bandwidth_hz=float(raw.get("bandwidth_hz", 1.0e6)), draws=int(raw.get("draws", 50)),
        seed=int(raw.get("seed", 1)), solver=raw.get("solver", "scale"),
        workers=int(raw.get("workers", 1)))
    cfg = build_config(
        architecture=scenario.architecture, k_total=scenario.k_total,
        k_streaming=scenario.k_streaming, rng=np.random.default_rng([scenario.seed, 0]),
        arrival_rate=scenario.arrival_rate, queue_packets=float(raw.get("queue_packets", 25.0)),
        packet_bits=float(raw.get("packet_bits", 1024.0)), l_max=scenario.l_max,
        n_subcarriers=scenario.n_subcarriers, bandwidth_hz=scenario.bandwidth_hz,
        m_f=raw.get("m_f"), noise_dbm_hz=float(raw.get("noise_dbm_hz", -174.0)),
        tolerances=Tolerances(**tol_raw), mask_dbm=raw.get("mask_dbm"))
    return cfg, scenario


def load_config(path: str | Path | None) -> tuple[NetworkConfig, Scenario]:
    """A YAML config file (or None: every default) -> (network, scenario)."""
    import yaml
    raw = {} if path is None else (yaml.safe_load(Path(path).read_text()) or {})
    return parse_config(raw)


def git_revision() -> str:
    try:
        r = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True,
                           text=True, timeout=5, cwd=Path(__file__).parent)
        return r.stdout.strip() or "unknown"
    except Exception:
        return "unknown"


def config_hash(payload: dict) -> str:
    blob = json.dumps(payload, sort_keys=True, default=str)
    return hashlib.sha256(blob.encode()).hexdigest()[:16]


def header_lines(tag: str, payload: dict, git_rev: str | None = None) -> list[str]:
    blob = json.dumps(payload, sort_keys=True, default=str)
    return [f"# {tag}", f"# config_hash: {config_hash(payload)}",
            f"# git_rev: {git_revision() if git_rev is None else git_rev}", f"# config: {blob}"]


def sweep_lines(scenario: Scenario, rows: list[SweepRow], git_rev: str | None = None) -> list[str]:
    lines = header_lines("sweep", asdict(scenario), git_rev)
    cols = "value,mean_ee,mean_rate,mean_power,mean_iterations,n_feasible,n_draws"
    if scenario.include_timing:
        cols += ",mean_wall_s"
    lines.append(cols)
    for r in rows:
        row = (f"{r.value:.10g},{r.mean_ee:.10g},{r.mean_rate:.10g},{r.mean_power:.10g},"
               f"{r.mean_iterations:.10g},{r.n_feasible},{r.n_draws}")
        if scenario.include_timing:
            row += f",{r.mean_wall_s:.4f}"
        lines.append(row)
    return lines


def _reference_run_sweep(scenario: Scenario):
    try:
        from hcran_noma import scenarios as ref
    except ImportError as exc:
        raise SystemExit(f"--backend reference needs the hcran_noma package: {exc}")
    return ref.run_sweep(ref.Scenario(**asdict(scenario)))


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1803_07772_b200.config")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sw = sub.add_parser("sweep", help="figure sweep -> CSV (cli.py:199-240)")
    sw.add_argument("--config")
    sw.add_argument("--backend", choices=["b200", "reference"], default="b200")
    sw.add_argument("--arch")
    sw.add_argument("--sweep")
    sw.add_argument("--values")
    sw.add_argument("--draws", type=int)
    sw.add_argument("--seed", type=int)
    sw.add_argument("--oma", action="store_true")
    sw.add_argument("--timing", action="store_true")
    sw.add_argument("--out")
    args = ap.parse_args(argv)
    _, scenario = load_config(args.config)
    over = {}
    if args.arch:
        over["architecture"] = args.arch
    if args.sweep:
        over["sweep"] = args.sweep
    if args.values:
        over["values"] = tuple(float(v) if "." in v else int(v) for v in args.values.split(","))
    if args.draws is not None:
        over["draws"] = args.draws
    if args.seed is not None:
        over["seed"] = args.seed
    if args.oma:
        over["l_max"] = 1
    if args.timing:
        over["include_timing"] = True
    scenario = replace(scenario, **over)
    rows = run_sweep(scenario) if args.backend == "b200" else _reference_run_sweep(scenario)
    out = Path(args.out or "sweep.csv")
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text("\n".join(sweep_lines(scenario, rows)) + "\n")
    print(f"wrote {out}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
