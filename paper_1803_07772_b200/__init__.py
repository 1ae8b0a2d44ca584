"""B200-native batched energy-efficiency solver for PD-NOMA H-CRANs
(arXiv 1803.07772): Dinkelbach -> SCALE rounds -> Lagrangian power sweeps ->
repair/selection, every instance solved on the GPU by one CTA.

Drop-in names of the reference package `hcran_noma` for this hot path
(/root/reference/pkg/src/hcran_noma/__init__.py:7-34): types (model.py),
the traffic transform, instance construction (scenarios.py), `ScaleSolver`,
`solve`, `InfeasibleProblemError`, `DinkelbachTrace`; plus `solve_batch` for
whole batches.  The compute path is libhcran_b200.so (sm_100a) only.
"""

from .model import (ChannelState, ConfigError, EnergyReport, NetworkConfig,
                    PowerAllocation, Tolerances, UserSpec)
from .traffic import TrafficSpec, delay_roots, max_delay_from_queue, min_rate_for_delay
from .scenarios import build_config, gen_channel, tiny_instance, workload_batch
from .solver import (B200Unavailable, DeviceProblem, DinkelbachTrace, InfeasibleProblemError,
                     InnerResult, ScaleSolver, SolveStats, energy_report, solve, solve_batch)
from .synth import synth_gamma

__all__ = [
    "ChannelState", "ConfigError", "EnergyReport", "NetworkConfig", "PowerAllocation",
    "Tolerances", "UserSpec", "TrafficSpec", "delay_roots", "max_delay_from_queue",
    "min_rate_for_delay", "build_config", "gen_channel", "tiny_instance", "workload_batch",
    "B200Unavailable", "DeviceProblem", "DinkelbachTrace", "InfeasibleProblemError", "InnerResult",
    "ScaleSolver", "SolveStats", "energy_report", "solve", "solve_batch", "synth_gamma",
]

__version__ = "0.1.0"
