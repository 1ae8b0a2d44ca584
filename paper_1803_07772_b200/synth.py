"""Device-side instance synthesis (the loader of scenarios.py:84-153 on the GPU).

`synth_gamma` writes the channel gains of draws [first, first + B) straight
into a CUDA tensor through hcran_b200_synth_gamma: users uniform in the 500 m
disc, Exp(1) fading times d^-3 path loss, one Philox4x32-10 stream per
(seed, draw).  The network template (RRH positions, budgets, masks, user
classes) is the workload's; only the user drop and the fading vary per draw,
as in the reference.  Used for config[3], whose 131,072 instances (~4 MiB of
gains each) cannot be generated on the host; the numbers differ from the
reference's numpy streams (same distributions, pinned by a KS test).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from .solver import _torch, library

DISC_RADIUS_M = 500.0  # scenarios.py DISC_RADIUS_M
PATHLOSS_EXP = 3.0     # gen_channel: d ** -3


def synth_gamma(cfg, first_draw: int, B: int, seed: int = 1, device=None, out=None, stream=None):
    torch = _torch()
    lib = library()
    dev = torch.device(device or "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    M, K, N = cfg.n_rrh, cfg.n_users, cfg.n_subcarriers
    with torch.cuda.device(dev):
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.stream(s):
            xy = torch.as_tensor(np.ascontiguousarray(cfg.rrh_positions, np.float64)).to(dev)
            if out is None:
                out = torch.empty((B, M, K, N), dtype=torch.float64, device=dev)
            sp = _abi.Synth(M=M, K=K, N=N, rrh_xy=xy.data_ptr(), disc_radius=DISC_RADIUS_M,
                            pathloss_exp=PATHLOSS_EXP, seed=seed)
            rc = lib.hcran_b200_synth_gamma(C.byref(sp), int(first_draw), int(B), out.data_ptr(),
                                            s.cuda_stream)
            if rc:
                raise RuntimeError(f"hcran_b200_synth_gamma: {_abi.ERRORS.get(rc, rc)}")
            out._hcran_keep = xy  # keep the positions alive until the stream has run
    return out
