"""Time the CPU oracle as it stands (TEST INFRASTRUCTURE — see oracle/__init__.py).

Used only by bench.py's ``cpu_baseline`` leg and its ``--impl reference`` arm.
The oracle is not tuned for this: it runs oracle.daso_sim.simulate unchanged,
numpy fp64, thread pools pinned to one core, on the sync-path microbench
workload (config 2: fixed synthetic gradient per rank, B/S schedule) over a
bounded sample of the parameter vector.
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import daso_sim
from .schedule import SchedConfig


def _pin_one_core():
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(k, "1")
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(1)
    except Exception:
        return None


def time_sync_path(P: int, G: int, B: int, S: int, n_sample: int, steps: int, warmup: int = 0,
                   lr: float = 0.1, mu: float = 0.9, wd: float = 1e-4, wire: str = "bf16",
                   x0: np.ndarray | None = None, grads: list | None = None) -> dict:
    """Seconds per simulated DASO batch (all P*G ranks) on n_sample parameters."""
    import synthetic
    _lim = _pin_one_core()
    W = P * G
    x0 = synthetic.microbench_x0(n_sample) if x0 is None else x0
    grads = [synthetic.microbench_grad(n_sample, r, 0) for r in range(W)] if grads is None else grads
    cfg = SchedConfig(B_init=B, S_init=S, total_epochs=1, steps_per_epoch=B * 4096)
    if warmup:
        daso_sim.simulate(P, G, cfg, warmup, x0, lambda r, k, w: grads[r], lr, mu, wd, wire=wire)
    t0 = time.perf_counter()
    daso_sim.simulate(P, G, cfg, steps, x0, lambda r, k, w: grads[r], lr, mu, wd, wire=wire)
    dt = time.perf_counter() - t0
    return {"seconds": dt, "steps": steps, "s_per_step": dt / steps, "n": n_sample, "ranks": W, "cores": 1}


def calibrated(P: int, G: int, B: int, S: int, n_sample: int, budget_s: float = 12.0, wire: str = "bf16") -> dict:
    """Pick a step count that fills about ``budget_s`` seconds of oracle work."""
    import synthetic
    x0 = synthetic.microbench_x0(n_sample)
    grads = [synthetic.microbench_grad(n_sample, r, 0) for r in range(P * G)]
    probe = time_sync_path(P, G, B, S, n_sample, 1, x0=x0, grads=grads, wire=wire)
    steps = int(max(2, min(2000, budget_s / max(probe["s_per_step"], 1e-6))))
    return time_sync_path(P, G, B, S, n_sample, steps, x0=x0, grads=grads, wire=wire)
