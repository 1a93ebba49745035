"""DASO per-batch step over all ranks of a virtual cluster
(TEST INFRASTRUCTURE — see oracle/__init__.py).

One process simulates W = P * G ranks (P nodes x G GPUs, rank = node*G + local).
For every global batch k, in this order (Fig. 2-5; readings R4-R12):

  1. every rank computes its gradient on its own data             (given)
  2. local synchronization: every GPU of node j gets the node mean of the
     gradients (Fig. 2: "gradients from each GPU are averaged, then each
     GPU's gradients are set to the result")                        [R4: fp32 sum x 1/G]
  3. local optimizer step on every rank (momentum SGD)
  4. schedule (oracle.schedule) decides: merge due? send?
  5. due merge (non-blocking case): each member m of the exchange group
     replaces its parameters by Eq. (1) with its own S_p, then broadcasts them to
     its node (Fig. 4: "sends its network parameters to all other
     node-local GPUs, which replace the old parameters")          [R6, R7, R8]
  6. send: the active group (rotating) snapshots its parameters through
     the wire format (P:86 bf16 packaging).  Blocking (warm-up / cool-down, or
     S = 0): the members average the snapshots right away (Fig. 3) and broadcast
     (Fig. 4).  Non-blocking: the snapshots are kept and merged S batches later.

P = 1: the global tier is disabled (R12).  G = 1: steps 2 and the broadcasts
are no-ops.  Momentum buffers are never communicated (R16); x0 is identical on
every rank and v0 = 0 (R17).
"""
from __future__ import annotations

from typing import Callable

import numpy as np

from . import numerics, sgd
from .schedule import SchedConfig, Schedule, plateau_arg
from .topology import check_cluster, rank_of


def simulate(P: int, G: int, cfg: SchedConfig, steps: int, x0: np.ndarray,
             grad_fn: Callable[[int, int, np.ndarray], np.ndarray],
             lr: float | Callable[[int], float], mu: float, wd: float,
             wire: str = "bf16", epoch_flags: list[int] | None = None,
             trace: bool = False) -> dict:
    """Run ``steps`` DASO batches; returns final per-rank x, v and the records.

    grad_fn(rank, step, x_rank) -> gradient of that rank's loss on its batch.
    lr: scalar or callable step -> lr (the host scalar passed to daso_step).
    trace=True also returns the per-step parameters of every rank.
    """
    check_cluster(P, G)
    W = P * G
    cfg = SchedConfig(**{**cfg.__dict__, "gpus_per_node": G})
    sched = Schedule(cfg)
    x = [np.array(x0, dtype=np.float64, copy=True) for _ in range(W)]
    v = [np.zeros_like(x[0]) for _ in range(W)]
    snap: list[np.ndarray] | None = None
    hist = []
    for k in range(steps):
        lr_k = lr(k) if callable(lr) else lr
        g = [np.asarray(grad_fn(r, k, x[r]), dtype=np.float64) for r in range(W)]
        # 2. local synchronization (node mean, ascending local id)
        for j in range(P):
            gbar = numerics.average([g[rank_of(j, l, G)] for l in range(G)])
            for l in range(G):
                g[rank_of(j, l, G)] = gbar
        # 3. local update
        for r in range(W):
            x[r], v[r] = sgd.sgd_step(x[r], v[r], g[r], lr_k, mu, wd)
        # 4. schedule
        rec = sched.next(plateau_arg(k, epoch_flags or [], cfg.steps_per_epoch))
        # 5. due merge, before any new send (R8)
        if rec.merge and P > 1:
            assert snap is not None
            for j in range(P):
                m = rank_of(j, rec.merge_group, G)
                x[m] = numerics.weighted_stale_average(x[m], snap, rec.merge_S)
                for l in range(G):
                    x[rank_of(j, l, G)] = x[m].copy()
            snap = None
        # 6. send
        if rec.send and P > 1:
            a = rec.send_group
            snaps = [numerics.wire(x[rank_of(i, a, G)], wire) for i in range(P)]
            if rec.blocking:
                avg = numerics.average(snaps)
                for j in range(P):
                    for l in range(G):
                        x[rank_of(j, l, G)] = avg.copy()
            else:
                snap = snaps
        if trace:
            hist.append([xi.copy() for xi in x])
    out = {"x": x, "v": v, "records": sched.records}
    if trace:
        out["trace"] = hist
    return out

