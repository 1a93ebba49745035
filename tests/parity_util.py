"""Shared checks of GPU trajectories against the CPU oracle (test infrastructure).

`check_trajectory` compares, for every rank and every step, the GPU parameters with
oracle.daso_sim run on the same seeded inputs:
  * ||gpu - oracle|| / ||oracle|| <= tol and elementwise |gpu - oracle| <= tol*(|x_o| + rms(x_o)),
    tol = 1e-5 (fp32 wire) / 1e-2 (bf16 wire) — the north star's bounds;
  * the schedule records bit-exact (every field);
  * node replicas bitwise identical (Fig. 4) where checksums / traces are given.
"""
from __future__ import annotations

import numpy as np

import synthetic
from oracle import daso_sim, toy
from oracle.schedule import SchedConfig


def toy_oracle(P, G, B, S, steps=20, d=1000, b=32, lr=0.01, mu=0.9, wd=1e-4, wire="bf16", warm=0, cool=0,
               epochs=1, spe=20, flags=""):
    cache = {}

    def grad_fn(r, k, w):
        if (r, k) not in cache:
            cache[(r, k)] = synthetic.toy_batch(d, b, r, k)
        return toy.grad(w, *cache[(r, k)])

    cfg = SchedConfig(B_init=B, S_init=S, warmup_epochs=warm, cooldown_epochs=cool, total_epochs=epochs,
                      steps_per_epoch=spe)
    return daso_sim.simulate(P, G, cfg, steps, np.zeros(d), grad_fn, lr, mu, wd, wire=wire,
                             epoch_flags=[int(c) for c in flags], trace=True)


def check_trajectory(traces, recs, ref, P, G, wire):
    """traces[r][k] = rank r's parameters after step k; recs[r][k] = its record dict."""
    tol = 1e-2 if wire == "bf16" else 1e-5
    worst = 0.0
    steps = len(ref["trace"])
    for r in range(P * G):
        for k in range(steps):
            got = np.asarray(traces[r][k], np.float64)
            xo = ref["trace"][k][r]
            rms = np.sqrt(np.mean(xo ** 2))
            err = np.abs(got - xo)
            assert np.all(err <= tol * (np.abs(xo) + rms)), (r, k, float(np.max(err / (np.abs(xo) + rms))))
            rel = np.linalg.norm(got - xo) / max(np.linalg.norm(xo), 1e-30)
            assert rel <= tol, (r, k, rel)
            worst = max(worst, rel)
            assert recs[r][k] == ref["records"][k].as_dict(), (r, k, recs[r][k], ref["records"][k].as_dict())
    for j in range(P):   # node replicas bitwise identical, every step
        for l in range(1, G):
            for k in range(steps):
                np.testing.assert_array_equal(np.asarray(traces[j * G + l][k]).view(np.uint32),
                                              np.asarray(traces[j * G][k]).view(np.uint32))
    return worst
