"""Appendix verification report (App. Eq. 5-6; readings R6, R21).

Records every rank's gradients along an independent plain-SGD trajectory (the local
phase between send and merge is plain SGD with mu = wd = 0 and G = 1), then checks the
oracle's state-form simulation against the gradient forms:
  * Eq. 5 with the local sum over k = 0..S holds to 1e-13 (reading A);
  * the one-step effective gradient derived from it reproduces the merge step exactly;
  * App. Eq. 6 as printed does NOT reproduce it except in the special case S = 1, P = 2
    (its coefficients P and 2S are swapped and its local-sum range is shifted by one:
    reading R21) — the test pins which cases agree so a change of reading is visible.
"""
import numpy as np
import pytest

import synthetic
from oracle import appendix, daso_sim, toy
from oracle.schedule import SchedConfig

D, BATCH = 48, 8


def grads_along_local_sgd(x0, eta, steps, rank):
    w, gs = x0.copy(), []
    for k in range(steps):
        X, y = synthetic.toy_batch(D, BATCH, rank, k)
        X = X.astype(np.float64)
        g = X.T @ (X @ w - y.astype(np.float64)) / BATCH
        gs.append(g)
        w = w - eta * g
    return gs


@pytest.mark.parametrize("S,B,P", [(1, 4, 2), (2, 2, 3), (3, 4, 2), (2, 8, 4)])
def test_appendix_gradient_forms(S, B, P):
    eta = 0.03
    x0 = synthetic.microbench_x0(D, seed=13).astype(np.float64)
    cfg = SchedConfig(B_init=B, S_init=S, total_epochs=1, steps_per_epoch=8 * B)
    out = daso_sim.simulate(P, 1, cfg, S + 1, x0, lambda r, k, w: toy.grad(w, *synthetic.toy_batch(D, BATCH, r, k)),
                            eta, 0.0, 0.0, wire="fp32", trace=True)
    alpha = eta / (2 * S + P)
    for l in range(P):
        gl = grads_along_local_sgd(x0, eta, S + 1, l)
        snaps = [grads_along_local_sgd(x0, eta, 1, i)[0] for i in range(P)]
        x_merge = out["trace"][S][l]
        np.testing.assert_allclose(x_merge, appendix.eq5_reading_a(x0, gl, snaps, eta, S, P), rtol=0, atol=1e-13)
        # the batch before the merge is plain local SGD from x0 (App. Eq. 2)
        x_before = x0 - eta * np.sum(gl[:S], axis=0)
        geff = appendix.effective_gradient(gl, snaps, S, P)
        np.testing.assert_allclose(x_merge, x_before - alpha * geff, rtol=0, atol=1e-13)
        g6 = appendix.eq6_as_printed(gl, snaps, S, P)
        rel = np.linalg.norm(g6 - geff) / np.linalg.norm(geff)
        if S == 1 and P == 2:
            # the printed form swaps the roles of P and 2S and shifts the local-sum range by one;
            # with S = 1 and P = 2S both garbles cancel and Eq. 6 happens to be exact
            assert rel < 1e-12
        else:
            assert rel > 0.1, "App. Eq. 6 as printed unexpectedly matches (reading R21 would be moot)"
