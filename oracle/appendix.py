"""The appendix's gradient form of DASO's global synchronisation, as a verification report
(TEST INFRASTRUCTURE — see oracle/__init__.py).

App. P:294-327 rewrite Eq. (1) in terms of gradients (momentum 0, weight decay 0, one GPU per
node so the local average is the GPU's own gradient):

  Eq. 5  x_{t+S} = x_t - alpha (2S sum_{k=0}^{S-1} G_l(x_{l:t+k}) + sum_i G_p(x^i_{p:t})),
                     alpha = eta / (2S + P)
  Eq. 6  G^DASO(x_{t+S-1}) = P sum_{beta=0}^{S-1} G_l(x_{l:t+S-beta})
                                         - 2S G_l(x_{l:t+S-1}) + sum_i G_p(x^i_{p:t})

This module evaluates both from the gradients recorded along a simulated trajectory and
reports how they compare with the state-form simulation (oracle.daso_sim):
  * under reading R6 (A) — snapshots after batch t's update, merge after batch t+S's — the
    state form equals Eq. 5 with the local sum running to S (k = 0..S), exactly;
  * the single-step "effective gradient" defined by x_{t+S} = x_{t+S-1} - alpha G_eff follows
    from Eq. 5 and App. Eq. 2:  G_eff = 2S G_l,S - P sum_{k=0}^{S-1} G_l,k + sum_i G_i,0
    (reading A indices); Eq. 6 as printed has the coefficients P and 2S swapped and the
    local-sum range shifted by one, so the two agree only for S = 1, P = 2 — the garble
    recorded as reading R21.
"""
from __future__ import annotations

import numpy as np


def eq5_reading_a(x0, local_grads, snap_grads, eta, S, P):
    """x_S by Eq. 5 with the local sum over k = 0..S (reading R6 (A))."""
    alpha = eta / (2 * S + P)
    return x0 - alpha * (2 * S * np.sum(local_grads[:S + 1], axis=0) + np.sum(snap_grads, axis=0))


def effective_gradient(local_grads, snap_grads, S, P):
    """G_eff with x_S = x_{S-1} - alpha * G_eff, derived from Eq. 5 (reading A) and App. Eq. 2."""
    return 2 * S * local_grads[S] - P * np.sum(local_grads[:S], axis=0) + np.sum(snap_grads, axis=0)


def eq6_as_printed(local_grads, snap_grads, S, P):
    """App. Eq. 6 literally, mapping G_l(x_{l:t+j}) to the gradient taken at local step j
    (the paper's x_{t+S} has no gradient of its own in the simulation; index S is the merge
    batch's gradient under reading A)."""
    first = P * np.sum([local_grads[S - b] for b in range(S)], axis=0)
    return first - 2 * S * local_grads[S - 1] + np.sum(snap_grads, axis=0)
