"""Node-local optimizer step (TEST INFRASTRUCTURE — see oracle/__init__.py).

App. Eq. 1: x_{t+1} = x_t - eta * G(x_t), extended with the local
optimizer the experiments use: "SGD with a momentum of 0.9 and weight
decay of 0.0001" (torch.optim.SGD semantics: dampening 0, no Nesterov):

    d = g + wd * x
    v = mu * v + d
    x = x - lr * v
"""
from __future__ import annotations

import numpy as np


def sgd_step(x: np.ndarray, v: np.ndarray, g: np.ndarray, lr: float, mu: float, wd: float
             ) -> tuple[np.ndarray, np.ndarray]:
    x = np.asarray(x, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    d = g + wd * x
    v_new = mu * v + d
    x_new = x - lr * v_new
    return x_new, v_new
