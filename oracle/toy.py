"""Toy model of config 1: least-squares linear regression, no bias
(TEST INFRASTRUCTURE — see oracle/__init__.py).

    f(w; X, y) = ||X w - y||^2 / (2 b),   grad = X^T (X w - y) / b

(the minibatch estimator G(x_t) of App. P:273, for a linear model).
"""
from __future__ import annotations

import numpy as np


def loss(w: np.ndarray, X: np.ndarray, y: np.ndarray) -> float:
    X = np.asarray(X, dtype=np.float64)
    r = X @ np.asarray(w, dtype=np.float64) - np.asarray(y, dtype=np.float64)
    return float(r @ r) / (2.0 * X.shape[0])


def grad(w: np.ndarray, X: np.ndarray, y: np.ndarray) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    r = X @ np.asarray(w, dtype=np.float64) - np.asarray(y, dtype=np.float64)
    return X.T @ r / X.shape[0]
