"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the DASO method: it only draws random
numbers (and casts them to the fp32 input format both sides consume). Both
``oracle/`` and the GPU tests / bench import it; neither imports the other.

Recipes (DESIGN.md §"Input recipe"):

* toy DASO sim (config 1): linear regression, d params, per-rank batch b;
  X_{r,k} ~ N(0,1)^{b x d}, y = X w* + 0.1 eps, w* ~ N(0, 1/d).
  Generator for (rank r, step k): PCG64(SeedSequence([2104, r, k])).
* sync-path microbench (config 2): x0 ~ N(0, 0.02^2) (seed 0), identical on
  all ranks; g_{r,k} ~ N(0, 0.01^2) with SeedSequence([17, r, k]).
* plateau patterns (config 5): Bernoulli(p) per epoch, SeedSequence([7, tag]).
"""
from __future__ import annotations

import numpy as np

TOY_SEED = 2104
GRAD_SEED = 17
PLATEAU_SEED = 7


def _rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(key))))


def toy_wstar(d: int) -> np.ndarray:
    """w* ~ N(0, 1/d), fp32 (the ground-truth weights of the toy regression)."""
    return (_rng(TOY_SEED, 1 << 30).standard_normal(d) / np.sqrt(d)).astype(np.float32)


def toy_batch(d: int, b: int, rank: int, step: int) -> tuple[np.ndarray, np.ndarray]:
    """(X [b,d] fp32, y [b] fp32) for global rank ``rank`` at global step ``step``."""
    g = _rng(TOY_SEED, rank, step)
    X = g.standard_normal((b, d)).astype(np.float32)
    eps = g.standard_normal(b).astype(np.float32)
    wstar = toy_wstar(d)
    # y is an input, generated in fp64 from the fp32 draws then stored as fp32
    y = (X.astype(np.float64) @ wstar.astype(np.float64) + 0.1 * eps.astype(np.float64)).astype(np.float32)
    return X, y


def microbench_x0(n: int, seed: int = 0) -> np.ndarray:
    """Initial parameters x0 ~ N(0, 0.02^2), fp32, identical on every rank."""
    return (0.02 * _rng(seed).standard_normal(n)).astype(np.float32)


def microbench_grad(n: int, rank: int, step: int) -> np.ndarray:
    """Per-rank synthetic gradient g ~ N(0, 0.01^2), fp32."""
    return (0.01 * _rng(GRAD_SEED, rank, step).standard_normal(n)).astype(np.float32)


def plateau_pattern(epochs: int, p: float = 0.3, tag: int = 0) -> list[int]:
    """Per-epoch plateau flags (1 = the training loss plateaued at that epoch's end)."""
    u = _rng(PLATEAU_SEED, tag).random(epochs)
    return [int(v < p) for v in u]


def lr_constant(lr: float, steps: int) -> list[float]:
    return [float(lr)] * steps
