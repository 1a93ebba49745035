"""Flat-vector arithmetic of DASO (TEST INFRASTRUCTURE — see oracle/__init__.py).

All state is numpy float64.  Summations run in ascending rank order,
sequentially (reading R18), so results are reproducible bit for bit.
"""
from __future__ import annotations

import numpy as np


def average(vectors: list[np.ndarray]) -> np.ndarray:
    """Elementwise mean, ascending-index sequential sum.

    P:75 (Fig. 2): "The gradients from each GPU are averaged"; P:83 (Fig. 3):
    "The network parameters are averaged by each GPU in the group".
    """
    if len(vectors) == 0:
        raise ValueError("argument error: empty list")
    acc = np.zeros_like(np.asarray(vectors[0], dtype=np.float64))
    for v in vectors:
        v = np.asarray(v, dtype=np.float64)
        if v.shape != acc.shape:
            raise ValueError("shape error")
        acc = acc + v
    return acc / len(vectors)


def weighted_stale_average(local: np.ndarray, stale: list[np.ndarray], S: int) -> np.ndarray:
    """Eq. (1), P:89-92:

        x_{t+S} = ( 2S * x^l_{t+S-1} + sum_{i=1}^{P} x^i_t ) / (2S + P)

    ``local`` is this GPU's current parameters (after this batch's local update,
    reading R7), ``stale`` the P parameter snapshots received from the group
    members — including this GPU's own snapshot (reading R2) — and P = len(stale)
    is the group size = number of nodes (reading R1).  Written exactly as the
    paper's formula (numerator, then division).
    """
    if S < 1:
        raise ValueError("argument error: S must be >= 1 (S = 0 is the plain average)")
    if len(stale) == 0:
        raise ValueError("argument error: empty stale list")
    P = len(stale)
    s = np.zeros_like(np.asarray(local, dtype=np.float64))
    for xi in stale:  # ascending node order
        s = s + np.asarray(xi, dtype=np.float64)
    return (2.0 * S * np.asarray(local, dtype=np.float64) + s) / (2.0 * S + P)


def to_fp32(x: np.ndarray) -> np.ndarray:
    """IEEE binary32 round-to-nearest-even (numpy's cast)."""
    return np.asarray(x, dtype=np.float64).astype(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 -> fp32 round trip, round-to-nearest-even on the 16 dropped
    mantissa bits (reading R18).

    P:86: "parameters are cast to a 16-bit datatype representation during buffer
    packaging ... Once received, the parameters are cast back to their original
    datatype"; "DASO compresses to brain floating point 16".
    The parameters' original datatype is fp32, so the oracle first forms the
    fp32 value and rounds that (bit-level, written out below).
    Finite inputs only (training has diverged otherwise).
    """
    f = to_fp32(x)
    if not np.all(np.isfinite(f)):
        raise ValueError("argument error: non-finite value in bf16 pack")
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)          # last kept mantissa bit
    u = (u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)  # RNE on the dropped 16 bits
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def wire(x: np.ndarray, kind: str) -> np.ndarray:
    """Value of x after travelling through the global network.

    kind "bf16": P:86 / P:162 buffer packaging in bf16 (the north-star default);
    kind "fp32": "Datatype casting is not beneficial in this scenario"
    (the paper-literal non-blocking wire, reading R3): the parameters travel in
    their original datatype, uncast — the identity on the oracle's state.
    """
    if kind == "bf16":
        return bf16_round(x)
    if kind == "fp32":
        return np.array(x, dtype=np.float64, copy=True)
    raise ValueError(f"unknown wire kind {kind!r}")
