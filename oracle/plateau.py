"""Loss-plateau detector and learning-rate schedule (TEST INFRASTRUCTURE — see
oracle/__init__.py).

Paper:
  * P:162 "When the training loss plateaus, i.e. the training loss is not decreasing by
    more than a set percentage threshold, the scheduler decreases the learning rate by
    a set factor."
  * P:172 "learning rate warm-up phase of five epochs ... The maximum learning rate is
    scaled with the number of global processes. The learning rate decays by a factor of
    0.5 when the training cross entropy loss is stable for 5 epochs."
  * P:212 "decays the learning rate by a factor of 0.75 when the loss is judged to be
    stable for 5 epochs ... warm up phase of 5 epochs, in which the learning rate is
    slowly increased from 0.0 to 0.4"
  * P:99 "Each time the training loss plateaus, B and W are reduced ..."

Reading R20: one detector per run, evaluated on each epoch's mean
training loss.  An epoch "improves" iff loss < best - threshold * |best| (relative
threshold); otherwise it is a stable epoch.  The plateau fires when `patience`
consecutive epochs are stable; the stable count then restarts (the best loss is
kept).  The same events drive the LR decay and DASO's B/S halving.
LR: linear warm-up per step from 0 to peak over the warm-up epochs
(lr_k = peak * (k + 1) / warmup_steps), then peak * factor ** (plateaus so far);
peak = base_lr * world_size.
"""
from __future__ import annotations

import math


class PlateauDetector:
    def __init__(self, patience: int = 5, threshold: float = 0.01):
        if patience < 1 or threshold < 0:
            raise ValueError("config error: patience >= 1, threshold >= 0")
        self.patience = patience
        self.threshold = threshold
        self.best = math.inf
        self.stable = 0

    def update(self, loss: float) -> int:
        if not math.isfinite(loss):
            raise ValueError("divergence: non-finite loss")
        if self.best == math.inf or loss < self.best - self.threshold * abs(self.best):
            self.best = loss
            self.stable = 0
            return 0
        self.stable += 1
        if self.stable >= self.patience:
            self.stable = 0
            return 1
        return 0


def lr_at(step: int, steps_per_epoch: int, base_lr: float, world: int, warmup_epochs: int,
          factor: float, n_plateaus: int) -> float:
    peak = base_lr * world
    warm = warmup_epochs * steps_per_epoch
    if step < warm:
        return peak * (step + 1) / warm
    return peak * factor ** n_plateaus
