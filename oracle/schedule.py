"""DASO phase / B,S schedule (TEST INFRASTRUCTURE — see oracle/__init__.py).

Written from P:97-99 (§3):
  * "Training ... can be divided into three key phases: warm-up, cycling, and
    cool-down. The warm-up and cool-down phases utilize blocking global
    synchronizations, while the cycling phase uses non-blocking global
    synchronizations ... warm-up and cool-down phases occur for a set number of
    epochs at the beginning and end of training"
  * "In the cycling phase, the number of forward-backward passes between global
    synchronizations (B) and the number of batches to wait for global
    synchronization data (W) are varied. B is specified manually ... For W, an
    initial value of B/4 ... Each time the training loss plateaus, B and W are
    reduced by a factor of two, down to a minimum of one. When B, W = 1 and the
    loss has plateaued, both are reset to their initial values"
  * "In the blocking case, all synchronization steps are performed after each
    batch"; "the average was calculated ... every B-th batch".
W is called S here, as in Eq. (1) and Fig. 5.

Readings: R6 (merge S batches after the send, after that batch's
update), R8 (a due merge runs before a new send in the same batch), R9
(rotation: group = number of previous syncs mod G, blocking syncs included),
R10 (plateau checked at epoch ends, applied from the next epoch's first batch;
cycles restart every epoch; every B of the halving chain divides the epoch
length), R13 (halving / reset rule), R14 (warm-up / cool-down in epochs),
R15 (first cycling batch sends), S = 0 accepted = blocking every B batches.
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict

WARMUP, CYCLING, COOLDOWN = 0, 1, 2


@dataclass
class SchedConfig:
    B_init: int
    S_init: int = -1          # < 0: max(1, B_init // 4)   ("an initial value of B/4")
    warmup_epochs: int = 0
    cooldown_epochs: int = 0
    total_epochs: int = 1
    steps_per_epoch: int = 1 << 20
    gpus_per_node: int = 1    # only used for the rotation index

    def resolved_S(self) -> int:
        return max(1, self.B_init // 4) if self.S_init < 0 else self.S_init


def validate(cfg: SchedConfig) -> None:
    """Config errors (reading R10)."""
    S = cfg.resolved_S()
    if cfg.B_init < 1 or cfg.gpus_per_node < 1:
        raise ValueError("config error: B >= 1, G >= 1 required")
    if not 0 <= S <= cfg.B_init:
        raise ValueError("config error: 0 <= S <= B required")
    if cfg.total_epochs < 1 or cfg.steps_per_epoch < 1:
        raise ValueError("config error: total_epochs, steps_per_epoch >= 1 required")
    if cfg.warmup_epochs < 0 or cfg.cooldown_epochs < 0 or cfg.warmup_epochs + cfg.cooldown_epochs > cfg.total_epochs:
        raise ValueError("config error: warmup + cooldown <= total required")
    b = cfg.B_init
    while True:
        if cfg.steps_per_epoch % b != 0:
            raise ValueError("config error: every B of the halving chain must divide steps_per_epoch")
        if b == 1:
            break
        b = max(1, b // 2)


def phase_of(epoch: int, cfg: SchedConfig) -> int:
    """P:97. SPEC S:469-477 examples."""
    if epoch < cfg.warmup_epochs:
        return WARMUP
    if epoch >= cfg.total_epochs - cfg.cooldown_epochs:
        return COOLDOWN
    return CYCLING


def halve_or_reset(B: int, S: int, B_init: int, S_init: int) -> tuple[int, int, int]:
    """P:99 plateau rule (reading R13). Returns (B, S, action) with action
    1 = halved, 2 = reset."""
    if B > 1 or S > 1:
        return max(1, B // 2), (0 if S == 0 else max(1, S // 2)), 1
    return B_init, S_init, 2


@dataclass
class Record:
    step: int
    epoch: int
    phase: int
    B: int
    S: int
    batch_in_cycle: int
    plateau_action: int   # 0 none, 1 halved, 2 reset (applied at this step)
    send: int
    blocking: int
    send_group: int
    n_syncs: int          # global syncs issued up to and including this step
    merge: int
    merge_S: int
    merge_group: int
    merge_sent: int
    pending: int          # exchange in flight after this step
    due: int

    def as_dict(self) -> dict:
        return asdict(self)


@dataclass
class Schedule:
    cfg: SchedConfig
    B: int = 0
    S: int = 0
    step: int = 0
    batch_in_cycle: int = 0
    n_syncs: int = 0
    pend: dict | None = None
    records: list = field(default_factory=list)

    def __post_init__(self):
        validate(self.cfg)
        self.B = self.cfg.B_init
        self.S = self.cfg.resolved_S()

    def next(self, plateau: int = 0) -> Record:
        """Advance by one batch.  ``plateau`` is consulted only at the first
        batch of an epoch e >= 1 and reports whether the training loss
        plateaued at the end of epoch e-1 (reading R10); it acts only if epoch
        e-1 was a cycling epoch ("In the cycling phase ...")."""
        cfg = self.cfg
        k = self.step
        spe = cfg.steps_per_epoch
        e = k // spe
        action = 0
        if k % spe == 0:
            if k > 0 and plateau == 1 and phase_of(e - 1, cfg) == CYCLING:
                self.B, self.S, action = halve_or_reset(self.B, self.S, cfg.B_init, cfg.resolved_S())
            self.batch_in_cycle = 0            # cycles restart every epoch (R10)
        ph = phase_of(e, cfg)

        # due merge first (R6, R8)
        merge = merge_S = 0
        merge_group = merge_sent = -1
        if self.pend is not None and self.pend["due"] == k:
            merge, merge_S = 1, self.pend["S"]
            merge_group, merge_sent = self.pend["group"], self.pend["sent"]
            self.pend = None

        if ph == CYCLING:
            bic = self.batch_in_cycle
            send = int(bic == 0)               # "every B-th batch", R15
            blocking = int(send and self.S == 0)
            self.batch_in_cycle = (bic + 1) % self.B
        else:
            bic = 0
            send, blocking = 1, 1              # P:86 blocking: after each batch
        send_group = -1
        if send:
            send_group = self.n_syncs % cfg.gpus_per_node    # rotation (R9)
            self.n_syncs += 1
            if not blocking:
                assert self.pend is None, "two exchanges in flight"
                self.pend = {"due": k + self.S, "S": self.S, "group": send_group, "sent": k}
        rec = Record(step=k, epoch=e, phase=ph, B=self.B, S=self.S, batch_in_cycle=bic,
                     plateau_action=action, send=send, blocking=blocking, send_group=send_group,
                     n_syncs=self.n_syncs, merge=merge, merge_S=merge_S, merge_group=merge_group,
                     merge_sent=merge_sent, pending=int(self.pend is not None),
                     due=(self.pend["due"] if self.pend is not None else -1))
        self.records.append(rec)
        self.step += 1
        return rec


def plateau_arg(step: int, epoch_flags: list[int], steps_per_epoch: int) -> int:
    """Per-step plateau argument from per-epoch flags: at the first batch of
    epoch e >= 1, flag[e-1]; 0 elsewhere."""
    if step > 0 and step % steps_per_epoch == 0:
        e = step // steps_per_epoch
        if e - 1 < len(epoch_flags):
            return int(epoch_flags[e - 1])
    return 0


def run_schedule(cfg: SchedConfig, steps: int, epoch_flags: list[int] | None = None) -> list[Record]:
    sch = Schedule(cfg)
    flags = epoch_flags or []
    return [sch.next(plateau_arg(k, flags, cfg.steps_per_epoch)) for k in range(steps)]
