"""Pins for oracle.schedule (CPU).

* golden hand examples for the halving/reset rule and phase_of (cited)
* brute force: every plateau pattern over E <= 8 epochs, several (B0, S0, G,
  warm-up, cool-down) configs, against a second, independently written
  epoch-level event generator below (closed-form positions i % B == 0, due
  steps from a dict) instead of the oracle's incremental counters
* invariants: 0 <= S <= B, one exchange in flight, merge exactly S_p batches
  after its send, sends once per B batches in cycling, every batch otherwise
* config 1 (toy) expectations from SURVEY §8(d): sends at k=0,4,8,12,16 with
  groups 0,1,0,1,0, merges at k=1,5,9,13,17
"""
import itertools
import json
import os

import pytest

from oracle.schedule import (CYCLING, COOLDOWN, WARMUP, SchedConfig, halve_or_reset, phase_of,
                             run_schedule, validate)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", GOLD["schedule_step"])
def test_halve_or_reset_golden(ex):
    if ex["fired"]:
        B, S, _ = halve_or_reset(ex["B"], ex["S"], ex["B_init"], ex["S_init"])
    else:
        B, S = ex["B"], ex["S"]
    assert [B, S] == ex["out"]


@pytest.mark.parametrize("ex", GOLD["phase_of"])
def test_phase_of_golden(ex):
    cfg = SchedConfig(B_init=1, warmup_epochs=ex["warmup"], cooldown_epochs=ex["cooldown"],
                      total_epochs=ex["total"], steps_per_epoch=1)
    assert phase_of(ex["epoch"], cfg) == ex["phase"]


def test_default_S_is_B_over_4():
    assert [SchedConfig(B_init=b).resolved_S() for b in (1, 2, 4, 8, 16)] == [1, 1, 1, 2, 4]


@pytest.mark.parametrize("bad", [
    dict(B_init=0), dict(B_init=4, S_init=5), dict(B_init=4, S_init=1, steps_per_epoch=6),
    dict(B_init=14, S_init=1, steps_per_epoch=14), dict(B_init=4, warmup_epochs=2, cooldown_epochs=2, total_epochs=3),
    dict(B_init=4, total_epochs=0), dict(B_init=4, gpus_per_node=0),
])
def test_config_errors(bad):
    base = dict(B_init=4, S_init=1, warmup_epochs=0, cooldown_epochs=0, total_epochs=1, steps_per_epoch=8)
    with pytest.raises(ValueError):
        validate(SchedConfig(**{**base, **bad}))


def test_toy_config_events():
    recs = run_schedule(SchedConfig(B_init=4, S_init=1, total_epochs=1, steps_per_epoch=20, gpus_per_node=2), 20)
    assert [r.step for r in recs if r.send] == [0, 4, 8, 12, 16]
    assert [r.send_group for r in recs if r.send] == [0, 1, 0, 1, 0]
    assert [r.step for r in recs if r.merge] == [1, 5, 9, 13, 17]
    assert all(r.merge_S == 1 and r.blocking == 0 for r in recs if r.merge)


# ---------------------------------------------------------------- independent generator
def independent_events(B0, S0, G, warm, cool, total, spe, flags):
    """Epoch-level restatement of P:97-99 written without the oracle's counters."""
    out = []
    B, S = B0, S0
    due = {}          # due step -> (S_p, group, sent)
    nsync = 0
    for e in range(total):
        action = 0
        if e > 0 and flags[e - 1] and (warm <= e - 1 < total - cool):
            if B == 1 and S <= 1:
                B, S, action = B0, S0, 2
            else:
                B, S, action = max(1, B // 2), (S // 2 if S == 0 else max(1, S // 2)), 1
        ph = WARMUP if e < warm else (COOLDOWN if e >= total - cool else CYCLING)
        for i in range(spe):
            k = e * spe + i
            m = due.pop(k, None)
            if ph == CYCLING:
                send, blocking, bic = int(i % B == 0), int(i % B == 0 and S == 0), i % B
            else:
                send, blocking, bic = 1, 1, 0
            grp = -1
            if send:
                grp = nsync % G
                nsync += 1
                if not blocking:
                    due[k + S] = (S, grp, k)
            pend = next(iter(due.items()), None)
            out.append(dict(step=k, epoch=e, phase=ph, B=B, S=S, batch_in_cycle=bic,
                            plateau_action=action if i == 0 else 0, send=send, blocking=blocking,
                            send_group=grp, n_syncs=nsync, merge=int(m is not None),
                            merge_S=m[0] if m else 0, merge_group=m[1] if m else -1,
                            merge_sent=m[2] if m else -1, pending=int(pend is not None),
                            due=pend[0] if pend else -1))
    return out


CONFIGS = [  # (B0, S0, G, warm, cool, total, spe)
    (4, 1, 4, 1, 1, 7, 8), (8, 2, 2, 0, 0, 8, 8), (2, 2, 3, 2, 1, 8, 4), (1, 1, 1, 0, 2, 6, 3),
    (4, 4, 2, 1, 0, 8, 4), (8, 0, 2, 1, 1, 8, 8), (6, 3, 2, 0, 0, 7, 6), (4, 1, 8, 2, 2, 8, 4),
]


@pytest.mark.parametrize("cfg", CONFIGS)
def test_schedule_bruteforce_vs_independent(cfg):
    B0, S0, G, warm, cool, total, spe = cfg
    c = SchedConfig(B_init=B0, S_init=S0, warmup_epochs=warm, cooldown_epochs=cool,
                    total_epochs=total, steps_per_epoch=spe, gpus_per_node=G)
    for flags in itertools.product((0, 1), repeat=total):
        got = [r.as_dict() for r in run_schedule(c, total * spe, list(flags))]
        assert got == independent_events(B0, S0, G, warm, cool, total, spe, flags), flags


@pytest.mark.parametrize("cfg", CONFIGS)
def test_schedule_invariants(cfg):
    B0, S0, G, warm, cool, total, spe = cfg
    c = SchedConfig(B_init=B0, S_init=S0, warmup_epochs=warm, cooldown_epochs=cool,
                    total_epochs=total, steps_per_epoch=spe, gpus_per_node=G)
    for flags in itertools.product((0, 1), repeat=min(total, 6)):
        recs = run_schedule(c, total * spe, list(flags))
        sends = {r.step: r for r in recs if r.send and not r.blocking}
        for r in recs:
            assert 0 <= r.S <= r.B
            assert r.phase == phase_of(r.epoch, c)
            if r.phase != CYCLING:
                assert r.send and r.blocking
            if r.merge:
                s = sends[r.merge_sent]
                assert r.step - r.merge_sent == r.merge_S == s.S and r.merge_group == s.send_group
        assert len(sends) == sum(r.merge for r in recs) + recs[-1].pending
        # phases appear in order warm-up* cycling* cool-down*
        ph = [r.phase for r in recs]
        assert ph == sorted(ph)


def test_ac7_schedule_table():
    """SPEC AC-7 style table: always-plateau from B0 in {1,2,4,8} walks
    the halving chain to (1,1) then resets."""
    expect = {1: [(1, 1), (1, 1), (1, 1)], 2: [(2, 1), (1, 1), (2, 1), (1, 1)],
              4: [(4, 1), (2, 1), (1, 1), (4, 1), (2, 1)],
              8: [(8, 2), (4, 1), (2, 1), (1, 1), (8, 2), (4, 1)]}
    for B0, chain in expect.items():
        c = SchedConfig(B_init=B0, total_epochs=len(chain), steps_per_epoch=8)
        recs = run_schedule(c, len(chain) * 8, [1] * len(chain))
        assert [(recs[e * 8].B, recs[e * 8].S) for e in range(len(chain))] == chain


def test_plateau_ignored_outside_cycling():
    c = SchedConfig(B_init=4, S_init=1, warmup_epochs=2, cooldown_epochs=0, total_epochs=4, steps_per_epoch=4)
    recs = run_schedule(c, 16, [1, 0, 0, 0])
    assert all(r.B == 4 for r in recs)
    recs = run_schedule(c, 16, [0, 0, 1, 0])
    assert [r.B for r in recs[12:]] == [2] * 4
