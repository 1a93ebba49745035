"""The C++ schedule of libdaso.so (daso_sched_*) against the independent CPU
oracle (oracle/schedule.py): every record field bit-exact, every step.

Covers config 5 of SURVEY §8(d) (1000 steps = 50 epochs x 20, warm-up 5,
cool-down 5, B0 = 4, S0 = 1; plateau patterns Bernoulli(0.3) seed 7, all-true,
all-false; G in {1, 2, 4, 8}) and exhaustive plateau patterns on short runs.
"""
import itertools
import math

import pytest

import synthetic
from oracle.schedule import SchedConfig, plateau_arg, run_schedule
from paper_2104_05588_b200 import DasoError, Schedule


def abi_records(B0, S0, warm, cool, total, spe, G, flags, steps):
    s = Schedule(B0, S0, warm, cool, total, spe, G)
    return [s.next(plateau_arg(k, flags, spe)) for k in range(steps)]


def oracle_records(B0, S0, warm, cool, total, spe, G, flags, steps):
    cfg = SchedConfig(B_init=B0, S_init=S0, warmup_epochs=warm, cooldown_epochs=cool, total_epochs=total,
                      steps_per_epoch=spe, gpus_per_node=G)
    return [r.as_dict() for r in run_schedule(cfg, steps, flags)]


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("pattern", ["bernoulli", "all", "none"])
def test_config5_sweep_bit_exact(G, pattern):
    epochs, spe = 50, 20
    flags = {"bernoulli": synthetic.plateau_pattern(epochs, 0.3), "all": [1] * epochs, "none": [0] * epochs}[pattern]
    args = (4, 1, 5, 5, epochs, spe, G, flags, epochs * spe)
    assert abi_records(*args) == oracle_records(*args)


@pytest.mark.parametrize("cfg", [
    (4, 1, 1, 1, 6, 8, 4), (8, 2, 0, 0, 6, 8, 2), (2, 2, 2, 1, 6, 4, 3), (1, 1, 0, 2, 6, 3, 1),
    (4, 4, 1, 0, 6, 4, 2), (8, 0, 1, 1, 6, 8, 2), (6, 3, 0, 0, 6, 6, 2), (16, -1, 1, 1, 6, 16, 8),
])
def test_exhaustive_plateau_patterns_bit_exact(cfg):
    B0, S0, warm, cool, total, spe, G = cfg
    for flags in itertools.product((0, 1), repeat=total):
        args = (B0, S0, warm, cool, total, spe, G, list(flags), total * spe + 5)   # run past the end too
        assert abi_records(*args) == oracle_records(*args), flags


def test_toy_config_records():
    recs = abi_records(4, 1, 0, 0, 1, 20, 2, [], 20)
    assert [r["step"] for r in recs if r["send"]] == [0, 4, 8, 12, 16]
    assert [r["send_group"] for r in recs if r["send"]] == [0, 1, 0, 1, 0]
    assert [r["step"] for r in recs if r["merge"]] == [1, 5, 9, 13, 17]


@pytest.mark.parametrize("bad", [
    (0, 0, 0, 0, 1, 8, 1), (4, 5, 0, 0, 1, 8, 1), (4, 1, 0, 0, 1, 6, 1), (14, 1, 0, 0, 1, 14, 1),
    (4, 1, 2, 2, 3, 8, 1), (4, 1, 0, 0, 0, 8, 1), (4, 1, 0, 0, 1, 0, 1), (4, 1, 0, 0, 1, 8, 0),
])
def test_config_errors_match_oracle(bad):
    with pytest.raises(DasoError) as e:
        Schedule(*bad)
    assert e.value.status == 1
    B0, S0, warm, cool, total, spe, G = bad
    with pytest.raises(ValueError):
        oracle_records(B0, S0, warm, cool, total, spe, G, [], 1)


def test_random_configs_property_bit_exact():
    """Property test: random valid configurations and plateau patterns, C++ == oracle."""
    hyp = pytest.importorskip("hypothesis")
    st = hyp.strategies

    @st.composite
    def configs(draw):
        B0 = draw(st.sampled_from([1, 2, 3, 4, 6, 8, 12, 16]))
        chain, b = [], B0
        while True:
            chain.append(b)
            if b == 1:
                break
            b = max(1, b // 2)
        lcm = 1
        for c in chain:
            lcm = lcm * c // math.gcd(lcm, c)
        spe = lcm * draw(st.integers(1, 3))
        S0 = draw(st.integers(-1, B0))
        total = draw(st.integers(1, 7))
        warm = draw(st.integers(0, total))
        cool = draw(st.integers(0, total - warm))
        G = draw(st.integers(1, 8))
        flags = draw(st.lists(st.integers(0, 1), min_size=total, max_size=total))
        return B0, S0, warm, cool, total, spe, G, flags

    @hyp.settings(max_examples=150, deadline=None)
    @hyp.given(configs())
    def check(c):
        B0, S0, warm, cool, total, spe, G, flags = c
        args = (B0, S0, warm, cool, total, spe, G, flags, total * spe + 3)
        assert abi_records(*args) == oracle_records(*args)

    check()
