"""Plateau detector and LR schedule (reading R20).

Oracle pins: torch.optim.lr_scheduler.ReduceLROnPlateau (a library routine; mode
'min', relative threshold, cooldown 0: it fires after patience+1 bad epochs, so
torch patience = ours - 1) on random positive loss sequences; hand examples.
C ABI (daso_plateau_*, daso_lr_at) vs the oracle: identical fired sequences and LRs.
"""
import numpy as np
import pytest

from oracle.plateau import PlateauDetector, lr_at
import paper_2104_05588_b200 as daso


def loss_sequences(seed, count=60, epochs=40):
    rng = np.random.default_rng(seed)
    for _ in range(count):
        base = np.exp(-np.cumsum(rng.uniform(0, 0.05, epochs) * (rng.random(epochs) < 0.5)))
        yield list(base * (1 + 0.01 * rng.standard_normal(epochs)) + 0.1)


@pytest.mark.parametrize("patience,threshold", [(1, 0.0), (2, 0.01), (5, 0.01), (3, 0.05)])
def test_oracle_matches_torch_reduce_lr_on_plateau(patience, threshold):
    torch = pytest.importorskip("torch")
    for losses in loss_sequences(patience * 7 + int(threshold * 100)):
        det = PlateauDetector(patience, threshold)
        mine = [det.update(l) for l in losses]
        p = torch.nn.Parameter(torch.zeros(1))
        opt = torch.optim.SGD([p], lr=1.0)
        sch = torch.optim.lr_scheduler.ReduceLROnPlateau(opt, mode="min", factor=0.5, patience=patience - 1,
                                                         threshold=threshold, threshold_mode="rel", cooldown=0,
                                                         eps=0.0)
        theirs = []
        for l in losses:
            before = opt.param_groups[0]["lr"]
            sch.step(l)
            theirs.append(int(opt.param_groups[0]["lr"] < before))
        assert mine == theirs


def test_hand_examples():
    d = PlateauDetector(5, 0.01)
    assert [d.update(1.0) for _ in range(11)] == [0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1]   # constant loss
    d = PlateauDetector(5, 0.01)
    assert not any(d.update(0.9 ** e) for e in range(40))                                # 10%/epoch decrease
    d = PlateauDetector(2, 0.01)
    assert [d.update(v) for v in [1.0, 0.995, 0.994, 0.5]] == [0, 0, 1, 0]               # < 1% is stable
    with pytest.raises(ValueError):
        PlateauDetector(0, 0.01)
    with pytest.raises(ValueError):
        PlateauDetector(2, 0.01).update(float("nan"))


def test_lr_hand_values():
    # peak scaled with the number of processes; warm-up from 0; decay by factor
    assert lr_at(0, 10, 0.1, 4, 5, 0.5, 0) == pytest.approx(0.4 / 50)
    assert lr_at(49, 10, 0.1, 4, 5, 0.5, 0) == pytest.approx(0.4)
    assert lr_at(50, 10, 0.1, 4, 5, 0.5, 2) == pytest.approx(0.1)
    assert lr_at(0, 10, 0.1, 1, 0, 0.75, 1) == pytest.approx(0.075)


@pytest.mark.parametrize("patience,threshold", [(1, 0.0), (2, 0.01), (5, 0.01), (4, 0.2)])
def test_abi_detector_bit_exact_vs_oracle(patience, threshold):
    rng = np.random.default_rng(patience)
    for losses in list(loss_sequences(patience, 30)) + [list(rng.standard_normal(50)) for _ in range(10)]:
        a, b = PlateauDetector(patience, threshold), daso.PlateauDetector(patience, threshold)
        assert [a.update(l) for l in losses] == [b.update(l) for l in losses]


def test_abi_lr_matches_oracle():
    for step in range(0, 200, 7):
        for npl in range(4):
            assert daso.daso_lr_at(step, 20, 0.0125, 8, 5, 0.75, npl) == lr_at(step, 20, 0.0125, 8, 5, 0.75, npl)


def test_abi_errors():
    with pytest.raises(daso.DasoError):
        daso.PlateauDetector(0, 0.01)
    with pytest.raises(daso.DasoError):
        daso.PlateauDetector(2, 0.01).update(float("inf"))
    with pytest.raises(daso.DasoError):
        daso.daso_lr_at(0, 0, 0.1, 1, 1, 0.5, 0)
