"""Pins for oracle.numerics / oracle.sgd / oracle.topology (CPU, no GPU).

What fixes each function independently of the oracle's own code:
  * golden hand-derived examples (tests/golden/spec_examples.json, each cited)
  * library routines: torch's fp32->bf16 cast (RNE) and torch.optim.SGD
  * mathematical identities: Eq. (1) weights sum to one, fixed point,
    convex hull, bf16 idempotence and its 2^-8 relative error bound
  * brute-force partition property of the group map
"""
import json
import os

import numpy as np
import pytest

from oracle import numerics, sgd, topology

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _bits_to_f32(h: str) -> float:
    return float(np.array([int(h, 16)], dtype=np.uint32).view(np.float32)[0])


# ---------------------------------------------------------------- topology
@pytest.mark.parametrize("ex", GOLD["group_maps"])
def test_group_map_golden(ex):
    assert topology.global_groups(ex["num_nodes"], ex["gpus_per_node"]) == ex["groups"]
    assert topology.node_groups(ex["num_nodes"], ex["gpus_per_node"]) == ex["node_groups"]


@pytest.mark.parametrize("ex", GOLD["rotation"])
def test_rotation_golden(ex):
    assert topology.active_group(ex["cycle_index"], ex["groups"]) == ex["active"]


@pytest.mark.parametrize("ex", GOLD["rank_lookup"])
def test_rank_lookup_golden(ex):
    assert topology.rank_lookup(ex["rank"], ex["num_nodes"], ex["gpus_per_node"]) == (ex["node"], ex["local"])


def test_rank_lookup_range_and_config_errors():
    with pytest.raises(IndexError):
        topology.rank_lookup(8, 2, 4)
    with pytest.raises(ValueError):
        topology.node_groups(0, 4)
    with pytest.raises(ValueError):
        topology.global_groups(2, 0)


def test_group_partition_bruteforce():
    """every rank in exactly one group and one node group, W <= 1024."""
    for P in range(1, 33):
        for G in range(1, 33):
            if P * G > 1024:
                continue
            gg = topology.global_groups(P, G)
            ng = topology.node_groups(P, G)
            assert sorted(r for grp in gg for r in grp) == list(range(P * G))
            assert sorted(r for grp in ng for r in grp) == list(range(P * G))
            assert all(len(grp) == P for grp in gg) and all(len(grp) == G for grp in ng)
            # a group holds one GPU per node, all with the same local id
            for k, grp in enumerate(gg):
                assert [topology.rank_lookup(r, P, G) for r in grp] == [(j, k) for j in range(P)]


def test_rotation_period():
    for G in range(1, 9):
        seq = [topology.active_group(c, G) for c in range(3 * G)]
        assert sorted(seq[:G]) == list(range(G)) and seq[:G] == seq[G:2 * G]


# ---------------------------------------------------------------- average
@pytest.mark.parametrize("ex", GOLD["average"])
def test_average_golden(ex):
    np.testing.assert_array_equal(numerics.average([np.array(v, float) for v in ex["vectors"]]), ex["out"])


def test_average_singleton_and_errors():
    v = np.random.default_rng(0).standard_normal(17)
    np.testing.assert_array_equal(numerics.average([v]), v)
    with pytest.raises(ValueError):
        numerics.average([])
    with pytest.raises(ValueError):
        numerics.average([np.zeros(2), np.zeros(3)])


# ---------------------------------------------------------------- Eq. (1)
@pytest.mark.parametrize("ex", GOLD["eq1"])
def test_eq1_golden(ex):
    out = numerics.weighted_stale_average(np.array(ex["local"], float),
                                          [np.array(s, float) for s in ex["stale"]], ex["S"])
    np.testing.assert_allclose(out, ex["out"], rtol=0, atol=1e-15)


def test_eq1_weights_sum_to_one_and_are_2S_and_1():
    """Weights by linearity: unit vectors isolate each weight."""
    for S in range(1, 6):
        for P in range(1, 9):
            w_local = numerics.weighted_stale_average(np.ones(1), [np.zeros(1)] * P, S)[0]
            assert w_local == pytest.approx(2 * S / (2 * S + P), abs=1e-15)
            for i in range(P):
                st = [np.zeros(1)] * P
                st = st[:i] + [np.ones(1)] + st[i + 1:]
                assert numerics.weighted_stale_average(np.zeros(1), st, S)[0] == pytest.approx(1 / (2 * S + P), abs=1e-15)
            assert w_local + P / (2 * S + P) == pytest.approx(1.0, abs=1e-15)


def test_eq1_fixed_point_and_convex_hull():
    rng = np.random.default_rng(1)
    for S in (1, 2, 4):
        for P in (1, 2, 3, 8):
            c = rng.standard_normal(50)
            np.testing.assert_allclose(numerics.weighted_stale_average(c, [c] * P, S), c, rtol=1e-15, atol=0)
            loc = rng.standard_normal(50)
            st = [rng.standard_normal(50) for _ in range(P)]
            out = numerics.weighted_stale_average(loc, st, S)
            lo = np.minimum.reduce([loc] + st)
            hi = np.maximum.reduce([loc] + st)
            assert np.all(out >= lo - 1e-15) and np.all(out <= hi + 1e-15)


def test_eq1_argument_errors():
    with pytest.raises(ValueError):
        numerics.weighted_stale_average(np.zeros(1), [np.zeros(1)], 0)
    with pytest.raises(ValueError):
        numerics.weighted_stale_average(np.zeros(1), [], 1)


# ---------------------------------------------------------------- bf16 packing
@pytest.mark.parametrize("ex", GOLD["bf16"])
def test_bf16_golden(ex):
    if "in_bits" in ex:
        got = numerics.bf16_round(np.array([_bits_to_f32(ex["in_bits"])]))[0]
        assert np.float32(got).view(np.uint32) == int(ex["out_bits"], 16)
    else:
        assert numerics.bf16_round(np.array([ex["in"]]))[0] == ex["out"]


def test_bf16_matches_torch_cast():
    """Library routine: torch's fp32 -> bfloat16 conversion is RNE."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(2)
    vals = np.concatenate([
        rng.standard_normal(200000) * 10.0 ** rng.integers(-30, 30, 200000),
        rng.integers(0, 2 ** 31 - 2 ** 24, 20000).astype(np.uint32).view(np.float32).astype(np.float64),  # random bit patterns
        np.array([0.0, -0.0, 1.0, -1.0, 3.3895313892515355e38, 1e-40, -1e-40]),
    ])
    vals = vals[np.isfinite(vals.astype(np.float32))]
    ref = torch.from_numpy(vals.astype(np.float32)).to(torch.bfloat16).to(torch.float32).numpy()
    got = numerics.bf16_round(vals).astype(np.float32)
    np.testing.assert_array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_bf16_idempotent_and_error_bound():
    rng = np.random.default_rng(3)
    v = rng.standard_normal(100000) * np.exp(rng.uniform(-40, 40, 100000))
    q = numerics.bf16_round(v)
    np.testing.assert_array_equal(numerics.bf16_round(q), q)
    f = v.astype(np.float32).astype(np.float64)
    assert np.max(np.abs(q - f) / np.abs(f)) <= 2.0 ** -8
    with pytest.raises(ValueError):
        numerics.bf16_round(np.array([np.nan]))


def test_blocking_bf16_golden():
    for ex in GOLD["blocking_bf16"]:
        snaps = [numerics.wire(np.array(p, float), "bf16") for p in ex["params"]]
        np.testing.assert_array_equal(numerics.average(snaps), ex["out"])


def test_wire_fp32_is_identity():
    v = np.random.default_rng(4).standard_normal(33)
    np.testing.assert_array_equal(numerics.wire(v, "fp32"), v)


# ---------------------------------------------------------------- SGD
@pytest.mark.parametrize("ex", GOLD["sgd"])
def test_sgd_golden(ex):
    x, v = np.array(ex["x"], float), np.zeros(len(ex["x"]))
    for t in range(ex["steps"]):
        x, v = sgd.sgd_step(x, v, np.array(ex["g"], float), ex["lr"], ex["mu"], ex["wd"])
        np.testing.assert_allclose(x, ex["trajectory"][t], rtol=0, atol=1e-15)


def test_sgd_matches_torch_optim_sgd():
    """Library routine: torch.optim.SGD(momentum, weight_decay), float64."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    x0 = rng.standard_normal(64)
    grads = [rng.standard_normal(64) for _ in range(7)]
    p = torch.nn.Parameter(torch.tensor(x0, dtype=torch.float64))
    opt = torch.optim.SGD([p], lr=0.05, momentum=0.9, weight_decay=1e-4)
    x, v = x0.copy(), np.zeros(64)
    for g in grads:
        p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
        x, v = sgd.sgd_step(x, v, g, 0.05, 0.9, 1e-4)
        np.testing.assert_allclose(x, p.detach().numpy(), rtol=1e-14, atol=1e-15)


def test_sgd_composed_equals_app_eq2():
    """App. Eq. 2: mu = wd = 0, S steps = x_t - eta * sum of grads."""
    rng = np.random.default_rng(6)
    x0 = rng.standard_normal(10)
    gs = [rng.standard_normal(10) for _ in range(5)]
    x, v = x0.copy(), np.zeros(10)
    for g in gs:
        x, v = sgd.sgd_step(x, v, g, 0.3, 0.0, 0.0)
    np.testing.assert_allclose(x, x0 - 0.3 * np.sum(gs, axis=0), rtol=0, atol=1e-12)
