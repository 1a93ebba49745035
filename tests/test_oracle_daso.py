"""Pins for oracle.daso_sim (CPU).

Each test fixes the simulator by something other than itself:
  * B=1, S=0 with the uncast (fp32) wire is exactly synchronous SGD on the
    concatenated batch of all W ranks (north star; SPEC AC-2) — checked
    against an independent 10-line full-batch SGD loop written here, <= 1e-12
  * the staleness timing (reading R6 (A)) has a closed form from App. Eq. 5
    (P:303-315): with mu = wd = 0 and a common start,
        x_l = x0 - eta/(2S+P) * (2S * sum_{k=0}^{S} G_{l,k} + sum_i G_{i,0})
    checked against gradients recorded by an independent per-rank GD loop
  * degenerate cases: 1x1 = plain SGD; P = 1 = node-local synchronous SGD
  * invariants: node replicas bitwise identical every step (Fig. 4), all
    ranks identical after a blocking sync (Fig. 3), determinism (SPEC AC-9)
"""
import numpy as np
import pytest

import synthetic
from oracle import daso_sim, toy
from oracle.schedule import SchedConfig

D, BATCH = 64, 8


def toy_grad_fn(d=D, b=BATCH):
    cache = {}

    def fn(rank, step, w):
        key = (rank, step)
        if key not in cache:
            cache[key] = synthetic.toy_batch(d, b, rank, step)
        X, y = cache[key]
        return toy.grad(w, X, y)
    return fn


def _indep_grad(w, X, y):
    X = X.astype(np.float64)
    return X.T @ (X @ w - y.astype(np.float64)) / X.shape[0]


@pytest.mark.parametrize("P,G", [(2, 2), (3, 1), (1, 3), (2, 3)])
@pytest.mark.parametrize("mu,wd", [(0.0, 0.0), (0.9, 1e-4)])
def test_blocking_fp32_equals_sync_sgd_on_concatenated_batch(P, G, mu, wd):
    W, steps, lr = P * G, 12, 0.05
    x0 = synthetic.microbench_x0(D, seed=3).astype(np.float64)
    for cfg in (SchedConfig(B_init=1, S_init=0, total_epochs=1, steps_per_epoch=steps),
                SchedConfig(B_init=4, S_init=1, warmup_epochs=3, cooldown_epochs=0, total_epochs=3, steps_per_epoch=4)):
        out = daso_sim.simulate(P, G, cfg, steps, x0, toy_grad_fn(), lr, mu, wd, wire="fp32")
        # independent synchronous SGD over the concatenated batch
        x, v = x0.copy(), np.zeros(D)
        for k in range(steps):
            batches = [synthetic.toy_batch(D, BATCH, r, k) for r in range(W)]
            Xc = np.concatenate([b[0] for b in batches])
            yc = np.concatenate([b[1] for b in batches])
            g = _indep_grad(x, Xc, yc) + wd * x
            v = mu * v + g
            x = x - lr * v
        for r in range(W):
            np.testing.assert_allclose(out["x"][r], x, rtol=0, atol=1e-12)


@pytest.mark.parametrize("S,B,P", [(1, 1, 2), (1, 4, 2), (2, 2, 3), (2, 8, 2), (3, 4, 4)])
def test_staleness_closed_form_app_eq5(S, B, P):
    eta = 0.02
    x0 = synthetic.microbench_x0(D, seed=9).astype(np.float64)
    cfg = SchedConfig(B_init=B, S_init=S, total_epochs=1, steps_per_epoch=8 * B)
    out = daso_sim.simulate(P, 1, cfg, S + 1, x0, toy_grad_fn(), eta, 0.0, 0.0, wire="fp32", trace=True)
    assert out["records"][S].merge == 1 and out["records"][0].send == 1
    # independent per-rank gradient descent, recording G_{l,k}
    Gs = []
    for l in range(P):
        w, gl = x0.copy(), []
        for k in range(S + 1):
            X, y = synthetic.toy_batch(D, BATCH, l, k)
            g = _indep_grad(w, X, y)
            gl.append(g)
            w = w - eta * g
        Gs.append(gl)
    for l in range(P):
        expect = x0 - eta / (2 * S + P) * (2 * S * np.sum(Gs[l], axis=0) + np.sum([Gs[i][0] for i in range(P)], axis=0))
        np.testing.assert_allclose(out["trace"][S][l], expect, rtol=0, atol=1e-13)


def test_one_by_one_is_plain_sgd():
    x0 = synthetic.microbench_x0(D, seed=5).astype(np.float64)
    cfg = SchedConfig(B_init=4, S_init=1, warmup_epochs=1, cooldown_epochs=1, total_epochs=4, steps_per_epoch=4)
    out = daso_sim.simulate(1, 1, cfg, 16, x0, toy_grad_fn(), 0.03, 0.9, 1e-4, wire="bf16")
    x, v = x0.copy(), np.zeros(D)
    for k in range(16):
        X, y = synthetic.toy_batch(D, BATCH, 0, k)
        v = 0.9 * v + _indep_grad(x, X, y) + 1e-4 * x
        x = x - 0.03 * v
    np.testing.assert_allclose(out["x"][0], x, rtol=0, atol=1e-13)


def test_single_node_is_node_local_sync_sgd():
    """P = 1: the global tier is disabled (R12); the node is plain synchronous DP."""
    G = 3
    x0 = synthetic.microbench_x0(D, seed=6).astype(np.float64)
    cfg = SchedConfig(B_init=2, S_init=1, total_epochs=1, steps_per_epoch=16)
    out = daso_sim.simulate(1, G, cfg, 10, x0, toy_grad_fn(), 0.03, 0.9, 1e-4, wire="bf16")
    x, v = x0.copy(), np.zeros(D)
    for k in range(10):
        g = sum(_indep_grad(x, *synthetic.toy_batch(D, BATCH, r, k)) for r in range(G)) / G
        v = 0.9 * v + g + 1e-4 * x
        x = x - 0.03 * v
    for r in range(G):
        np.testing.assert_allclose(out["x"][r], x, rtol=0, atol=1e-13)


def test_replica_invariants_and_determinism():
    P, G = 2, 3
    x0 = synthetic.microbench_x0(D, seed=7).astype(np.float64)
    cfg = SchedConfig(B_init=4, S_init=2, warmup_epochs=1, cooldown_epochs=1, total_epochs=4, steps_per_epoch=8)
    a = daso_sim.simulate(P, G, cfg, 32, x0, toy_grad_fn(), 0.02, 0.9, 1e-4, wire="bf16",
                          epoch_flags=[0, 1, 0, 0], trace=True)
    b = daso_sim.simulate(P, G, cfg, 32, x0, toy_grad_fn(), 0.02, 0.9, 1e-4, wire="bf16",
                          epoch_flags=[0, 1, 0, 0], trace=True)
    for k, (xs, rec) in enumerate(zip(a["trace"], a["records"])):
        for j in range(P):
            for l in range(1, G):
                np.testing.assert_array_equal(xs[j * G + l], xs[j * G])
        if rec.send and rec.blocking:
            for r in range(1, P * G):
                np.testing.assert_array_equal(xs[r], xs[0])
        for r in range(P * G):
            np.testing.assert_array_equal(xs[r], b["trace"][k][r])
    # nodes do drift apart between non-blocking syncs (the method is not a no-op)
    cyc = [k for k, r in enumerate(a["records"]) if r.phase == 1 and not r.merge and not r.send]
    assert any(not np.array_equal(a["trace"][k][0], a["trace"][k][G]) for k in cyc)


def test_toy_config1_converges():
    """Config 1 (2x2, B=4, S=1, 20 steps) decreases the full-data loss."""
    d, b, P, G = 1000, 32, 2, 2
    fn = toy_grad_fn(d, b)
    cfg = SchedConfig(B_init=4, S_init=1, total_epochs=1, steps_per_epoch=20)
    out = daso_sim.simulate(P, G, cfg, 20, np.zeros(d), fn, 0.01, 0.9, 1e-4, wire="bf16")
    X, y = synthetic.toy_batch(d, 256, 999, 0)
    assert toy.loss(out["x"][0], X, y) < 0.5 * toy.loss(np.zeros(d), X, y)


def test_toy_gradient_finite_differences():
    X, y = synthetic.toy_batch(12, 5, 0, 0)
    w = np.random.default_rng(0).standard_normal(12)
    g = toy.grad(w, X, y)
    h = 1e-6
    fd = np.array([(toy.loss(w + h * e, X, y) - toy.loss(w - h * e, X, y)) / (2 * h) for e in np.eye(12)])
    np.testing.assert_allclose(g, fd, rtol=0, atol=1e-6)
    # full-batch gradient = mean of equal-shard gradients
    Xs, ys = np.split(X.astype(np.float64)[:4], 2), np.split(y.astype(np.float64)[:4], 2)
    np.testing.assert_allclose(toy.grad(w, X[:4], y[:4]), 0.5 * (toy.grad(w, Xs[0], ys[0]) + toy.grad(w, Xs[1], ys[1])),
                               rtol=0, atol=1e-12)


# ---------------------------------------------------------------------------
# Hand-derived pins of the bf16 wire THROUGH simulate ("parameters are cast to a
# 16-bit datatype representation during buffer packaging ... cast back to their original
# datatype"; Eq. (1)).  2 nodes x 1 GPU, mu = wd = 0, lr = 1, and a gradient
# g = w - target so that every local state is an exact, hand-chosen value.  The values
# are dyadic with more than 8 significant bits, so bf16 RNE changes them, incl. both tie
# directions; the expected numbers below were derived by hand (bf16 keeps 8 significant
# bits: 1 + 3*2^-9 -> 1 + 2^-7 (round up), 1 + 2^-8 -> 1 (tie, to even), 0.5 + 2^-10 -> 0.5
# (quarter ulp, down), 3 + 2^-7 -> 3 (tie, to even), fl64(1/3) -> 0.333984375).
# A composition mistake (casting the local state instead of the stale snapshot, casting
# after the merge, dropping the own snapshot, a wrong S weight) changes every number.
_T0 = [[1 + 3 * 2 ** -9, 1 + 2 ** -8, 1 / 3], [0.5 + 2 ** -10, 3 + 2 ** -7, 1 / 3]]   # after batch 0
_T1 = [[4.0, 2.0, 4.0], [1.0, -1.0, 4.0]]                                               # after batch 1


def _target_grad(r, k, w):
    return w - np.array((_T0 if k == 0 else _T1)[r])


@pytest.mark.parametrize("wire", ["bf16", "fp32"])
def test_bf16_wire_merge_hand_pin(wire):
    """B = 2, S = 1: send after batch 0, Eq. (1) merge after batch 1's update:
        x = (2S x_local + sum_i wire(x_i,0)) / (2S + P) = (2 x_local + s_0 + s_1) / 4."""
    cfg = SchedConfig(B_init=2, S_init=1, total_epochs=1, steps_per_epoch=8)
    out = daso_sim.simulate(2, 1, cfg, 2, np.zeros(3), _target_grad, 1.0, 0.0, 0.0, wire=wire, trace=True)
    assert out["records"][0].send == 1 and out["records"][1].merge == 1
    np.testing.assert_array_equal(out["trace"][0][0], _T0[0])          # batch 0: plain local updates
    np.testing.assert_array_equal(out["trace"][0][1], _T0[1])
    if wire == "bf16":
        # snapshots bf16: node 0 [1.0078125, 1.0, 0.333984375], node 1 [0.5, 3.0, 0.333984375]
        want = [[(8 + 1.0078125 + 0.5) / 4, (4 + 1.0 + 3.0) / 4, (8 + 2 * 0.333984375) / 4],
                [(2 + 1.0078125 + 0.5) / 4, (-2 + 1.0 + 3.0) / 4, (8 + 2 * 0.333984375) / 4]]
        assert want[0] == [2.376953125, 2.0, 2.1669921875]                # the hand values
        assert want[1] == [0.876953125, 0.5, 2.1669921875]
    else:
        # fp32 wire ("casting is not beneficial"): the snapshots are the exact states
        want = [[(8 + 1.005859375 + 0.5009765625) / 4, (4 + 1.00390625 + 3.0078125) / 4, (8 + 2 / 3) / 4],
                [(2 + 1.005859375 + 0.5009765625) / 4, (-2 + 1.00390625 + 3.0078125) / 4, (8 + 2 / 3) / 4]]
        assert want[0][:2] == [2.376708984375, 2.0029296875]
    for r in range(2):
        np.testing.assert_allclose(out["trace"][1][r], want[r], rtol=0, atol=1e-15)


def test_bf16_wire_blocking_average_hand_pin():
    """B = 1, S = 0 (blocking, Fig. 3, P:83 / P:86): after batch 0 both nodes hold the
    plain mean of the two bf16 snapshots: [(1.0078125 + 0.5)/2, (1 + 3)/2, 0.333984375]."""
    cfg = SchedConfig(B_init=1, S_init=0, total_epochs=1, steps_per_epoch=8)
    out = daso_sim.simulate(2, 1, cfg, 1, np.zeros(3), _target_grad, 1.0, 0.0, 0.0, wire="bf16", trace=True)
    assert out["records"][0].send == 1 and out["records"][0].blocking == 1
    for r in range(2):
        np.testing.assert_array_equal(out["trace"][0][r], [0.75390625, 2.0, 0.333984375])
