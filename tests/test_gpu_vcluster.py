"""Multi-rank DASO on ONE GPU: the virtual cluster (daso_vcluster_*, include/daso.h) runs the
product batch of every one of the W = P x G ranks — daso_step_ex, the fused node-tier kernel
over the sibling ranks' buffers (Fig. 2 node average + Fig. 4 parameter broadcast, P:75,
P:103), the bf16 pack, the Eq. (1) merge and the blocking average (Fig. 3)
— with a loopback group all-gather, and is compared with the CPU oracle every step, on every
rank: parameters within 1e-5 (fp32 wire) / 1e-2 (bf16 wire), schedule records bit-exact, node
replicas bitwise identical.  Covers the 8-GPU topologies of BASELINE configs 2/5 (2x4, 4x2,
8x1) and the 4-GPU ones, both wires, both data paths of the fused kernel (register / TMA).
No launch waits on another launch (the node barriers are pre-satisfied; see step_fused)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import synthetic  # noqa: E402
import paper_2104_05588_b200 as daso  # noqa: E402
from oracle import daso_sim  # noqa: E402
from oracle.schedule import SchedConfig, run_schedule  # noqa: E402
from parity_util import check_trajectory, toy_oracle  # noqa: E402


def run_vc(P, G, B, S, steps=20, d=1000, b=32, lr=0.01, mu=0.9, wd=1e-4, wire="bf16", warm=0, cool=0, epochs=1,
           spe=20, flags="", mode="fused", kernel=None, keep_trace=True, exchange="nccl"):
    torch.cuda.set_device(0)
    torch.backends.cuda.matmul.allow_tf32 = False
    prev = daso.daso_kernel_impl(kernel) if kernel else None
    W = P * G
    vc = daso.VCluster(W, G, B, S, d, warmup_epochs=warm, cooldown_epochs=cool, total_epochs=epochs,
                       steps_per_epoch=spe, momentum=mu, weight_decay=wd, wire=wire, mode=mode, exchange=exchange)
    try:
        fl = [int(c) for c in flags]
        traces = [[] for _ in range(W)]
        recs = [[] for _ in range(W)]
        for k in range(steps):
            for r in range(W):
                X, y = (torch.from_numpy(a).cuda() for a in synthetic.toy_batch(d, b, r, k))
                w = vc.x(r)[:d]
                vc.g(r)[:d] = X.T @ (X @ w - y) / b              # this rank's backward (toy gradient)
            plateau = fl[k // spe - 1] if k > 0 and k % spe == 0 and k // spe - 1 < len(fl) else 0
            rs = vc.step(lr, plateau)
            for r in range(W):
                recs[r].append(rs[r])
                if keep_trace:
                    traces[r].append(vc.x(r)[:d].cpu().numpy().copy())
        for r in range(W):
            assert vc.rank(r).check_finite()
        return traces, recs
    finally:
        vc.destroy()
        if prev is not None:
            daso.daso_kernel_impl(prev)


TOPOS = [(2, 2), (1, 4), (2, 4), (4, 2), (8, 1), (2, 1), (1, 2), (4, 1)]


@pytest.mark.parametrize("P,G", TOPOS)
@pytest.mark.parametrize("wire", ["bf16", "fp32"])
def test_vcluster_toy_config1(P, G, wire):
    """Config 1's toy (linear regression d = 1000, B = 4, S = 1, 20 steps) at every topology."""
    traces, recs = run_vc(P, G, 4, 1, wire=wire)
    check_trajectory(traces, recs, toy_oracle(P, G, 4, 1, wire=wire), P, G, wire)


@pytest.mark.parametrize("P,G", [(2, 2), (1, 4), (2, 4), (4, 2)])
@pytest.mark.parametrize("wire", ["bf16", "fp32"])
def test_vcluster_peer_data_paths_bit_identical(P, G, wire):
    """d = 40,000: shards of 10,000..20,000 span several 2048-parameter tiles plus a ragged tail.
    The fused node-tier kernel's three data paths — register (128-bit LDG/STG on peer
    addresses), TMA-staged (one thread issues bulk copies between CTA barriers) and
    warp-specialised TMA (the default: a driver warp and compute warps decoupled by mbarriers)
    — compute the same arithmetic in the same order: bitwise equal, and all match the oracle."""
    kw = dict(steps=10, d=40000, wire=wire)
    runs = {k: run_vc(P, G, 4, 1, kernel=k, **kw) for k in ("ldg", "tma", "auto")}
    a, ra = runs["ldg"]
    for k in ("tma", "auto"):
        b, rb = runs[k]
        for r in range(P * G):
            for t in range(10):
                np.testing.assert_array_equal(a[r][t].view(np.uint32), b[r][t].view(np.uint32))
        assert ra == rb
    check_trajectory(a, ra, toy_oracle(P, G, 4, 1, steps=10, d=40000, wire=wire), P, G, wire)


@pytest.mark.parametrize("P,G", [(2, 4), (4, 2), (8, 1), (2, 2)])
@pytest.mark.parametrize("wire", ["bf16", "fp32"])
def test_vcluster_full_schedule(P, G, wire):
    """Warm-up (blocking: pack -> all-gather -> average -> re-publish), cycling with plateau
    halving/reset, cool-down: 5 epochs x 8 batches."""
    kw = dict(steps=40, warm=1, cool=1, epochs=5, spe=8, flags="01100", wire=wire)
    traces, recs = run_vc(P, G, 4, 1, **kw)
    check_trajectory(traces, recs, toy_oracle(P, G, 4, 1, **kw), P, G, wire)


@pytest.mark.parametrize("P,G", [(2, 4), (4, 2), (8, 1)])
def test_vcluster_blocking_fp32_is_flat_sync(P, G):
    """B = 1, S = 0, fp32 wire: DASO == synchronous SGD on the concatenated batch; all W
    ranks bitwise identical after every batch."""
    traces, recs = run_vc(P, G, 1, 0, wire="fp32")
    check_trajectory(traces, recs, toy_oracle(P, G, 1, 0, wire="fp32"), P, G, "fp32")
    for r in range(1, P * G):
        for k in range(20):
            np.testing.assert_array_equal(traces[r][k].view(np.uint32), traces[0][k].view(np.uint32))


@pytest.mark.parametrize("P,G", [(2, 2), (2, 4)])
def test_vcluster_S_equals_B(P, G):
    """S = B = 2 (R8: the due merge runs before the new send in the same batch)."""
    traces, recs = run_vc(P, G, 2, 2, wire="fp32")
    check_trajectory(traces, recs, toy_oracle(P, G, 2, 2, wire="fp32"), P, G, "fp32")


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("mode", ["faithful", "sharded"])
def test_vcluster_one_gpu_per_node_modes(P, mode):
    """P x 1 in the faithful (paper structure) and sharded modes, full schedule."""
    kw = dict(steps=40, warm=1, cool=1, epochs=5, spe=8, flags="01100", wire="bf16")
    traces, recs = run_vc(P, 1, 4, 1, mode=mode, **kw)
    check_trajectory(traces, recs, toy_oracle(P, 1, 4, 1, **kw), P, 1, "bf16")


@pytest.mark.parametrize("P,G,B,S,mode", [(2, 2, 4, 1, "fused"), (2, 4, 4, 1, "fused"), (4, 2, 4, 1, "fused"),
                                          (8, 1, 4, 1, "fused"), (2, 2, 2, 2, "fused"), (4, 1, 2, 2, "faithful"),
                                          (2, 2, 1, 0, "fused"), (4, 1, 1, 0, "fused")])
@pytest.mark.parametrize("wire", ["bf16", "fp32"])
def test_vcluster_copy_engine_exchange(P, G, B, S, mode, wire):
    """The global tier's copy-engine exchange (DASO_EXCH_CE, the bench default) for real, between the
    sibling ranks on one GPU: same-device cudaMemcpyAsync pushes into the group members' slots, the
    cuStreamWriteValue64 arrival flags and consumed acks, cuStreamWaitValue64 at the merge — the full
    schedule (blocking warm-up / cool-down, cycling with plateau halving; S = B puts the flow-control
    acks on the critical path of every cycle) against the oracle."""
    spe = 8 if B <= 4 else 16
    kw = dict(steps=40, warm=1, cool=1, epochs=5, spe=spe, flags="01100", wire=wire, mode=mode)
    traces, recs = run_vc(P, G, B, S, exchange="ce", **kw)
    kw.pop("mode")
    check_trajectory(traces, recs, toy_oracle(P, G, B, S, **kw), P, G, wire)


def test_vcluster_config5_schedule_2x4():
    """Config 5: 1000 batches = 50 epochs x 20, warm-up 5, cool-down 5, B0 = 4,
    S0 = 1, plateau flags Bernoulli(0.3) (seed 7), topology 2x4 through daso_step on every
    virtual rank: every record equals the oracle's bit for bit; parameters finite."""
    flags = "".join(str(f) for f in synthetic.plateau_pattern(50, 0.3))
    traces, recs = run_vc(2, 4, 4, 1, steps=1000, d=64, b=8, warm=5, cool=5, epochs=50, spe=20, flags=flags,
                          keep_trace=False)
    cfg = SchedConfig(B_init=4, S_init=1, warmup_epochs=5, cooldown_epochs=5, total_epochs=50, steps_per_epoch=20,
                      gpus_per_node=4)
    ref = [r.as_dict() for r in run_schedule(cfg, 1000, [int(c) for c in flags])]
    for r in range(8):
        assert recs[r] == ref


@pytest.mark.parametrize("wire", ["bf16", "fp32"])
def test_vcluster_full_size_2x4_sampled(wire):
    """BASELINE config 2 at full size and its primary topology: n = 25,557,032 fp32 params,
    2 nodes x 4 GPUs, B = 4, S = 1, seeded per-rank gradients, 6 batches (send, merge, plain,
    plain, send, merge) through the fused kernel at its bench launch configuration; 20,004
    sampled parameters of every rank against the oracle simulating exactly those elements
    (DASO is elementwise in the parameters given the gradients)."""
    import mp_micro
    N, P, G, steps = mp_micro.N, 2, 4, 6
    idx = mp_micro.sample_indices()
    torch.cuda.set_device(0)
    vc = daso.VCluster(P * G, G, 4, 1, N, total_epochs=1, steps_per_epoch=4 << 20, momentum=0.9,
                       weight_decay=1e-4, wire=wire, mode="fused")
    try:
        x0 = torch.from_numpy(synthetic.microbench_x0(N)).cuda()
        for r in range(P * G):
            vc.x(r)[:N] = x0
        tidx = torch.from_numpy(idx).cuda()
        trace = [[] for _ in range(P * G)]
        for k in range(steps):
            for r in range(P * G):
                vc.g(r)[:N] = torch.from_numpy(synthetic.microbench_grad(N, r, k)).cuda()
            vc.step(0.1)
            for r in range(P * G):
                trace[r].append(vc.x(r)[tidx].cpu().numpy())
        for r in range(P * G):
            assert vc.rank(r).check_finite()
    finally:
        vc.destroy()
    grads = {(r, k): synthetic.microbench_grad(N, r, k)[idx] for r in range(P * G) for k in range(steps)}
    cfg = SchedConfig(B_init=4, S_init=1, total_epochs=1, steps_per_epoch=4 << 20)
    ref = daso_sim.simulate(P, G, cfg, steps, synthetic.microbench_x0(N)[idx], lambda r, k, w: grads[(r, k)],
                            0.1, 0.9, 1e-4, wire=wire, trace=True)
    tol = 1e-2 if wire == "bf16" else 1e-5
    for r in range(P * G):
        for k in range(steps):
            xo = ref["trace"][k][r]
            rms = np.sqrt(np.mean(xo ** 2))
            assert np.all(np.abs(trace[r][k] - xo) <= tol * (np.abs(xo) + rms)), (r, k)
            assert np.linalg.norm(trace[r][k] - xo) <= tol * np.linalg.norm(xo)
    for j in range(P):
        for l in range(1, G):
            for k in range(steps):
                np.testing.assert_array_equal(trace[j * G + l][k], trace[j * G][k])


@pytest.mark.parametrize("P,G", [(2, 2), (2, 4), (4, 2)])
def test_vcluster_fused_trace_accounting(P, G, monkeypatch):
    """The library's per-launch byte accounting (daso_trace) for the fused node tier: a plain batch is
    one node-tier launch moving 2 (G-1) * 4 B per shard element over NVLink per direction (peer
    gradient reads + peer parameter stores); a blocking batch is the node-tier kernel without its
    parameter stores (OP_NOX, gradient reads only) plus the average/re-publish launch (stores only),
    so the same NVLink bytes over two launches.  (Fig. 3 / Fig. 4.)"""
    torch.cuda.set_device(0)
    d = 4099
    seg = daso.daso_padded_numel(d, G) // G
    per_batch = 2.0 * (G - 1) * 4.0 * seg
    # (B, S, exchange, launches per batch, extra NVLink bytes per batch): with the copy-engine transport
    # a blocking batch's node-tier kernel also stores the packed bf16 row into the P-1 other group
    # members' slots (kernel push, DASO_BLOCKING_PUSH=2), 2 B per shard element each; with the default (1)
    # the copy engines push after the kernel (exchange bytes, not kernel bytes)
    # (default mode 1: the node-tier kernel pushes for groups of P >= 3, the copy engines for P = 2)
    for B, S, ex, mode, launches, extra in [(4, 1, "nccl", "1", 1, 0.0), (1, 0, "nccl", "1", 2, 0.0),
                                            (1, 0, "ce", "2", 2, (P - 1) * 2.0 * seg),
                                            (1, 0, "ce", "1", 2, (P - 1) * 2.0 * seg if P >= 3 else 0.0)]:
        monkeypatch.setenv("DASO_BLOCKING_PUSH", mode)
        vc = daso.VCluster(P * G, G, B, S, d, total_epochs=1, steps_per_epoch=B * 64, mode="fused", exchange=ex)
        try:
            for r in range(P * G):
                vc.rank(r).trace_enable(True)
            steps = 3
            for k in range(steps):
                for r in range(P * G):
                    vc.g(r)[:d] = torch.from_numpy(synthetic.microbench_grad(d, r, k)).cuda()
                vc.step(0.01)
            for r in range(P * G):
                t = vc.rank(r).trace_read(reset=True)
                assert t["kernel_launches"] == steps * launches, (B, S, ex, mode, r, t)
                assert t["kernel_nvl_bytes"] == pytest.approx(steps * (per_batch + extra)), (B, S, ex, mode, r, t)
                assert vc.rank(r).check_finite()
        finally:
            vc.destroy()


@pytest.mark.parametrize("P,G", [(2, 2), (4, 1), (2, 4), (8, 1), (4, 2)])
def test_vcluster_blocking_kernel_push_equals_copy_engines(P, G, monkeypatch):
    """Blocking syncs with the CE transport: the pack kernel storing the packed row into every group
    member's slot (kernel push; DASO_BLOCKING_PUSH=2 also from the fused node-tier kernel at G > 1) and
    the copy-engine pushes after it (DASO_BLOCKING_PUSH=0) deliver the same rows, so every rank's
    trajectory is bitwise identical (Fig. 3)."""
    kw = dict(steps=24, warm=1, cool=1, epochs=3, spe=8, flags="1", wire="bf16", exchange="ce")
    monkeypatch.setenv("DASO_BLOCKING_PUSH", "0")
    ce, recs_ce = run_vc(P, G, 4, 1, **kw)
    monkeypatch.setenv("DASO_BLOCKING_PUSH", "2")
    kp, recs_kp = run_vc(P, G, 4, 1, **kw)
    assert recs_ce == recs_kp
    for r in range(P * G):
        for k in range(len(ce[r])):
            np.testing.assert_array_equal(ce[r][k].view(np.uint32), kp[r][k].view(np.uint32))


@pytest.mark.parametrize("P,G", [(2, 2), (2, 4), (4, 2)])
def test_vcluster_avg_publish_paths_bit_identical(P, G, monkeypatch):
    """The fused blocking tail's two data paths — register stores to the node peers (DASO_AVG_PUBLISH=ldg)
    and shared-memory tiles with bulk stores (tma, default) — give bitwise identical trajectories on a
    multi-tile shard with a ragged tail (d = 40,000), every batch blocking (B = 1, S = 0; Fig. 3 / 4)."""
    kw = dict(steps=6, d=40_000, wire="bf16", exchange="ce")
    monkeypatch.setenv("DASO_AVG_PUBLISH", "ldg")
    a, recs_a = run_vc(P, G, 1, 0, **kw)
    monkeypatch.setenv("DASO_AVG_PUBLISH", "tma")
    b, recs_b = run_vc(P, G, 1, 0, **kw)
    assert recs_a == recs_b
    for r in range(P * G):
        for k in range(len(a[r])):
            np.testing.assert_array_equal(a[r][k].view(np.uint32), b[r][k].view(np.uint32))


def _run_vc_microbench(P, G, n, steps, B=4, S=1):
    vc = daso.VCluster(P * G, G, B, S, n, total_epochs=1, steps_per_epoch=B << 20, mode="fused")
    try:
        x0 = torch.from_numpy(synthetic.microbench_x0(n)).cuda()
        for r in range(P * G):
            vc.x(r)[:n] = x0
        out = []
        for k in range(steps):
            for r in range(P * G):
                vc.g(r)[:n] = torch.from_numpy(synthetic.microbench_grad(n, r, k)).cuda()
            vc.step(0.1)
            out.append([vc.x(r)[:n].cpu().numpy().view(np.uint32).copy() for r in range(P * G)])
        for r in range(P * G):
            assert vc.rank(r).check_finite()
        return out
    finally:
        vc.destroy()


@pytest.mark.parametrize("P,G", [(1, 2), (2, 2)])
def test_vcluster_ws_output_buffers_bit_identical(P, G, monkeypatch):
    """The warp-specialised node-tier kernel with 2 (default) and 4 shared-memory output buffers
    (DASO_PEER_OUT) on shards of 1.5M parameters — several tiles per persistent CTA, so the buffer
    rotation and the release of buffers whose bulk stores have read them are exercised — gives
    bitwise identical parameters for every rank and step, including a merge and a send (B = 4, S = 1)."""
    n = 3_000_000
    monkeypatch.setenv("DASO_PEER_OUT", "2")
    a = _run_vc_microbench(P, G, n, 3)
    monkeypatch.setenv("DASO_PEER_OUT", "4")
    b = _run_vc_microbench(P, G, n, 3)
    for k in range(3):
        for r in range(P * G):
            np.testing.assert_array_equal(a[k][r], b[k][r])


@pytest.mark.parametrize("P,G", [(2, 2), (4, 1)])
def test_vcluster_full_size_blocking_sampled(P, G, monkeypatch):
    """Blocking syncs (B = 1, S = 0: every batch Fig. 3 average + Fig. 4 re-publish) at config 2's
    full size through the copy-engine exchange: at 2x2 the node-tier kernel without its parameter
    stores and the bulk-store average / re-publish kernel on 12.8M-parameter shards (many tiles per
    CTA: the output-buffer rotation and the next-tile prefetch run), at 4x1 the local K2 pushing
    the packed row into the group members' slots and the P-specialised K4.  Sampled parameters of
    every rank against the oracle (elementwise given the gradients), node replicas bitwise equal,
    and the register-store tail bitwise equal to the bulk-store tail."""
    import mp_micro
    N, steps = mp_micro.N, 3
    idx = mp_micro.sample_indices()
    torch.cuda.set_device(0)
    tidx = torch.from_numpy(idx).cuda()

    def run():
        vc = daso.VCluster(P * G, G, 1, 0, N, total_epochs=1, steps_per_epoch=1 << 20, momentum=0.9,
                           weight_decay=1e-4, wire="bf16", mode="fused", exchange="ce")
        try:
            x0 = torch.from_numpy(synthetic.microbench_x0(N)).cuda()
            for r in range(P * G):
                vc.x(r)[:N] = x0
            trace = [[] for _ in range(P * G)]
            for k in range(steps):
                for r in range(P * G):
                    vc.g(r)[:N] = torch.from_numpy(synthetic.microbench_grad(N, r, k)).cuda()
                vc.step(0.1)
                for r in range(P * G):
                    trace[r].append(vc.x(r)[tidx].cpu().numpy())
            for r in range(P * G):
                assert vc.rank(r).check_finite()
            return trace
        finally:
            vc.destroy()

    monkeypatch.setenv("DASO_AVG_PUBLISH", "tma")
    trace = run()
    grads = {(r, k): synthetic.microbench_grad(N, r, k)[idx] for r in range(P * G) for k in range(steps)}
    cfg = SchedConfig(B_init=1, S_init=0, total_epochs=1, steps_per_epoch=1 << 20)
    ref = daso_sim.simulate(P, G, cfg, steps, synthetic.microbench_x0(N)[idx], lambda r, k, w: grads[(r, k)],
                            0.1, 0.9, 1e-4, wire="bf16", trace=True)
    for r in range(P * G):
        for k in range(steps):
            xo = ref["trace"][k][r]
            rms = np.sqrt(np.mean(xo ** 2))
            assert np.all(np.abs(trace[r][k] - xo) <= 1e-2 * (np.abs(xo) + rms)), (r, k)
    for j in range(P):
        for l in range(1, G):
            for k in range(steps):
                np.testing.assert_array_equal(trace[j * G + l][k], trace[j * G][k])
    if G > 1:
        monkeypatch.setenv("DASO_AVG_PUBLISH", "ldg")
        other = run()
        for r in range(P * G):
            for k in range(steps):
                np.testing.assert_array_equal(other[r][k].view(np.uint32), trace[r][k].view(np.uint32))
