#!/usr/bin/env python
"""DASO sync-path benchmark on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1)

One step = one DASO batch of the whole hot path through the C ABI (daso_step), driven
by the B/S schedule.  In the default fused mode: one node-tier kernel per GPU reduces the
node's gradient shards over NVLink, applies the update (+ Eq. (1) merge when due, + bf16
pack when sending) and stores the new parameter shard into every node peer; every B-th
batch the packed shard goes to the group members by copy-engine pushes on the library's
side streams (non-blocking, merged S batches later); blocking batches (S = 0) end with the
average / re-publish kernel.  (faithful mode: NCCL node all-reduce, fused update kernel,
node broadcast after merges, group all-gather.)
Workload: n = 25,557,032 fp32 parameters (ResNet-50-sized), synthetic seeded
gradients, B = 4, S = 1, topology P x G virtual nodes: N=1 -> 1x1,
2 -> 2x1, 4 -> 2x2, 8 -> 2x4.

Mode: default "fused" — the node tier (gradient reduce over the node's
GPUs + update/merge/pack + parameter all-gather) in one kernel over NVLink peer
memory; "faithful" = the paper's structure (node all-reduce, rotating group exchange,
node broadcast); "sharded" = the same with NCCL reduce-scatter / all-gather.  All
three are parity-tested against the oracle.

Timing: W untimed warm-up steps; then K steps, each bracketed by CUDA events on the
compute stream (the stream daso_step runs on).  Between steps, outside the events,
the gradient bucket is refreshed from a resident copy (a backward pass would
overwrite it; without the refresh the node all-reduce would grow it G-fold per
step) and L2 is flushed by reading a 256 MB buffer.  Barrier + synchronize on both
sides; max over ranks.  value = fp32 parameter bytes synchronised per second over
all ranks = 4 n N / t_step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_PARAMS = 25_557_032          # torchvision resnet50: 25,557,032 params in 161 tensors
METRIC = "DASO sync ms/step & GB/s, samples/s (ResNet-50, 25.6M params) at 1/2/4/8 B200"
TOPO = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 4)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", 1)))
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--B", type=int, default=4)
    ap.add_argument("--S", type=int, default=1)
    ap.add_argument("--n", type=int, default=N_PARAMS)
    ap.add_argument("--topology", default="", help="PxG, default by --gpus")
    ap.add_argument("--mode", choices=["faithful", "sharded", "fused"], default="fused")
    ap.add_argument("--wire", choices=["bf16", "fp32"], default="bf16")
    ap.add_argument("--lr", type=float, default=0.1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--nccl-max-ctas", type=int, default=0, help="cap the side-stream exchange's NCCL CTAs")
    ap.add_argument("--exchange", choices=["nccl", "ce"], default="ce",
                    help="global-tier transport: copy-engine pushes (DASO_EXCH_CE, default: no SMs, hidden behind "
                         "compute under SM contention) or NCCL all-gather (DASO_EXCH_NCCL)")
    ap.add_argument("--compute-ms", type=float, default=0.0,
                    help="untimed synthetic fwd/bwd stand-in (bf16 GEMMs) between steps, to measure how much of "
                         "the global exchange the next batch's compute hides")
    ap.add_argument("--overlap-compute-ms", type=float, default=1.0,
                    help="fwd/bwd stand-in per batch inside the hidden-fraction cycles (P > 1); config 3's "
                         "real fwd/bwd (~55 ms at 256/GPU) hides the exchange trivially but drowns it in noise")
    ap.add_argument("--cycles", type=int, default=30, help="B-cycles per leg of the hidden-fraction measurement")
    ap.add_argument("--gemm-cycles", type=int, default=120,
                    help="B-cycles per leg with the GEMM stand-in (its cycle-to-cycle jitter is ~10x the exchange)")
    ap.add_argument("--overlap-compute", choices=["gemm", "sleep", "both"], default="both",
                    help="fwd/bwd stand-in of the hidden-fraction cycles: bf16 GEMMs (SM/HBM contention, jittery), "
                         "a deterministic device sleep (precise), or both")
    ap.add_argument("--dump-steps", action="store_true", help="add every timed step's ms and kind to the line")
    ap.add_argument("--no-kernels", action="store_true", help="skip the per-kernel roofline table (N=1)")
    ap.add_argument("--no-vcluster", action="store_true", help="skip the one-GPU 2x4 virtual-cluster block (N=1)")
    ap.add_argument("--ref-div", type=int, default=4,
                    help="reference arm: oracle sample = n / ref-div parameters per step (scaled per parameter)")
    return ap.parse_args()


def topology(a, world):
    if a.topology:
        P, G = (int(v) for v in a.topology.lower().split("x"))
    else:
        P, G = TOPO.get(world, (world, 1))
    if P * G != world:
        raise SystemExit(f"topology {P}x{G} does not match world {world}")
    return P, G


def ncu_traffic(kernel_prefix: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the dominant kernel
    from the committed `ncu --set full` capture summary (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p))
    e = d.get(kernel_prefix)
    return (e["dram_bytes_per_launch"], e.get("source")) if e else (None, None)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML poller for SM clock and throttle reasons during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
        self._stop = threading.Event()

    def sample(self):
        if not self.ok:
            return
        self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
        try:
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for bit, name in self.REASONS.items():
            if r & bit and name != "gpu_idle":
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.002)

    def __enter__(self):
        self.sample()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self.t.join()
        self.sample()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_compute(ms: float, dev):
    """A stand-in for the next batch's forward/backward: bf16 8192^3 GEMMs totalling ~ms."""
    if ms <= 0:
        return lambda: None
    import torch
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    b = torch.randn_like(a)
    c = torch.empty_like(a)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    reps = max(1, round(ms / (e0.elapsed_time(e1) / 10)))

    def run():
        for _ in range(reps):
            torch.matmul(a, b, out=c)
    return run


def dist_setup():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("gloo")
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_baseline(P, G, B, S, n, wire):
    from oracle import bench as obench
    r = obench.calibrated(P, G, B, S, n, budget_s=12.0, wire=wire)
    gbs = 4.0 * r["n"] * r["ranks"] / r["s_per_step"] / 1e9
    return {"value": gbs, "unit": "GB/s", "cores": r["cores"], "kind": "oracle",
            "ms_per_step": r["s_per_step"] * 1e3 * (n / r["n"]),
            "sample": (f"oracle.daso_sim (numpy fp64, 1 core of {os.cpu_count()}) on {r['n']:,} of {n:,} params, "
                       f"all {r['ranks']} ranks of {P}x{G} simulated, {r['steps']} steps, {r['seconds']:.1f} s; "
                       f"value scaled per param")}


def run_reference(a):
    rank, world, _ = dist_setup()
    if rank != 0:
        return
    P, G = topology(a, world)
    from oracle import bench as obench
    # n/4 by default: at that size every fp64 state vector (51 MB) is far larger than the host's
    # caches, so the per-parameter cost is the full-size one (a 1/16 sample fit in cache and read
    # ~2x faster than full size in round 1)
    n_sample = max(1 << 16, a.n // max(1, a.ref_div))
    r = obench.time_sync_path(P, G, a.B, a.S, n_sample, a.steps, warmup=a.warmup, lr=a.lr, wire=a.wire)
    gbs = 4.0 * n_sample * P * G / r["s_per_step"] / 1e9
    sample = (f"oracle.daso_sim (numpy fp64, 1 core of {os.cpu_count()}) on {n_sample:,} of {a.n:,} params per "
              f"step, all {P * G} ranks of {P}x{G} simulated; value scaled per param")
    line = {"metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": r["s_per_step"] * 1e3 * (a.n / n_sample), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": "sync-path microbench (config 2)", "n_params": a.n, "topology": f"{P}x{G}",
                       "B": a.B, "S": a.S, "wire": a.wire},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def kernel_table(n: int, peak: float, iters: int = 30, warmup: int = 5) -> dict:
    """Per-kernel HBM roofline of every fused kernel on the sync path at n parameters (SURVEY §8(d),
    DESIGN.md §6), launched through the C ABI on resident buffers, CUDA events on the launching
    stream around each launch, a 256 MB read between launches so each starts from a cold, clean
    L2.  achieved = algorithmic bytes per launch / mean launch time; frac = achieved / peak."""
    import torch
    import paper_2104_05588_b200 as daso
    stride = daso.daso_padded_numel(n, 8)
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = (torch.randn(stride, device="cuda", generator=gen) * 0.02)[:n]
    v = torch.zeros(stride, device="cuda")[:n]
    g = (torch.randn(stride, device="cuda", generator=gen) * 0.01)[:n]
    slot = (torch.randn(8, stride, device="cuda", generator=gen) * 0.02).to(torch.bfloat16)
    pk = torch.zeros(stride, dtype=torch.bfloat16, device="cuda")
    wb = 2
    cases = {
        "K1_update": (lambda: daso.daso_k_update(x, v, g, 1e-3, 0.9, 1e-4, 0.5), 20),
        "K2_update_pack": (lambda: daso.daso_k_update(x, v, g, 1e-3, 0.9, 1e-4, 0.5, pack_out=pk), 20 + wb),
        "K3_update_merge_P2": (lambda: daso.daso_k_update_merge(x, v, g, 1e-3, 0.9, 1e-4, 0.5, slot[:2], 1), 20 + 2 * wb),
        "K3_update_merge_pack_P2": (lambda: daso.daso_k_update_merge(x, v, g, 1e-3, 0.9, 1e-4, 0.5, slot[:2], 1,
                                                                      pack_out=pk), 20 + 3 * wb),
        "K3_update_merge_P8": (lambda: daso.daso_k_update_merge(x, v, g, 1e-3, 0.9, 1e-4, 0.5, slot[:8], 1), 20 + 8 * wb),
        "K4_average_P2": (lambda: daso.daso_k_average(x, slot[:2]), 2 * wb + 4),
        "K4_average_P8": (lambda: daso.daso_k_average(x, slot[:8]), 8 * wb + 4),
        "pack_only": (lambda: daso.daso_k_pack(x, pk), 4 + wb),
    }
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    # untimed device work queued after the flush, so the launch under the events never waits for the
    # host (the ctypes call into the library takes a few microseconds)
    slack = make_sleep(0.02)
    rows = {}
    for name, (fn, bpp) in cases.items():
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        stream = torch.cuda.current_stream()
        for e0, e1 in ev:
            flush.sum()
            slack()
            e0.record(stream)
            fn()
            e1.record(stream)
        torch.cuda.synchronize()
        us = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
        mean = sum(us) / len(us)
        gbs = bpp * n / (mean * 1e-6) / 1e9
        rows[name] = {"bytes_per_param": bpp, "bytes_per_launch": bpp * n, "us_mean": mean, "us_p10": us[len(us) // 10],
                      "us_p90": us[(9 * len(us)) // 10], "achieved_gbs": gbs, "frac": gbs / peak}
    return rows


def vcluster_block(n: int, B: int, S: int, peak: float, exchange: str, steps: int = 16, warm: int = 8) -> dict:
    """The headline 2x4 batch on ONE GPU: a virtual cluster (daso_vcluster_*) runs all 8 ranks' product
    batches — the fused node-tier kernel (G = 4), bf16 pack, loopback group all-gather, Eq. (1) merge —
    with every peer buffer in this GPU's HBM.  Each launch's algorithmic bytes (per shard element
    12 + 8G (+ P*wb merge) (+ wb pack)) all hit local HBM here, so the node-tier kernel
    gets an HBM roofline; the NVLink roofline needs real GPUs (the N > 1 lines)."""
    import torch
    import paper_2104_05588_b200 as daso
    vc = daso.VCluster(8, 4, B, S, n, total_epochs=1, steps_per_epoch=B * (1 << 20), mode="fused",
                       exchange=exchange)
    try:
        gen = torch.Generator(device="cuda").manual_seed(0)
        x0 = torch.randn(n, device="cuda", generator=gen) * 0.02
        for r in range(8):
            vc.x(r)[:n] = x0
            vc.g(r)[:n] = torch.randn(n, device="cuda", generator=gen) * 0.01
        for _ in range(warm):
            vc.step(0.01)
        torch.cuda.synchronize()
        for r in range(8):
            vc.rank(r).trace_read(reset=True)
            vc.rank(r).trace_enable(True)
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            vc.step(0.01)
        e1.record(stream)
        torch.cuda.synchronize()
        tr = [vc.rank(r).trace_read(reset=True) for r in range(8)]
        ok = all(vc.rank(r).check_finite() for r in range(8))
    finally:
        vc.destroy()
    k = sum(t["kernel_launches"] for t in tr)
    ms = sum(t["kernel_ms"] for t in tr)
    by = sum(t["kernel_bytes"] for t in tr)
    gbs = by / (ms * 1e-3) / 1e9 if ms else None
    return {"topology": "2x4 (8 virtual ranks on one GPU)", "B": B, "S": S, "exchange": exchange, "steps": steps,
            "ms_per_cluster_batch": e0.elapsed_time(e1) / steps, "kernel_launches": k,
            "us_per_launch": ms / max(k, 1) * 1e3, "bytes_per_launch": by / max(k, 1),
            "achieved_gbs": gbs, "frac_of_hbm": gbs / peak if gbs else None, "finite": ok,
            "note": "timing includes the 8 ranks' batches run one after another plus the loopback copies; "
                    "the per-launch figures are the library's CUDA-event spans of its kernels"}


def pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(q * len(xs)))] if xs else None


def make_compute_small(ms: float, dev):
    """Fine-grained fwd/bwd stand-in for the hidden-fraction cycles: bf16 4096^3 GEMMs (~0.1 ms
    each) totalling ~ms, so legs with and without the exchange differ by little more than the
    exchange itself."""
    if ms <= 0:
        return lambda: None
    import torch
    a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    b = torch.randn_like(a)
    c = torch.empty_like(a)
    for _ in range(5):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    reps = max(1, round(ms / (e0.elapsed_time(e1) / 20)))

    def run():
        for _ in range(reps):
            torch.matmul(a, b, out=c)
    return run


def make_sleep(ms: float):
    """Deterministic fwd/bwd stand-in for the hidden-fraction cycles: one spinning thread
    (torch.cuda._sleep) for ~ms of device time.  Unlike GEMMs it has no run-to-run jitter, so a
    40-100 us exchange is resolvable; it does not model SM or HBM contention (the GEMM legs do)."""
    if ms <= 0:
        return lambda: None
    import torch
    torch.cuda._sleep(1000)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.cuda._sleep(10_000_000)
    e1.record()
    torch.cuda.synchronize()
    cycles = int(10_000_000 * ms / e0.elapsed_time(e1))
    return lambda: torch.cuda._sleep(cycles)


def exposed_from_cycles(t_with, t_without):
    """Exposed exchange time per cycle: the median of the paired differences of alternating cycles
    (cycle 2i with the exchange, 2i+1 without): drift across the run cancels, only the drift between
    the two adjacent cycles of a pair remains."""
    return statistics.median([w - wo for w, wo in zip(t_with, t_without)])


def hidden_fraction(exposed, n_exch_per_cycle, t_ag):
    """1 - exposed / (exchanges per cycle x T_AG,alone); a cycle faster with the exchange
    than without counts as fully hidden."""
    return 1.0 - max(0.0, exposed) / (n_exch_per_cycle * t_ag) if t_ag > 0 else None


def overlap_cycles(ctx, a, g, g_src, stream, world, compute, n_exch_per_cycle, t_ag, cycles=None):
    """SURVEY §8(d) hidden fraction: hidden = 1 - (T_with - T_without) / T_AG,alone, per B-cycle.
    One cycle = B batches of [fwd/bwd stand-in (bf16 GEMMs) ; gradient refresh ; daso_step], timed by
    CUDA events on the compute stream from the cycle's first batch to the end of its last.  In
    steady state every cycle contains exactly one merge, whose batch makes the compute stream wait
    for its exchange, so each cycle's time includes exactly one exchange's exposed part and any
    slowdown the concurrent all-gather causes to the GEMMs and the fused kernels.  T_without: the
    same cycles with the group all-gather suppressed (daso_set_exchange(0)).  The two legs
    alternate block by block (a block is 1 cycle, or 2 when S = B so that the timed cycle's merge
    waits for an exchange of its own leg) to cancel clock and power drift; T_AG,alone is measured
    before the bench's first step (daso_exchange_alone).  The exposed time is the median of the
    paired differences (cycle 2i with the exchange minus cycle 2i+1 without): drift across the run
    cancels, only the drift within a pair remains; the difference of the two legs' medians is reported
    beside it."""
    import torch
    block = 1 if a.S < a.B else 2
    cycles = cycles or a.cycles

    def batch():
        compute()
        g.copy_(g_src)
        ctx.step(a.lr)

    while ctx.query()["batch_in_cycle"] != a.B - 1:   # align: the next batch starts a cycle
        batch()
    legs = {True: [], False: []}
    for c in range(2 * cycles):
        enabled = c % 2 == 0
        ctx.set_exchange(enabled)
        for _ in range(block - 1):
            for _ in range(a.B):
                batch()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.B):
            batch()
        e1.record(stream)
        legs[enabled].append((e0, e1))
    ctx.set_exchange(True)
    torch.cuda.synchronize()
    t_with = [e0.elapsed_time(e1) for e0, e1 in legs[True]]
    t_without = [e0.elapsed_time(e1) for e0, e1 in legs[False]]
    w_med = max_over_ranks(statistics.median(t_with), world)
    wo_med = max_over_ranks(statistics.median(t_without), world)
    exposed = max_over_ranks(exposed_from_cycles(t_with, t_without), world)
    hidden = hidden_fraction(exposed, n_exch_per_cycle, t_ag)
    spread = max_over_ranks(pct(t_without, 0.9) - pct(t_without, 0.1), world)
    return {"def": "1 - (T_cycle,with - T_cycle,without) / (exchanges per cycle x T_AG,alone); exposed = median of "
                   "the paired differences of alternating cycles, max over ranks; T_AG,alone before the first step",
            "cycles_per_leg": cycles, "compute_ms_per_batch": a.overlap_compute_ms,
            "T_cycle_with_ms": w_med, "T_cycle_without_ms": wo_med, "exposed_ms": exposed,
            "exposed_ms_from_leg_medians": w_med - wo_med,
            "T_cycle_without_p10_p90_spread_ms": spread,
            "T_AG_alone_ms": t_ag, "exchanges_per_cycle": n_exch_per_cycle, "hidden_fraction": hidden}


def run_ours(a):
    import torch
    import synthetic
    import paper_2104_05588_b200 as daso

    rank, world, local = dist_setup()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    P, G = topology(a, world)
    n = a.n
    dev = torch.device("cuda", local)
    uid = daso.rendezvous_unique_id() if world > 1 else daso.daso_get_unique_id()
    ctx = daso.daso_init(world, G, a.B, a.S, rank=rank, uid=uid, total_epochs=1,
                         steps_per_epoch=a.B * (1 << 20), momentum=0.9, weight_decay=1e-4, wire=a.wire,
                         mode=a.mode, nccl_max_ctas=a.nccl_max_ctas, exchange=a.exchange)
    n_pad = daso.daso_padded_numel(n, G)
    x = torch.zeros(n_pad, dtype=torch.float32, device=dev)
    g = torch.zeros_like(x)
    v = torch.zeros_like(x)
    x[:n] = torch.from_numpy(synthetic.microbench_x0(n)).to(dev)
    g_src = torch.zeros_like(x)
    l2_flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)   # 256 MB > 126 MB L2
    g_src[:n] = torch.from_numpy(synthetic.microbench_grad(n, rank, 0)).to(dev)
    ctx.bind(x, g, v, n)
    stream = torch.cuda.current_stream()
    t_ag = max_over_ranks(ctx.exchange_alone(10), world) if P > 1 else 0.0   # T_AG,alone: nothing in flight yet

    compute = make_compute(a.compute_ms, dev)
    for _ in range(a.warmup):
        g.copy_(g_src)
        compute()
        ctx.step(a.lr)
    torch.cuda.synchronize()
    ctx.trace_read(reset=True)
    ctx.trace_enable(True)
    barrier(world)
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    kind_of = []
    slack = make_sleep(0.2)         # untimed device work queued before every step: the host always runs
                                    # ahead, so host-side jitter never leaves the GPU idle inside a window
    with ClockSampler(local) as clk:
        for k in range(a.steps):
            g.copy_(g_src)
            compute()
            l2_flush.sum()          # read-only L2 flush: the step starts cold with a clean L2
            slack()
            ev0[k].record(stream)
            r = ctx.step(a.lr)
            ev1[k].record(stream)
            # the batch kind that EXECUTED: with P = 1 the global tier is disabled (R12), so every
            # batch is a plain update whatever the schedule record says
            kind_of.append("plain" if P == 1 else "blocking" if r["blocking"] else
                           "merge+send" if (r["merge"] and r["send"]) else "merge" if r["merge"] else
                           "send" if r["send"] else "plain")
        torch.cuda.synchronize()
    barrier(world)
    step_ms = [e0.elapsed_time(e1) for e0, e1 in zip(ev0, ev1)]
    t_ms = max_over_ranks(sum(step_ms), world)
    tr = ctx.trace_read(reset=True)
    ctx.trace_enable(False)
    finite = ctx.check_finite()
    launches_total = int(sum_over_ranks(float(tr["kernel_launches"]), world))

    ms_per_step = t_ms / a.steps
    value = 4.0 * n * world / (ms_per_step * 1e-3) / 1e9
    peak, peak_src = peaks()
    kern_gbs = tr["kernel_bytes"] / (tr["kernel_ms"] * 1e-3) / 1e9 if tr["kernel_ms"] > 0 else None
    kern_gbs = max_over_ranks(-kern_gbs, world) * -1 if kern_gbs is not None and world > 1 else kern_gbs
    roofline = {"bound": "hbm", "achieved": kern_gbs, "peak": peak, "unit": "GB/s",
                "frac": (kern_gbs / peak) if kern_gbs else None, "traffic": None,
                "kernel": "fused_kernel (K1/K2/K3: update [+merge] [+bf16 pack])",
                "bytes_per_launch": tr["kernel_bytes"] / max(tr["kernel_launches"], 1),
                "ms_per_launch": tr["kernel_ms"] / max(tr["kernel_launches"], 1), "peak_source": peak_src}
    traffic, tsrc = ncu_traffic(f"fused_kernel/{P}x{G}/{a.mode}/B{a.B}S{a.S}")
    if traffic is not None:
        roofline["traffic"] = traffic
        roofline["traffic_source"] = tsrc
        # DRAM bytes ncu saw inside one launch / this run's launch time: part of each launch's
        # writes (~25 % for K1) is still dirty in L2 when the kernel ends and drains afterwards,
        # so "frac" (algorithmic bytes) can read a little above 1 while this stays below it.
        ms_launch = tr["kernel_ms"] / max(tr["kernel_launches"], 1)
        if ms_launch > 0:
            roofline["frac_in_kernel_dram"] = traffic / (ms_launch * 1e-3) / 1e9 / peak
    plain = [t for t, kk in zip(step_ms, kind_of) if kk == "plain"]
    p50_plain = max_over_ranks(statistics.median(plain), world) if plain else None
    if a.mode == "fused" and G > 1:
        # the fused node-tier kernel is NVLink-bound: per direction per GPU, (G-1)/G * 4n bytes of
        # gradient shards (peer reads) plus (G-1)/G * 4n bytes of parameter shards (peer stores)
        # (blocking batches split this over two launches: the node-tier kernel's gradient reads and the
        # average/re-publish kernel's parameter stores; the library traces each launch's own bytes)
        nvl_bytes = 2.0 * (G - 1) * 4.0 * daso.daso_padded_numel(n, G) / G
        nvl_gbs = tr["kernel_nvl_bytes"] / (tr["kernel_ms"] * 1e-3) / 1e9
        nvl_gbs = -max_over_ranks(-nvl_gbs, world)
        roofline = {"bound": "nvlink", "achieved": nvl_gbs, "peak": 770.0, "unit": "GB/s",
                    "frac": nvl_gbs / 770.0, "traffic": None,
                    "kernel": ("peer_tma_kernel (node gradient reduce over NVLink + update [+merge] [+pack] + "
                               "parameter all-gather by NVLink stores)"),
                    "bytes_per_launch": tr["kernel_nvl_bytes"] / max(tr["kernel_launches"], 1),
                    "bytes_def": "NVLink bytes per direction per GPU",
                    "ms_per_launch": tr["kernel_ms"] / max(tr["kernel_launches"], 1),
                    "peak_source": "measured peer copy 770 GB/s per direction (B200_PROFILING.md)",
                    "frac_at_p50_plain_step": (nvl_bytes / (p50_plain * 1e-3) / 1e9 / 770.0) if p50_plain else None,
                    "probe_ceiling_gbs": 660.0,
                    "frac_of_probe_ceiling": nvl_gbs / 660.0,
                    "probe": "tools/nvlink_kernels.cu tma_rw: this kernel's NVLink traffic pattern with no arithmetic, "
                             "no local x/v traffic and no barriers reaches 0.857 x 770 = 660 GB/s per direction at "
                             "G = 2 and 4 (profiles/r02/multi4_a/nvk_g*.jsonl)",
                    "hbm": roofline}
    phases = {k: (tr[k] / a.steps if k.endswith("_ms") else tr[k]) for k in tr}
    if tr["local_ms"] > 0:
        phases["local_busbw_gbs"] = tr["local_bytes"] / (tr["local_ms"] * 1e-3) / 1e9
    if tr["exch_ms"] > 0:
        phases["exch_gbs"] = tr["exch_bytes"] / (tr["exch_ms"] * 1e-3) / 1e9
        phases["hidden_fraction"] = max(0.0, 1.0 - tr["wait_ms"] / tr["exch_ms"])
    phases["p50_step_ms"] = statistics.median(step_ms)
    kinds = {}
    for kd in sorted(set(kind_of)):
        xs = [t for t, kk in zip(step_ms, kind_of) if kk == kd]
        kinds[kd] = {"count": len(xs), "ms_p10": pct(xs, 0.1), "ms_p50": statistics.median(xs), "ms_p90": pct(xs, 0.9)}
    kinds_max = {}
    for kd, d in kinds.items():   # max over ranks of each percentile
        kinds_max[kd] = {k: (max_over_ranks(v, world) if k.startswith("ms") else v) for k, v in d.items()}

    # ---- §8(d) hidden fraction of the global exchange (P > 1) -------------------------------------
    overlap = None
    if P > 1:
        nx = 1 if a.S > 0 else a.B          # exchanges issued per B-cycle
        overlap = {}
        if a.overlap_compute in ("sleep", "both"):
            overlap["sleep"] = overlap_cycles(ctx, a, g, g_src, stream, world, make_sleep(a.overlap_compute_ms), nx,
                                              t_ag)
        if a.overlap_compute in ("gemm", "both"):
            overlap["gemm"] = overlap_cycles(ctx, a, g, g_src, stream, world,
                                             make_compute_small(a.overlap_compute_ms, dev), nx, t_ag,
                                             cycles=max(a.cycles, a.gemm_cycles))

    # ---- e2e through the C ABI with host buffers (daso_step_host) -------------------------------
    e2e = None
    if not a.no_e2e:
        hg = torch.empty(n, dtype=torch.float32, pin_memory=True)
        hg.copy_(g_src[:n].cpu())
        for _ in range(3):
            ctx.step_host(hg, a.lr)
        barrier(world)
        torch.cuda.synchronize()
        k2 = a.e2e_steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k2):
            _, flag = ctx.step_host(hg, a.lr)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        te = max_over_ranks(e0.elapsed_time(e1), world) / k2
        e2e = {"value": 4.0 * n * world / (te * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": te,
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4,
               "what": "daso_step_host per batch: the step's gradients copied in from pinned host memory, the "
                       "whole sync path, the 4-byte non-finite flag (the step's result) copied back; the "
                       "parameters stay device-resident, as in training (the next forward reads them there)"}
    ctx.finalize()

    kernels = None
    vcb = None
    if world == 1 and not a.no_kernels:
        with ClockSampler(local) as kclk:
            kernels = kernel_table(n, peak)
        if not a.no_vcluster:
            with ClockSampler(local) as vclk:
                vcb = vcluster_block(n, a.B, a.S, peak, a.exchange)
            vcb["clocks"] = vclk.summary()
        kernels = {"n_params": n, "peak_gbs": peak, "peak_source": peak_src, "clocks": kclk.summary(),
                   "timing": "CUDA events on the launching stream around each launch, 256 MB L2 flush between "
                             "launches, 30 launches after 5 warm-up; achieved = algorithmic bytes / mean time",
                   "kernels": kernels}

    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "sync-path microbench (config 2): n=25,557,032 fp32 params, synthetic grads",
                       "n_params": n, "topology": f"{P}x{G}", "B": a.B, "S": a.S, "mode": a.mode, "exchange": a.exchange,
                       "wire": a.wire, "parallelism": f"daso {P} virtual nodes x {G} GPUs",
                       "l2": "flushed before every timed step (untimed read of a 256 MB buffer after the "
                             "gradient refresh); the inputs (x, v, g = 307 MB) also exceed the 126 MB L2",
                       "value_def": "4 B x n params x N GPUs / ms_per_step",
                       "timed_window": "per batch: daso_step on the compute stream (node tier, fused kernel, "
                                       "exchange issue and the wait at a merge); the side-stream all-gather "
                                       "overlaps the untimed refresh/flush between steps -- the full-cycle "
                                       "timing with the exchange inside the window is `overlap`",
                       "compute_ms_between_steps": a.compute_ms},
            "hidden_fraction": ({k: v["hidden_fraction"] for k, v in overlap.items()} if overlap else None),
            "step_kinds": kinds_max, "overlap": overlap, "kernels": kernels, "vcluster_2x4": vcb,
            "steps_dump": ({"ms": step_ms, "kind": kind_of} if a.dump_steps else None),
            "roofline": roofline, "phases": phases, "gpu_launches": launches_total,
            "gpu_launches_per_rank": tr["kernel_launches"],
            "clocks": clk.summary(), "e2e": e2e, "finite": finite}
    if world == 1 and not a.no_cpu:
        line["cpu_baseline"] = cpu_baseline(P, G, a.B, a.S, n, a.wire)
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
    try:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
