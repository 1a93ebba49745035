#!/usr/bin/env python
"""Per-kernel HBM roofline table for the fused DASO kernels at ResNet-50 size.

    python tools/kernel_bench.py [--n 25557032] [--iters 50] [--only K1,K3]

Each kernel is launched through the C ABI (daso_k_*) on resident buffers, timed
with CUDA events on the launching stream around each launch; between launches a
256 MB buffer is read (untimed) so every launch starts from a cold, clean L2.  achieved =
algorithmic bytes per launch / mean launch time.  Also the target
command for `ncu --set full` (use --iters 3).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=25_557_032)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--P", type=int, default=2)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    import torch
    import paper_2104_05588_b200 as daso

    n, P = a.n, a.P
    stride = daso.daso_padded_numel(n, 8)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(stride, device="cuda", generator=gen) * 0.02
    v = torch.zeros_like(x)
    g = torch.randn(stride, device="cuda", generator=gen) * 0.01
    slot = (torch.randn(max(P, 8), stride, device="cuda", generator=gen) * 0.02).to(torch.bfloat16)
    pk = torch.zeros(stride, dtype=torch.bfloat16, device="cuda")
    wb = 2
    cases = {
        "K1_update": (lambda: daso.daso_k_update(x, v, g, 1e-3, 0.9, 1e-4, 0.5), 20),
        "K2_update_pack": (lambda: daso.daso_k_update(x, v, g, 1e-3, 0.9, 1e-4, 0.5, pack_out=pk), 20 + wb),
        f"K3_update_merge_P{P}": (lambda: daso.daso_k_update_merge(x, v, g, 1e-3, 0.9, 1e-4, 0.5, slot[:P], 1), 20 + P * wb),
        f"K3_update_merge_pack_P{P}": (lambda: daso.daso_k_update_merge(x, v, g, 1e-3, 0.9, 1e-4, 0.5, slot[:P], 1,
                                                                         pack_out=pk), 20 + (P + 1) * wb),
        "K3_update_merge_P8": (lambda: daso.daso_k_update_merge(x, v, g, 1e-3, 0.9, 1e-4, 0.5, slot[:8], 1), 20 + 8 * wb),
        f"K4_average_P{P}": (lambda: daso.daso_k_average(x, slot[:P]), P * wb + 4),
        "K4_average_P4": (lambda: daso.daso_k_average(x, slot[:4]), 4 * wb + 4),
        "pack_only": (lambda: daso.daso_k_pack(x, pk), 4 + wb),
    }
    xs = x[:n]
    # restrict to n elements (the ABI takes numel from x)
    x, v, g = x[:n], v[:n], g[:n]
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")   # 256 MB > 126 MB L2
    only = set(a.only.split(",")) if a.only else None
    rows = {}
    for name, (fn, bpp) in cases.items():
        if only and not any(name.startswith(o) for o in only):
            continue
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.iters)]
        for e0, e1 in ev:
            flush.sum()                 # evict L2 with clean lines (untimed; no dirty write-back to pay)
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        ms = sum(e0.elapsed_time(e1) for e0, e1 in ev) / a.iters
        gbs = bpp * n / (ms * 1e-3) / 1e9
        rows[name] = {"bytes_per_param": bpp, "us": ms * 1e3, "GB/s": gbs, "frac_of_measured_peak": gbs / peak}
    del xs
    print(json.dumps({"n": n, "peak_gbs": peak, "kernels": rows}, indent=1))


if __name__ == "__main__":
    main()
