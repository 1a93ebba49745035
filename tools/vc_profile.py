#!/usr/bin/env python
"""ncu target for the fused node-tier kernel on ONE GPU: a virtual cluster (daso_vcluster_*)
at the sync-path microbench size (n = 25,557,032) runs a few DASO batches, so `ncu --set full
-k regex:peer_` captures peer_ws_kernel / peer_tma_kernel launches with their counters.  The
peers' buffers are on the same GPU here, so the traffic is HBM instead of NVLink: the capture
shows the kernel's own cost (instructions, stalls, shared memory, bulk-copy issue) and its DRAM
bytes per launch, not the link behaviour.  Also prints CUDA-event times per launch kind.

    python tools/vc_profile.py [--topology 1x2] [--steps 6]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--topology", default="1x2")
    ap.add_argument("--n", type=int, default=25_557_032)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--B", type=int, default=4)
    ap.add_argument("--S", type=int, default=1, help="S = 0 with B = 1: every batch a blocking sync (OP_NOX "
                    "node-tier kernel + average/re-publish kernel)")
    ap.add_argument("--exchange", choices=["nccl", "ce"], default="nccl")
    a = ap.parse_args()
    import torch
    import paper_2104_05588_b200 as daso
    P, G = (int(v) for v in a.topology.split("x"))
    torch.cuda.set_device(0)
    vc = daso.VCluster(P * G, G, a.B, a.S, a.n, total_epochs=1, steps_per_epoch=max(a.B, 1) << 20, mode="fused",
                       exchange=a.exchange)
    gen = torch.Generator(device="cuda").manual_seed(0)
    x0 = torch.randn(a.n, device="cuda", generator=gen) * 0.02
    for r in range(P * G):
        vc.x(r)[:a.n] = x0
        vc.g(r)[:a.n] = torch.randn(a.n, device="cuda", generator=gen) * 0.01
        vc.rank(r).trace_enable(True)
    torch.cuda.synchronize()
    for _ in range(a.steps):
        vc.step(0.01)
    torch.cuda.synchronize()
    tr = [vc.rank(r).trace_read() for r in range(P * G)]
    vc.destroy()
    k = sum(t["kernel_launches"] for t in tr)
    ms = sum(t["kernel_ms"] for t in tr)
    by = sum(t["kernel_bytes"] for t in tr)
    print(json.dumps({"topology": a.topology, "B": a.B, "S": a.S, "exchange": a.exchange, "n": a.n, "launches": k, "us_per_launch": ms / max(k, 1) * 1e3,
                      "hbm_bytes_per_launch": by / max(k, 1), "hbm_gbs": by / (ms * 1e-3) / 1e9 if ms else None}))


if __name__ == "__main__":
    main()
