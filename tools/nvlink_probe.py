#!/usr/bin/env python
"""Measure NVLink peer-copy bandwidth on this box (one process, several GPUs): the
reference for the fused peer kernel's roofline.

    python tools/nvlink_probe.py [--gpus 2] [--mb 256]

* uni:  GPU0 -> GPU1 copy engine (cudaMemcpyPeerAsync via torch), GB/s per direction
* bidi: GPU0 -> GPU1 and GPU1 -> GPU0 at the same time, GB/s per direction
* ring-bidi (gpus >= 4): every GPU sends to its right neighbour and receives from its left,
  plus the reverse ring, all at once (each GPU's link carries both directions)
"""
import argparse
import json

import torch


def timed(fns, streams, iters=20):
    for f, s in zip(fns, streams):
        with torch.cuda.stream(s):
            f()
    for d in range(torch.cuda.device_count()):
        torch.cuda.synchronize(d)
    ev = []
    for s in streams:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev.append((e0, e1))
    for (e0, _), s in zip(ev, streams):
        e0.record(s)
    for _ in range(iters):
        for f, s in zip(fns, streams):
            with torch.cuda.stream(s):
                f()
    for (_, e1), s in zip(ev, streams):
        e1.record(s)
    for d in range(torch.cuda.device_count()):
        torch.cuda.synchronize(d)
    return max(e0.elapsed_time(e1) for e0, e1 in ev) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--mb", type=int, default=256)
    a = ap.parse_args()
    n = a.mb * (1 << 20) // 4
    G = min(a.gpus, torch.cuda.device_count())
    src = [torch.ones(n, device=f"cuda:{d}") for d in range(G)]
    dst = [torch.empty(n, device=f"cuda:{d}") for d in range(G)]
    dst2 = [torch.empty(n, device=f"cuda:{d}") for d in range(G)]
    st = [torch.cuda.Stream(device=d) for d in range(G)]
    st2 = [torch.cuda.Stream(device=d) for d in range(G)]
    out = {"bytes": 4 * n}
    ms = timed([lambda: dst[1].copy_(src[0], non_blocking=True)], [st[0]])
    out["uni_gbs"] = 4 * n / (ms * 1e-3) / 1e9
    ms = timed([lambda: dst[1].copy_(src[0], non_blocking=True), lambda: dst[0].copy_(src[1], non_blocking=True)],
               [st[0], st[1]])
    out["bidi_gbs_per_direction"] = 4 * n / (ms * 1e-3) / 1e9
    if G >= 4:
        fns, ss = [], []
        for d in range(G):
            r, l = (d + 1) % G, (d - 1) % G
            fns.append(lambda d=d, r=r: dst[r].copy_(src[d], non_blocking=True))
            ss.append(st[d])
            fns.append(lambda d=d, l=l: dst2[l].copy_(src[d], non_blocking=True))
            ss.append(st2[d])
        ms = timed(fns, ss)
        out["ring_bidi_gbs_per_direction"] = 2 * 4 * n / (ms * 1e-3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
