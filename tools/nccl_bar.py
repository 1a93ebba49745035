#!/usr/bin/env python
"""NCCL's own node-tier collectives on this box, as the bar for the fused / NVLS kernels
(DESIGN.md §7): all-reduce, reduce-scatter and all-gather of the ResNet-50 gradient bucket
(n = 25,557,056 fp32) over G GPUs, timed with CUDA events, max over ranks, nccl-tests bus
bandwidth convention (AR 2(G-1)/G S, RS/AG (G-1)/G S per rank).  Run once per algorithm:

    NCCL_ALGO=NVLS torchrun --nproc-per-node 4 tools/nccl_bar.py --tag nvls
    NCCL_ALGO=Ring torchrun --nproc-per-node 4 tools/nccl_bar.py --tag ring
"""
import argparse
import json
import os

import torch
import torch.distributed as dist


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=25_557_056)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--tag", default=os.environ.get("NCCL_ALGO", "default"))
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    n = a.n // world * world
    buf = torch.randn(n, device="cuda")
    shard = torch.empty(n // world, device="cuda")
    S = 4.0 * n
    ops = {
        "all_reduce": (lambda: dist.all_reduce(buf), 2.0 * (world - 1) / world * S),
        "reduce_scatter": (lambda: dist.reduce_scatter_tensor(shard, buf), (world - 1) / world * S),
        "all_gather": (lambda: dist.all_gather_into_tensor(buf, shard), (world - 1) / world * S),
    }
    out = {"tag": a.tag, "world": world, "n": n, "bytes": S}
    for name, (fn, bus) in ops.items():
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / a.iters], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        out[name] = {"us": ms * 1e3, "busbw_gbs": bus / (ms * 1e-3) / 1e9, "bus_bytes": bus}
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
