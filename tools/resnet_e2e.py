#!/usr/bin/env python
"""End-to-end ResNet-50 training throughput on synthetic ImageNet-shaped batches
(SURVEY §8(d) config 3): DASO through libdaso.so vs a synchronous all-reduce
(the same library with one virtual node, P = 1, G = W) vs torch DDP + torch SGD.

    torchrun --nproc-per-node N tools/resnet_e2e.py --impl daso|sync|ddp [--batch 256]

Model: torchvision resnet50 (25,557,032 params, 161 tensors), random init,
channels_last, bf16 autocast for forward/backward only; fp32 master params,
grads and momentum in the flat buckets (K0 gather at bind, params and .grad are
views).  Data: per-rank seeded N(0,1) images [batch, 3, 224, 224] and uniform
labels, resident on the GPU.  SGD 0.9 / 1e-4; DASO B = 4, S = 1 with
warm-up 1 / cool-down 1 epochs of 10 steps.  Prints one JSON line (rank 0):
samples/s over all ranks (max-over-ranks time), and the per-step sync-path time
from the library's CUDA-event tracing.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=["daso", "sync", "ddp"], default="daso")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--gpus-per-node", type=int, default=0, help="DASO G (default: 2 if world >= 4 else 1)")
    ap.add_argument("--mode", default="faithful")
    ap.add_argument("--lr", type=float, default=0.1)
    a = ap.parse_args()

    import torch
    import torch.distributed as dist
    import torchvision

    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo")
    torch.manual_seed(0)                       # identical init on every rank (R17)
    model = torchvision.models.resnet50().to(dev).to(memory_format=torch.channels_last)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    images = torch.randn(a.batch, 3, 224, 224, device=dev, generator=gen).to(memory_format=torch.channels_last)
    labels = torch.randint(0, 1000, (a.batch,), device=dev, generator=gen)
    loss_fn = torch.nn.CrossEntropyLoss()

    ctx = None
    if a.impl == "ddp":
        if world > 1:
            pg = dist.new_group(backend="nccl")
            net = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local], process_group=pg)
        else:
            net = model
        opt = torch.optim.SGD(model.parameters(), lr=a.lr, momentum=0.9, weight_decay=1e-4)
    else:
        import paper_2104_05588_b200 as daso
        if a.impl == "sync":
            P, G, B, S = 1, world, 1, 0
        else:
            G = a.gpus_per_node or (2 if world >= 4 else 1)
            P, B, S = world // G, 4, 1
        uid = daso.rendezvous_unique_id() if world > 1 else daso.daso_get_unique_id()
        ctx = daso.daso_init(world, G, B, S, rank=rank, uid=uid, warmup_epochs=1, cooldown_epochs=1,
                             total_epochs=1000, steps_per_epoch=10 * 4, mode=a.mode)
        flat = daso.FlatParams(model.parameters(), gpus_per_node=G)
        ctx.bind(flat.x, flat.g, flat.v, flat.n)
        net = model

    def step():
        if ctx is None:
            opt.zero_grad(set_to_none=False)
        else:
            flat.g.zero_()
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = loss_fn(net(images), labels)
        loss.backward()
        if ctx is None:
            opt.step()
        else:
            ctx.step(a.lr)
        return loss

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if ctx is not None:
        ctx.trace_read(reset=True)
        ctx.trace_enable(True)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    out = {"workload": "resnet50 synthetic 224x224 (config 3)", "impl": a.impl, "n_gpus": world,
           "batch_per_gpu": a.batch, "steps": a.steps, "ms_per_step": ms / a.steps,
           "samples_per_s": a.batch * world * a.steps / (ms * 1e-3), "loss": float(loss.item())}
    if ctx is not None:
        tr = ctx.trace_read(reset=True)
        sync_ms = (tr["kernel_ms"] + tr["local_ms"] + tr["node_ms"] + tr["wait_ms"]) / a.steps
        out.update({"topology": f"{ctx.P}x{ctx.G}", "mode": a.mode, "sync_path_ms_per_step": sync_ms,
                    "sync_share": sync_ms / (ms / a.steps), "finite": ctx.check_finite()})
        ctx.finalize()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
