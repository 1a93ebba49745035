#!/usr/bin/env python
"""End-to-end training throughput on synthetic batches shaped like the paper's two
workloads: ResNet-50 / ImageNet 224x224 and a hierarchical
multi-scale attention segmentation net / Cityscapes 1024x2048 (config 4).
DASO through libdaso.so vs a synchronous all-reduce (the same library with one
virtual node, P = 1, G = W) vs torch DDP + torch SGD.

    torchrun --nproc-per-node N tools/e2e_train.py --model resnet50|hmsa --impl daso|sync|ddp

HMSA stand-in (HRNet-OCR has no code or weights here): Tao et al.'s hierarchical
multi-scale attention on a DeepLabV3-ResNet-50 trunk — the shared trunk + head predict
at scales 0.5 and 1.0, an attention head on the 0.5-scale features weights the two
(p = a * up(p_0.5) + (1 - a) * p_1.0), 19 classes, cross-entropy, batch-norm
synchronised within the node-local process group.

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


def HMSA(classes: int):
    import torch
    import torch.nn.functional as F
    import torchvision

    class _HMSA(torch.nn.Module):
        def __init__(self):
            super().__init__()
            seg = torchvision.models.segmentation.deeplabv3_resnet50(weights=None, weights_backbone=None,
                                                                     num_classes=classes, aux_loss=False)
            self.backbone, self.head = seg.backbone, seg.classifier
            self.attn = torch.nn.Sequential(torch.nn.Conv2d(2048, 256, 3, padding=1, bias=False),
                                            torch.nn.BatchNorm2d(256), torch.nn.ReLU(inplace=True),
                                            torch.nn.Conv2d(256, 1, 1), torch.nn.Sigmoid())

        def forward(self, x):
            lo = F.interpolate(x, scale_factor=0.5, mode="bilinear", align_corners=False)
            f_lo = self.backbone(lo)["out"]
            p_lo, att = self.head(f_lo), self.attn(f_lo)
            p_hi = self.head(self.backbone(x)["out"])
            size = p_hi.shape[-2:]
            p = F.interpolate(att * p_lo, size=size, mode="bilinear", align_corners=False) + \
                (1 - F.interpolate(att, size=size, mode="bilinear", align_corners=False)) * p_hi
            return F.interpolate(p, size=x.shape[-2:], mode="bilinear", align_corners=False)

    return _HMSA()


def train_loop(a, ctx, flat, net, images, labels, loss_fn, world, rank, overlap=None):
    """The whole DASO control loop on real (synthetic-data) losses: per epoch, the mean training
    loss over all ranks feeds the plateau detector (daso_plateau_*); a plateau decays the
    LR (daso_lr_at) and is passed to the next epoch's first daso_step, which halves or
    resets B and S.  Prints one JSON record per epoch on rank 0."""
    import torch
    import torch.distributed as dist
    import paper_2104_05588_b200 as daso
    det = daso.PlateauDetector(a.patience, a.threshold)
    n_plateaus, plateau_next, k = 0, 0, 0
    base_lr = a.lr / world                      # peak = base * world
    for e in range(a.train_epochs):
        total = torch.zeros((), device=images.device)
        for i in range(a.steps_per_epoch):
            lr = daso.daso_lr_at(k, a.steps_per_epoch, base_lr, world, a.lr_warmup_epochs, a.lr_factor, n_plateaus)
            flat.g.zero_()
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = loss_fn(net(images), labels)
            loss.backward()
            plateau = plateau_next if i == 0 else 0
            rec = overlap.step(lr, plateau) if overlap is not None else ctx.step(lr, plateau)
            total += loss.detach().float()
            k += 1
        mean = total / a.steps_per_epoch
        if world > 1:
            t = torch.tensor([float(mean.item())], dtype=torch.float64)
            dist.all_reduce(t)
            mean_loss = float(t.item()) / world
        else:
            mean_loss = float(mean.item())
        plateau_next = det.update(mean_loss)
        n_plateaus += plateau_next
        if rank == 0:
            print(json.dumps({"epoch": e, "mean_loss": mean_loss, "lr": lr, "plateau": plateau_next,
                              "phase": rec["phase"], "B": rec["B"], "S": rec["S"], "syncs": rec["n_syncs"]}),
                  flush=True)
    if not ctx.check_finite():
        raise RuntimeError("non-finite parameters")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", choices=["resnet50", "hmsa"], default="resnet50")
    ap.add_argument("--impl", choices=["daso", "sync", "ddp"], default="daso")
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (default 256 resnet50, 2 hmsa)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--gpus-per-node", type=int, default=0,
                    help="DASO G (default: 2 if world >= 4 else 1); also the node group of SyncBN")
    ap.add_argument("--mode", default="faithful")
    ap.add_argument("--exchange", choices=["nccl", "ce"], default="nccl", help="global-tier transport")
    ap.add_argument("--lr", type=float, default=0.1)
    ap.add_argument("--overlap", action="store_true",
                    help="faithful mode: node all-reduce in buckets overlapped with backward (N2)")
    ap.add_argument("--train-epochs", type=int, default=0,
                    help="instead of timing: train this many epochs with the full loop of P:97-99/P:162/P:172 — "
                         "epoch-mean loss -> plateau detector -> LR decay and DASO B/S halving (N4)")
    ap.add_argument("--steps-per-epoch", type=int, default=8)
    ap.add_argument("--timed-phase", choices=["cycling", "warmup"], default="cycling",
                    help="DASO phase of the timed steps (P:97): cycling (non-blocking exchange every B batches) "
                         "or warm-up (a blocking sync every batch)")
    ap.add_argument("--patience", type=int, default=2)
    ap.add_argument("--threshold", type=float, default=0.01)
    ap.add_argument("--lr-warmup-epochs", type=int, default=1)
    ap.add_argument("--lr-factor", type=float, default=0.5)
    a = ap.parse_args()
    if a.train_epochs and a.impl == "ddp":
        raise SystemExit("--train-epochs drives the DASO schedule: use --impl daso or sync")
    if a.overlap and a.mode != "faithful":
        raise SystemExit("--overlap needs --mode faithful (bucketed node all-reduce)")

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
    G_node = a.gpus_per_node or (2 if world >= 4 else 1)
    if a.impl == "sync":
        G_node = world
    if a.impl == "ddp":
        G_node = min(G_node, world)
    torch.manual_seed(0)                       # identical init on every rank (R17)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    if a.model == "resnet50":
        a.batch = a.batch or 256
        model = torchvision.models.resnet50()
        images = torch.randn(a.batch, 3, 224, 224, device=dev, generator=gen)
        labels = torch.randint(0, 1000, (a.batch,), device=dev, generator=gen)
    else:
        a.batch = a.batch or 2
        model = HMSA(19)
        images = torch.randn(a.batch, 3, 1024, 2048, device=dev, generator=gen)
        labels = torch.randint(0, 19, (a.batch, 1024, 2048), device=dev, generator=gen)
        if world > 1:   # node-local SyncBN
            groups = [dist.new_group(list(range(j * G_node, (j + 1) * G_node)), backend="nccl")
                      for j in range(world // G_node)]
            model = torch.nn.SyncBatchNorm.convert_sync_batchnorm(model, process_group=groups[rank // G_node])
    model = model.to(dev).to(memory_format=torch.channels_last)
    images = images.to(memory_format=torch.channels_last)
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
            G = G_node
            P, B, S = world // G, 4, 1
        uid = daso.rendezvous_unique_id() if world > 1 else daso.daso_get_unique_id()
        if a.train_epochs:
            ctx = daso.daso_init(world, G, B, S, rank=rank, uid=uid, warmup_epochs=1, cooldown_epochs=1,
                                 total_epochs=max(a.train_epochs, 2), steps_per_epoch=a.steps_per_epoch, mode=a.mode,
                                 exchange=a.exchange)
        else:   # the timed steps all fall in the first epoch: warm-up (blocking) or, without one, cycling
            ctx = daso.daso_init(world, G, B, S, rank=rank, uid=uid,
                                 warmup_epochs=1 if a.timed_phase == "warmup" else 0, cooldown_epochs=1,
                                 total_epochs=1000, steps_per_epoch=4 * (a.warmup + a.steps + 4), mode=a.mode,
                                 exchange=a.exchange)
        if a.mode == "fused" and "expandable_segments:True" in os.environ.get("PYTORCH_CUDA_ALLOC_CONF", ""):
            # cuMem-backed torch memory cannot be exported by CUDA IPC: let the library own the buckets
            flat = daso.FlatParams(model.parameters(), gpus_per_node=G, ctx=ctx)
        else:
            flat = daso.FlatParams(model.parameters(), gpus_per_node=G)
            ctx.bind(flat.x, flat.g, flat.v, flat.n)
        overlap = daso.OverlappedLocalSync(ctx, flat) if a.overlap else None
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
        elif overlap is not None:
            overlap.step(a.lr)
        else:
            ctx.step(a.lr)
        return loss

    if a.train_epochs and ctx is not None:
        train_loop(a, ctx, flat, net, images, labels, loss_fn, world, rank, overlap)
        ctx.finalize()
        if world > 1:
            dist.destroy_process_group()
        return

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
    wl = {"resnet50": "resnet50 synthetic 224x224 (config 3)",
          "hmsa": "hierarchical multi-scale attention seg. synthetic 1024x2048, 19 classes (config 4)"}[a.model]
    out = {"workload": wl, "impl": a.impl, "n_gpus": world, "params": sum(p.numel() for p in model.parameters()),
           "batch_per_gpu": a.batch, "steps": a.steps, "ms_per_step": ms / a.steps,
           "samples_per_s": a.batch * world * a.steps / (ms * 1e-3), "loss": float(loss.item())}
    if ctx is not None:
        tr = ctx.trace_read(reset=True)
        sync_ms = (tr["kernel_ms"] + tr["local_ms"] + tr["node_ms"] + tr["wait_ms"]) / a.steps
        out.update({"topology": f"{ctx.P}x{ctx.G}", "mode": a.mode, "exchange": a.exchange, "overlap": a.overlap,
                    "timed_phase": a.timed_phase if a.impl == "daso" else "sync every batch",
                    "sync_path_ms_per_step": sync_ms,
                    "sync_share": sync_ms / (ms / a.steps), "finite": ctx.check_finite()})
        ctx.finalize()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
