"""Per-rank worker for the toy DASO config on real GPUs.

Run under torchrun (one process per GPU; world = P*G virtual-node ranks):
    python -m torch.distributed.run --nproc-per-node W tests/mp_toy.py --P 2 --G 2 --out DIR ...
or in-process for world = 1 via run_toy().  Each rank computes its toy-regression
gradient with torch on its GPU (TF32 off), calls daso_step through the C ABI, and
saves its parameter trace, schedule records and node-replica checksums to
DIR/rank{r}.npz; tests/test_gpu_multi.py compares them with the CPU oracle.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synthetic  # noqa: E402


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=2)
    ap.add_argument("--G", type=int, default=2)
    ap.add_argument("--B", type=int, default=4)
    ap.add_argument("--S", type=int, default=1)
    ap.add_argument("--dim", dest="d", type=int, default=1000)
    ap.add_argument("--b", type=int, default=32)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--mu", type=float, default=0.9)
    ap.add_argument("--wd", type=float, default=1e-4)
    ap.add_argument("--warmup", type=int, default=0)
    ap.add_argument("--cooldown", type=int, default=0)
    ap.add_argument("--epochs", type=int, default=1)
    ap.add_argument("--spe", type=int, default=20)
    ap.add_argument("--flags", type=str, default="")
    ap.add_argument("--wire", default="bf16")
    ap.add_argument("--mode", default="faithful")
    ap.add_argument("--split", action="store_true", help="drive the split API instead of daso_step")
    ap.add_argument("--kernel", default="", help="ldg | tma: fused-kernel data path (daso_kernel_impl)")
    ap.add_argument("--exchange", default="nccl", help="nccl | ce (copy-engine group exchange)")
    ap.add_argument("--alloc", action="store_true", help="daso_alloc_bind instead of torch buckets")
    ap.add_argument("--out", required=True)
    return ap.parse_args(argv)


def run_toy(a, rank: int = 0, world: int = 1, uid: bytes | None = None):
    import torch
    import paper_2104_05588_b200 as daso
    from paper_2104_05588_b200 import Schedule

    if a.kernel:
        daso.daso_kernel_impl(a.kernel)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    dev = torch.device("cuda", torch.cuda.current_device())
    flags = [int(c) for c in a.flags] if a.flags else []
    uid = uid if uid is not None else daso.daso_get_unique_id()
    ctx = daso.daso_init(world, a.G, a.B, a.S, rank=rank, uid=uid, warmup_epochs=a.warmup,
                         cooldown_epochs=a.cooldown, total_epochs=a.epochs, steps_per_epoch=a.spe,
                         momentum=a.mu, weight_decay=a.wd, wire=a.wire, mode=a.mode, exchange=a.exchange)
    n_pad = daso.daso_padded_numel(a.d, a.G)
    if a.alloc:                                                   # library-owned (cudaMalloc) buckets
        x, g, v = ctx.alloc_bind(a.d)                             # zeroed: x0 = 0 on every rank (R17)
    else:
        x = torch.zeros(n_pad, dtype=torch.float32, device=dev)  # x0 = 0, identical on every rank (R17)
        g = torch.zeros_like(x)
        v = torch.zeros_like(x)
        ctx.bind(x, g, v, a.d)
    sched = Schedule(a.B, a.S, a.warmup, a.cooldown, a.epochs, a.spe, a.G) if a.split else None
    trace, recs, cks = [], [], []
    ck = torch.zeros(1, dtype=torch.int64, device=dev)
    for k in range(a.steps):
        X, y = synthetic.toy_batch(a.d, a.b, rank, k)
        Xt, yt = torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev)
        w = x[:a.d]
        g[:a.d] = Xt.T @ (Xt @ w - yt) / a.b                       # toy gradient (the "backward")
        plateau = 0
        if k > 0 and k % a.spe == 0 and k // a.spe - 1 < len(flags):
            plateau = flags[k // a.spe - 1]
        if a.split:
            r = sched.next(plateau)
            ctx.local_sync()
            if r["merge"]:
                ctx.local_update(a.lr)
                ctx.global_merge()
            else:
                ctx.local_update(a.lr)
            if r["send"]:
                ctx.global_send(r["send_group"], 0 if r["blocking"] else r["S"])
        else:
            r = ctx.step(a.lr, plateau)
        recs.append([r[f] for f in sorted(r)])
        trace.append(x[:a.d].cpu().numpy().copy())
        daso.daso_k_checksum(x[:a.d], ck)
        cks.append(int(ck.item()))
    assert ctx.check_finite()
    ctx.finalize()
    os.makedirs(a.out, exist_ok=True)
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), trace=np.stack(trace), recs=np.array(recs, np.int64),
             rec_fields=np.array(sorted(r)), cks=np.array(cks, dtype=np.uint64))
    return trace


def main():
    a = parse()
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("gloo")
    from paper_2104_05588_b200 import rendezvous_unique_id
    uid = rendezvous_unique_id()
    run_toy(a, rank, world, uid)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"ok": True, "world": world}))


if __name__ == "__main__":
    main()
