"""Worker: a small CNN trained with DASO through FlatParams, once with the node all-reduce
inside daso_step and once with OverlappedLocalSync (bucketed all-reduce launched from
gradient hooks during backward, daso_step_ex(grads_reduced)).  Saves both parameter
traces to DIR/rank{r}.npz for tests/test_gpu_multi.py."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def model():
    import torch
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Conv2d(3, 32, 3), torch.nn.ReLU(), torch.nn.Conv2d(32, 32, 3),
                               torch.nn.ReLU(), torch.nn.Flatten(), torch.nn.Linear(32 * 12 * 12, 64),
                               torch.nn.ReLU(), torch.nn.Linear(64, 10))


def run(overlap, rank, world, G, uid, steps):
    import torch
    import paper_2104_05588_b200 as daso
    dev = torch.device("cuda", torch.cuda.current_device())
    m = model().to(dev)
    flat = daso.FlatParams(m.parameters(), gpus_per_node=G)
    ctx = daso.daso_init(world, G, 4, 1, rank=rank, uid=uid, steps_per_epoch=64, wire="fp32")
    ctx.bind(flat.x, flat.g, flat.v, flat.n)
    ov = daso.OverlappedLocalSync(ctx, flat, bucket_mb=0.05) if overlap else None
    gen = torch.Generator(device=dev).manual_seed(100 + rank)
    trace = []
    for k in range(steps):
        xb = torch.randn(8, 3, 16, 16, device=dev, generator=gen)
        flat.g.zero_()
        m(xb).square().mean().backward()
        if ov:
            ov.step(0.05)
        else:
            ctx.step(0.05)
        trace.append(flat.x[:flat.n].cpu().numpy().copy())
    n_buckets = len(ov.buckets) if ov else 0
    ctx.finalize()
    return np.stack(trace), n_buckets


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--G", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("gloo")
    from paper_2104_05588_b200 import rendezvous_unique_id
    t0, _ = run(False, rank, world, a.G, rendezvous_unique_id(), a.steps)
    t1, nb = run(True, rank, world, a.G, rendezvous_unique_id(), a.steps)
    os.makedirs(a.out, exist_ok=True)
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), plain=t0, overlap=t1, n_buckets=nb)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
