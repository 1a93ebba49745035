"""Worker: a small CNN trained with DASO through FlatParams, once with the node all-reduce
inside daso_step and once with OverlappedLocalSync (bucketed all-reduce launched from
gradient hooks during backward, daso_step_ex(grads_reduced)) — SURVEY §8(f) N2.
Deterministic backward (torch.use_deterministic_algorithms, cuDNN deterministic).  Each
run records every step's local (pre-sync) gradient of this rank — in the overlapped run
by a hook registered before OverlappedLocalSync's, so the copy is enqueued before the
bucket's all-reduce — and the parameters after every step; tests/test_gpu_multi.py feeds
the recorded gradients to the CPU oracle and compares both trajectories with it."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

LR, MU, WD, B, S, SPE = 0.05, 0.9, 1e-4, 4, 1, 64


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
    x0 = flat.x[:flat.n].cpu().numpy().copy()
    ctx = daso.daso_init(world, G, B, S, rank=rank, uid=uid, steps_per_epoch=SPE, momentum=MU, weight_decay=WD,
                         wire="fp32")
    ctx.bind(flat.x, flat.g, flat.v, flat.n)
    rec = torch.zeros_like(flat.g)

    def recorder(o, k):
        def hook(_p):
            rec[o:o + k].copy_(flat.g[o:o + k])
        return hook
    # recording hooks first: they run before OverlappedLocalSync's hook of the same parameter
    for p, o in zip(flat.params, flat.offsets):
        p.register_post_accumulate_grad_hook(recorder(o, p.numel()))
    ov = daso.OverlappedLocalSync(ctx, flat, bucket_mb=0.05) if overlap else None
    gen = torch.Generator(device=dev).manual_seed(100 + rank)
    trace, grads = [], []
    for k in range(steps):
        xb = torch.randn(8, 3, 16, 16, device=dev, generator=gen)
        flat.g.zero_()
        m(xb).square().mean().backward()
        if ov:
            ov.step(LR)
        else:
            ctx.step(LR)
        grads.append(rec[:flat.n].cpu().numpy().copy())
        trace.append(flat.x[:flat.n].cpu().numpy().copy())
    n_buckets = len(ov.buckets) if ov else 0
    assert ctx.check_finite()
    ctx.finalize()
    return np.stack(trace), np.stack(grads), x0, n_buckets


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--G", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")
    import torch
    import torch.distributed as dist
    torch.use_deterministic_algorithms(True)
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("gloo")
    from paper_2104_05588_b200 import rendezvous_unique_id
    t0, g0, x0, _ = run(False, rank, world, a.G, rendezvous_unique_id(), a.steps)
    t1, g1, _, nb = run(True, rank, world, a.G, rendezvous_unique_id(), a.steps)
    os.makedirs(a.out, exist_ok=True)
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), plain=t0, overlap=t1, grads_plain=g0, grads_overlap=g1, x0=x0,
             n_buckets=nb)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
