"""Worker: the sync-path microbench at FULL size, n = 25,557,032,
in bench.py's launch configuration, for a few steps with the seeded per-rank gradients of
synthetic.microbench_grad(n, rank, step); saves x at a fixed sample of indices after every
step.  DASO is elementwise in the parameters once the gradients are given, so the CPU
oracle reproduces exactly these elements by simulating only the sampled indices
(tests/test_gpu_multi.py::test_full_size_microbench_sampled)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synthetic  # noqa: E402

N = 25_557_032


def sample_indices(n=N, k=20000, seed=11):
    idx = np.sort(np.random.default_rng(seed).choice(n, k, replace=False))
    return np.unique(np.concatenate([idx, [0, 1, n - 2, n - 1]]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--G", type=int, default=2)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--mode", default="fused")
    ap.add_argument("--wire", default="bf16")
    ap.add_argument("--exchange", default="nccl")
    ap.add_argument("--alloc", action="store_true", help="daso_alloc_bind instead of torch buckets")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    import paper_2104_05588_b200 as daso
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("gloo")
    uid = daso.rendezvous_unique_id()
    ctx = daso.daso_init(world, a.G, 4, 1, rank=rank, uid=uid, total_epochs=1, steps_per_epoch=4 << 20,
                         momentum=0.9, weight_decay=1e-4, wire=a.wire, mode=a.mode, exchange=a.exchange)
    n_pad = daso.daso_padded_numel(N, a.G)
    if a.alloc:                                   # library-owned (cudaMalloc) buckets
        x, g, v = ctx.alloc_bind(N)
    else:
        x = torch.zeros(n_pad, dtype=torch.float32, device=dev)
        g = torch.zeros_like(x)
        v = torch.zeros_like(x)
        ctx.bind(x, g, v, N)
    x[:N] = torch.from_numpy(synthetic.microbench_x0(N)).to(dev)
    idx = torch.from_numpy(sample_indices()).to(dev)
    trace = []
    for k in range(a.steps):
        g[:N] = torch.from_numpy(synthetic.microbench_grad(N, rank, k)).to(dev)
        ctx.step(0.1)
        trace.append(x[idx].cpu().numpy())
    assert ctx.check_finite()
    ctx.finalize()
    os.makedirs(a.out, exist_ok=True)
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), trace=np.stack(trace))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
