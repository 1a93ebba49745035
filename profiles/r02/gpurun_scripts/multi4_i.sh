#!/bin/bash
# round 2, 4-GPU call I (final): the whole GPU suite on 4 GPUs with the final library; default bench lines N=2, N=4
O=gpurun_out/r02m4i; mkdir -p $O
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/pytest_gpu_4gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu_4gpu.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $T --nproc-per-node 2 --master-port 30901 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err
timeout 600 $T --nproc-per-node 4 --master-port 30902 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err
tail -3 $O/pytest_gpu_4gpu.txt
