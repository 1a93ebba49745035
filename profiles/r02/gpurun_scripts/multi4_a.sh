#!/bin/bash
# round 2, 4-GPU call A: NVLink ceiling probes, NCCL bars, config-2 sweep at 2x2 and 1x4
O=gpurun_out/r02m4a; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/nvk tools/nvlink_kernels.cu
timeout 120 /tmp/nvk > $O/nvk_g4.jsonl 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 120 /tmp/nvk > $O/nvk_g2.jsonl 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 120 /tmp/nvk 25557056 132 3 > $O/nvk_g2_ns3.jsonl 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 120 /tmp/nvk 25557056 148 0 > $O/nvk_g2_148.jsonl 2>&1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for algo in NVLS Ring; do
  NCCL_ALGO=$algo timeout 300 $T --nproc-per-node 4 --master-port 29611 tools/nccl_bar.py --tag $algo > $O/nccl_$algo.json 2> $O/nccl_$algo.err
done
timeout 300 $T --nproc-per-node 2 --master-port 29612 tools/nccl_bar.py --tag default_g2 > $O/nccl_g2.json 2> $O/nccl_g2.err
B="timeout 400 $T --nproc-per-node 4 --master-port 29613 bench.py --gpus 4 --steps 100 --warmup 10 --no-e2e"
for bs in "1 1" "2 1" "4 1" "8 2" "1 0"; do
  set -- $bs
  $B --B $1 --S $2 > $O/bench_2x2_B$1S$2.json 2> $O/bench_2x2_B$1S$2.err
done
$B --topology 1x4 > $O/bench_1x4.json 2> $O/bench_1x4.err
$B --topology 4x1 > $O/bench_4x1.json 2> $O/bench_4x1.err
$B --mode faithful > $O/bench_2x2_faithful.json 2> $O/bench_2x2_faithful.err
$B --mode nvls --topology 1x4 > $O/bench_1x4_nvls.json 2> $O/bench_1x4_nvls.err
ls -la $O
