#!/bin/bash
# round 2, 4-GPU call D: copy-engine exchange parity + overlap vs NCCL; NVLink probe tile sizes
O=gpurun_out/r02m4d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -k "copy_engine or full_size" -q -p no:cacheprovider > $O/pytest_ce.txt 2>&1; echo rc=$? >> $O/pytest_ce.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=29950
for ex in ce nccl; do for c in 1 20; do
  port=$((port+1))
  timeout 400 $T --nproc-per-node 4 --master-port $port bench.py --gpus 4 --steps 200 --warmup 10 --no-e2e \
     --exchange $ex --overlap-compute-ms $c --cycles 20 > $O/ov_${ex}_c$c.json 2> $O/ov_${ex}_c$c.err
done; done
for rep in 1 2 3; do for topo in 2x2 4x1; do
  port=$((port+1))
  timeout 400 $T --nproc-per-node 4 --master-port $port bench.py --gpus 4 --topology $topo --steps 200 --warmup 10 \
     --exchange ce --cycles 10 > $O/ce_${topo}_$rep.json 2> $O/ce_${topo}_$rep.err
done; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/nvk tools/nvlink_kernels.cu
for t in 2048 4096 8192; do CUDA_VISIBLE_DEVICES=0,1 timeout 120 /tmp/nvk 25557056 132 0 $t > $O/nvk_g2_t$t.jsonl 2>&1; done
tail -3 $O/pytest_ce.txt
