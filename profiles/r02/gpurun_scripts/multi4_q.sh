#!/bin/bash
# round 2 (session 2), 4-GPU call Q: ResNet-50 end-to-end (config 3, 256/GPU) at 2x2 with the final library,
# DASO timed in the cycling phase (non-blocking exchange every B = 4 batches) and in the warm-up phase (a
# blocking sync every batch: what session 1's e2e lines timed, its 38 steps falling inside the 40-step warm-up
# epoch), beside the library's synchronous all-reduce and torch DDP
O=gpurun_out/r02m4q; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30700
for impl in "--impl daso --mode fused --exchange ce --timed-phase cycling" "--impl daso --mode fused --exchange ce --timed-phase warmup" "--impl sync --mode fused" "--impl ddp"; do
  port=$((port+1))
  timeout 600 $T --nproc-per-node 4 --master-port $port tools/e2e_train.py $impl --steps 30 --warmup 8 >> $O/e2e_resnet50.jsonl 2>> $O/e2e.err
done
cat $O/e2e_resnet50.jsonl
