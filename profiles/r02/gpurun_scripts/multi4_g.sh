#!/bin/bash
# round 2, 4-GPU call G: ResNet-50 end-to-end (config 3) at 1/2/4 GPUs with the final library:
# DASO fused + copy-engine exchange vs synchronous all-reduce (same library, P = 1) vs torch DDP
O=gpurun_out/r02m4g; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30500
for np in 1 2 4; do
  for impl in "--impl daso --mode fused --exchange ce" "--impl sync --mode fused" "--impl ddp"; do
    port=$((port+1))
    timeout 600 $T --nproc-per-node $np --master-port $port tools/e2e_train.py $impl --steps 30 --warmup 8 >> $O/e2e_resnet50.jsonl 2>> $O/e2e.err
  done
done
port=$((port+1)); timeout 900 $T --nproc-per-node 4 --master-port $port tools/e2e_train.py --model hmsa --impl ddp --steps 10 --warmup 3 >> $O/e2e_hmsa.jsonl 2>> $O/e2e.err
port=$((port+1)); timeout 900 $T --nproc-per-node 4 --master-port $port tools/e2e_train.py --model hmsa --impl daso --mode fused --exchange ce --steps 10 --warmup 3 >> $O/e2e_hmsa.jsonl 2>> $O/e2e.err
cat $O/e2e_resnet50.jsonl $O/e2e_hmsa.jsonl
