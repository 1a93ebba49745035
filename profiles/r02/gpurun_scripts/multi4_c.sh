#!/bin/bash
# round 2, 4-GPU call C: N2 test; exchange overlap vs compute length and NCCL CTA cap at 2x2
O=gpurun_out/r02m4c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -k "overlapped or config5" -q -p no:cacheprovider > $O/pytest_n2.txt 2>&1; echo rc=$? >> $O/pytest_n2.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=29900
for cap in 0 16; do for c in 1 5 20; do
  port=$((port+1))
  timeout 400 $T --nproc-per-node 4 --master-port $port bench.py --gpus 4 --steps 200 --warmup 10 --no-e2e \
     --nccl-max-ctas $cap --overlap-compute-ms $c --cycles 20 > $O/ov_cap${cap}_c$c.json 2> $O/ov_cap${cap}_c$c.err
done; done
for rep in 1 2 3; do
  port=$((port+1))
  timeout 400 $T --nproc-per-node 4 --master-port $port bench.py --gpus 4 --steps 200 --warmup 10 --no-e2e \
     --nccl-max-ctas 16 --cycles 4 > $O/fused_2x2_cap16_$rep.json 2> $O/fused_2x2_cap16_$rep.err
done
tail -3 $O/pytest_n2.txt
