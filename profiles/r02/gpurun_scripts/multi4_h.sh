#!/bin/bash
# round 2, 4-GPU call H: CE S=B tests; node-tier kernel grid 132 vs 148 CTAs (with the copy-engine exchange no
# SMs need to stay free for NCCL)
O=gpurun_out/r02m4h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -k "copy_engine" -q -p no:cacheprovider > $O/pytest_ce.txt 2>&1; echo rc=$? >> $O/pytest_ce.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30700
b() { np=$1; shift; port=$((port+1)); timeout 400 $T --nproc-per-node $np --master-port $port bench.py --gpus $np --steps 200 --warmup 10 --no-e2e "$@"; }
for rep in 1 2; do for ctas in 132 148; do
  DASO_PEER_TMA_CTAS=$ctas b 2 --topology 1x2 --cycles 4 > $O/c${ctas}_1x2_$rep.json 2> $O/c${ctas}_1x2_$rep.err
  DASO_PEER_TMA_CTAS=$ctas b 4 --topology 1x4 --cycles 4 > $O/c${ctas}_1x4_$rep.json 2> $O/c${ctas}_1x4_$rep.err
  DASO_PEER_TMA_CTAS=$ctas b 4 --cycles 10 > $O/c${ctas}_2x2_$rep.json 2> $O/c${ctas}_2x2_$rep.err
done; done
tail -3 $O/pytest_ce.txt
