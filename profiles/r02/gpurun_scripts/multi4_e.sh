#!/bin/bash
# round 2, 4-GPU call E: copy-engine exchange on parallel streams (parity, overlap with sleep/GEMM stand-ins,
# NCCL side by side), config-2 sweep with the CE exchange
O=gpurun_out/r02m4e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -k "copy_engine" -q -p no:cacheprovider > $O/pytest_ce.txt 2>&1; echo rc=$? >> $O/pytest_ce.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30100
b() { port=$((port+1)); timeout 400 $T --nproc-per-node 4 --master-port $port bench.py --gpus 4 --steps 200 --warmup 10 --no-e2e "$@"; }
for ex in ce nccl; do
  for topo in 2x2 4x1; do
    b --topology $topo --exchange $ex --overlap-compute-ms 1 --cycles 30 > $O/ov_${topo}_${ex}_c1.json 2> $O/ov_${topo}_${ex}_c1.err
  done
  b --topology 2x2 --exchange $ex --overlap-compute-ms 20 --overlap-compute sleep --cycles 10 > $O/ov_2x2_${ex}_sleep20.json 2> $O/ov_2x2_${ex}_sleep20.err
done
for bs in "1 1" "2 1" "4 1" "8 2" "1 0"; do
  set -- $bs
  b --B $1 --S $2 --exchange ce --cycles 20 > $O/sweep_ce_2x2_B$1S$2.json 2> $O/sweep_ce_2x2_B$1S$2.err
done
b --topology 1x4 --exchange ce --cycles 4 > $O/ce_1x4.json 2> $O/ce_1x4.err
tail -3 $O/pytest_ce.txt
