#!/bin/bash
# round 2, 4-GPU call F (final): the whole GPU suite on 4 GPUs; node-tier kernel timing x3 (1x2, 1x4, 2x2)
# with the final warp-specialised kernel; final bench lines at N=2 and N=4 (defaults)
O=gpurun_out/r02m4f; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_vcluster.py -x -q -p no:cacheprovider > $O/pytest_vc_first.txt 2>&1; echo rc=$? >> $O/pytest_vc_first.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30300
b() { np=$1; shift; port=$((port+1)); timeout 400 $T --nproc-per-node $np --master-port $port bench.py --gpus $np "$@"; }
for rep in 1 2 3; do
  b 2 --topology 1x2 --steps 200 --warmup 10 --no-e2e --cycles 4 > $O/ws_1x2_$rep.json 2> $O/ws_1x2_$rep.err
  b 4 --topology 1x4 --steps 200 --warmup 10 --no-e2e --cycles 4 > $O/ws_1x4_$rep.json 2> $O/ws_1x4_$rep.err
  b 4 --steps 200 --warmup 10 --no-e2e --cycles 10 > $O/ws_2x2_$rep.json 2> $O/ws_2x2_$rep.err
done
b 2 > $O/bench_n2_default.json 2> $O/bench_n2_default.err
b 4 > $O/bench_n4_default.json 2> $O/bench_n4_default.err
b 4 --impl reference --steps 20 --warmup 3 > $O/bench_n4_reference.json 2> $O/bench_n4_reference.err
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > $O/pytest_gpu_4gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu_4gpu.txt
tail -3 $O/pytest_gpu_4gpu.txt
