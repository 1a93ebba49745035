set -x
nvidia-smi topo -m | head -8
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu4.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_gpu4.log
for N in 2 4; do for M in faithful sharded; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 200 --warmup 10 --mode $M > gpurun_out/bench_${N}_${M}.log 2>&1; echo bench $N $M=$?; tail -1 gpurun_out/bench_${N}_${M}.log | cut -c1-2500
done; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --topology 4x1 --steps 200 --warmup 10 > gpurun_out/bench_4x1.log 2>&1; tail -1 gpurun_out/bench_4x1.log | cut -c1-2500
