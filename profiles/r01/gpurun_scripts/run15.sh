TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29520"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k "overlapped" > gpurun_out/pytest15.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest15.log
for N in 2 4; do for M in fused faithful; do
timeout 300 $TR --nproc-per-node $N bench.py --gpus $N --mode $M > gpurun_out/b15_${N}_$M.log 2>&1; echo "bench $N $M rc=$?"; tail -1 gpurun_out/b15_${N}_$M.log | cut -c1-400
done; done
for T in 1x4 4x1; do
timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology $T --no-e2e > gpurun_out/b15_$T.log 2>&1; echo "bench $T rc=$?"
done
for T in 2x2 4x1; do
timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology $T --no-e2e --compute-ms 20 --steps 60 > gpurun_out/b15c_$T.log 2>&1; echo "bench compute $T rc=$?"
done
timeout 300 $TR --nproc-per-node 2 bench.py --gpus 2 --impl reference > gpurun_out/b15_ref2.log 2>&1; echo ref2=$?
