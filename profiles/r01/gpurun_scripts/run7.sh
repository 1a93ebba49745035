TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29515"
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['topology'], d['config']['mode'], 'ms/step', round(d['ms_per_step'],4), 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['ms_per_launch'],4), {k: round(v,4) for k,v in d['phases'].items() if k in ('wait_ms','exch_ms','hidden_fraction','local_ms','node_ms')})"; }
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "tma" > gpurun_out/pytest_tma.log 2>&1; echo pytest_tma=$?; tail -3 gpurun_out/pytest_tma.log
for T in 2x2 1x4; do for K in tma ldg; do
DASO_KERNEL=$K timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology $T --steps 200 --warmup 10 --mode fused --no-e2e > gpurun_out/b7_${T}_$K.log 2>&1; echo "bench $T $K rc=$?"; tail -1 gpurun_out/b7_${T}_$K.log | summ
done; done
for T in 4x1 2x2; do for M in faithful fused; do
timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology $T --steps 100 --warmup 5 --mode $M --no-e2e --compute-ms 20 > gpurun_out/b7c_${T}_$M.log 2>&1; echo "bench compute $T $M rc=$?"; tail -1 gpurun_out/b7c_${T}_$M.log | summ
done; done
for I in "daso --mode faithful" "daso --mode fused" "sync"; do
timeout 600 $TR --nproc-per-node 4 tools/resnet_e2e.py --impl $I > gpurun_out/r7.log 2>&1; echo "resnet 4 $I rc=$?"; tail -1 gpurun_out/r7.log
done
timeout 600 python tools/resnet_e2e.py --impl daso > gpurun_out/r7_1.log 2>&1; tail -1 gpurun_out/r7_1.log
