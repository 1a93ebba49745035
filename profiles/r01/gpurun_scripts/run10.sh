TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29517"
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['topology'], d['config']['mode'], 'ms/step', round(d['ms_per_step'],4), 'value', round(d['value'],1), 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['ms_per_launch'],4), {k: round(v,4) for k,v in d['phases'].items() if k in ('wait_ms','exch_ms','hidden_fraction','local_ms','node_ms')})"; }
timeout 1200 python -m pytest tests/test_gpu_ctx.py tests/test_gpu_multi.py -q -x -k "ctx or fused or overlapped or tma or protocol or trace or step_host or kernel_impl or bind or split" > gpurun_out/pytest10.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest10.log
for T in 2x2 1x4; do
timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology $T --no-e2e > gpurun_out/b10_${T}.log 2>&1; echo "bench $T rc=$?"; tail -1 gpurun_out/b10_${T}.log | summ
done
timeout 300 $TR --nproc-per-node 2 bench.py --gpus 2 --topology 1x2 --no-e2e > gpurun_out/b10_1x2.log 2>&1; echo "bench 1x2 rc=$?"; tail -1 gpurun_out/b10_1x2.log | summ
timeout 900 $TR --nproc-per-node 4 tools/e2e_train.py --impl daso --overlap > gpurun_out/r10_overlap.log 2>&1; echo "resnet overlap rc=$?"; tail -1 gpurun_out/r10_overlap.log
