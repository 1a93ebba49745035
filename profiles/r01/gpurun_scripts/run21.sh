TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29525"
timeout 300 python -m pytest tests/test_gpu_multi.py -q -x -k "test_world4_toy_config1 and fused" > gpurun_out/pytest21.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest21.log
for N in 2 4; do timeout 300 $TR --nproc-per-node $N bench.py --gpus $N > gpurun_out/b21_$N.log 2>&1; echo "bench $N rc=$?"; done
timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology 1x4 --no-e2e > gpurun_out/b21_1x4.log 2>&1; echo "1x4 rc=$?"
for f in gpurun_out/b21_*.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['topology'], round(d['ms_per_step'],4), 'p50', round(d['phases']['p50_step_ms'],4), d['roofline']['bound'], round(d['roofline']['frac'],3), 'hidden', round(d['phases'].get('hidden_fraction',-1),3), 'e2e', d['e2e'] and round(d['e2e']['value'],1))"; done
