timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "fused" > gpurun_out/pytest_fused.log 2>&1; echo pytest_fused=$?; tail -4 gpurun_out/pytest_fused.log
for T in 2x2 1x4 4x1; do for M in fused faithful; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --topology $T --steps 200 --warmup 10 --mode $M --no-e2e > gpurun_out/b5_${T}_${M}.log 2>&1; echo bench $T $M=$?; tail -1 gpurun_out/b5_${T}_${M}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['topology'], d['config']['mode'], 'ms/step', round(d['ms_per_step'],4), 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), {k: round(v,4) for k,v in d['phases'].items() if k.endswith('_ms') or k.endswith('gbs') or k=='hidden_fraction'})"
done; done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all4.log 2>&1; echo pytest_all=$?; tail -4 gpurun_out/pytest_all4.log
