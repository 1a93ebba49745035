TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29521"
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['topology'], d['config']['mode'], 'ms/step', round(d['ms_per_step'],4), 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['ms_per_launch'],4), 'finite', d['finite'])"; }
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k "nvls" > gpurun_out/pytest16.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest16.log | grep -v "^\s*$" | tail -8
for T in 1x4 2x2 1x2; do
W=4; [ $T = 1x2 ] && W=2
for M in nvls fused; do
timeout 300 $TR --nproc-per-node $W bench.py --gpus $W --topology $T --no-e2e --mode $M --steps 100 --warmup 5 > gpurun_out/b16_${T}_$M.log 2>&1; echo -n "rc=$? "; tail -1 gpurun_out/b16_${T}_$M.log | summ
done; done
