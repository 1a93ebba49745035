TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29519"
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['topology'], d['config']['mode'], 'ms/step', round(d['ms_per_step'],4), 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['ms_per_launch'],4))"; }
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k "fused or tma" > gpurun_out/pytest13.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest13.log
for rep in 1 2; do for T in 1x2 2x2 1x4; do
W=4; [ $T = 1x2 ] && W=2
for K in auto ldg; do
DASO_KERNEL=$K timeout 300 $TR --nproc-per-node $W bench.py --gpus $W --topology $T --no-e2e --steps 100 --warmup 5 > gpurun_out/b13_${T}_${K}_$rep.log 2>&1; echo -n "$K rep$rep: "; tail -1 gpurun_out/b13_${T}_${K}_$rep.log | summ
done; done; done
