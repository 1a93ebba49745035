TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29523"
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['topology'], d['config']['mode'], 'ms/step', round(d['ms_per_step'],4), 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['ms_per_launch'],4), 'finite', d['finite'])"; }
for C in 16 32 64 148 296; do
DASO_NVLS_CTAS=$C timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology 1x4 --no-e2e --mode nvls --steps 100 --warmup 5 > gpurun_out/b18_$C.log 2>&1; echo -n "ctas $C rc=$? "; tail -1 gpurun_out/b18_$C.log | summ
done
