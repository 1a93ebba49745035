TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29522"
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['topology'], d['config']['mode'], 'ms/step', round(d['ms_per_step'],4), 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['ms_per_launch'],4), 'finite', d['finite'])"; }
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "nvls and (config1 or other_topologies or full_size)" > gpurun_out/pytest17.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest17.log
for BP in 2 4 8 16 32; do
DASO_NVLS_BPSM=$BP timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology 1x4 --no-e2e --mode nvls --steps 100 --warmup 5 > gpurun_out/b17_$BP.log 2>&1; echo -n "bpsm $BP rc=$? "; tail -1 gpurun_out/b17_$BP.log | summ
done
timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology 2x2 --no-e2e --mode nvls --steps 100 --warmup 5 > gpurun_out/b17_2x2.log 2>&1; echo -n "2x2 rc=$? "; tail -1 gpurun_out/b17_2x2.log | summ
