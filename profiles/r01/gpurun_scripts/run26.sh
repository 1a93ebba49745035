TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29526"
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['topology'], 'ms/step', round(d['ms_per_step'],4), 'p50', round(d['phases']['p50_step_ms'],4), 'kernel', round(d['roofline']['ms_per_launch'],4), 'frac', round(d['roofline']['frac'],3))"; }
timeout 120 python tools/kernel_bench.py --only K1,K2 | python -c "import json,sys; d=json.load(sys.stdin); print({k: round(v['us'],1) for k,v in d['kernels'].items()})"
for T in 1024 4096; do DASO_PEER_TILE=$T timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "tma or (config1 and fused)" > gpurun_out/pytest26_$T.log 2>&1; echo "pytest tile $T rc=$?"; tail -1 gpurun_out/pytest26_$T.log; done
DASO_PEER_CTAS_PER_SM=2 timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "tma" > gpurun_out/pytest26_c2.log 2>&1; echo "pytest ctas2 rc=$?"; tail -1 gpurun_out/pytest26_c2.log
for TOPO in 2x2 1x4; do for T in 1024 2048 4096; do for C in 1 2; do
DASO_PEER_TILE=$T DASO_PEER_CTAS_PER_SM=$C timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology $TOPO --no-e2e --steps 150 --warmup 5 > gpurun_out/b26.log 2>&1; echo -n "tile $T cps $C rc=$? "; tail -1 gpurun_out/b26.log | summ
done; done; done
