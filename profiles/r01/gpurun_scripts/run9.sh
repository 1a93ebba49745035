TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29516"
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['topology'], d['config']['mode'], 'ms/step', round(d['ms_per_step'],4), 'value', round(d['value'],1), 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['ms_per_launch'],4), {k: round(v,4) for k,v in d['phases'].items() if k in ('wait_ms','exch_ms','hidden_fraction','local_ms','node_ms')}, 'e2e', d['e2e'] and round(d['e2e']['value'],1))"; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_all9.log 2>&1; echo pytest_all=$?; tail -3 gpurun_out/pytest_all9.log
timeout 300 python bench.py > gpurun_out/b9_1.log 2>&1; tail -1 gpurun_out/b9_1.log | summ
for N in 2 4; do for M in fused faithful sharded; do
timeout 300 $TR --nproc-per-node $N bench.py --gpus $N --mode $M > gpurun_out/b9_${N}_$M.log 2>&1; echo "bench $N $M rc=$?"; tail -1 gpurun_out/b9_${N}_$M.log | summ
done; done
for T in 1x4 4x1; do for M in fused faithful; do
timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology $T --mode $M --no-e2e > gpurun_out/b9_${T}_$M.log 2>&1; echo "bench $T $M rc=$?"; tail -1 gpurun_out/b9_${T}_$M.log | summ
done; done
timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --impl reference > gpurun_out/b9_ref4.log 2>&1; echo ref=$?; tail -1 gpurun_out/b9_ref4.log | cut -c1-600
for I in daso ddp; do
timeout 900 $TR --nproc-per-node 4 tools/e2e_train.py --model hmsa --impl $I --steps 10 --warmup 3 > gpurun_out/h9_$I.log 2>&1; echo "hmsa 4 $I rc=$?"; tail -1 gpurun_out/h9_$I.log
done
timeout 900 $TR --nproc-per-node 4 tools/e2e_train.py --model hmsa --impl daso --mode fused --steps 10 --warmup 3 > gpurun_out/h9_fused.log 2>&1; echo "hmsa 4 fused rc=$?"; tail -1 gpurun_out/h9_fused.log
