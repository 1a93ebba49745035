TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29524"
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['topology'], 'ms/step', round(d['ms_per_step'],4), 'p50', round(d['phases']['p50_step_ms'],4), 'kernel', round(d['roofline']['ms_per_launch'],4), 'frac', round(d['roofline']['frac'],3), 'hidden', round(d['phases'].get('hidden_fraction',-1),3))"; }
for V in "A|" "B|--nccl-max-ctas 4" "C|--nccl-max-ctas 8" ; do
  tag=${V%%|*}; args=${V#*|}
  timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --no-e2e --steps 200 --warmup 10 $args > gpurun_out/b20_$tag.log 2>&1; echo -n "$tag [$args] rc=$? "; tail -1 gpurun_out/b20_$tag.log | summ
done
DASO_PEER_TMA_CTAS=132 timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --no-e2e --steps 200 --warmup 10 > gpurun_out/b20_D.log 2>&1; echo -n "D [ctas 132] rc=$? "; tail -1 gpurun_out/b20_D.log | summ
DASO_PEER_TMA_CTAS=132 timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --no-e2e --steps 200 --warmup 10 --nccl-max-ctas 8 > gpurun_out/b20_E.log 2>&1; echo -n "E [ctas 132, nccl 8] rc=$? "; tail -1 gpurun_out/b20_E.log | summ
