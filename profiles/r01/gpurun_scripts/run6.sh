TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29514"
for T in 2x2 1x4; do for BP in 2 4 8 16 64; do
DASO_PEER_BPSM=$BP timeout 300 $TR --nproc-per-node 4 bench.py --gpus 4 --topology $T --steps 200 --warmup 10 --mode fused --no-e2e > gpurun_out/b6_${T}_$BP.log 2>&1; echo "bench $T bpsm=$BP rc=$?"; tail -1 gpurun_out/b6_${T}_$BP.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['topology'], d['config']['mode'], 'ms/step', round(d['ms_per_step'],4), 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['ms_per_launch'],4))"
done; done
for I in daso sync ddp; do
timeout 600 $TR --nproc-per-node 4 tools/resnet_e2e.py --impl $I > gpurun_out/r6_4_$I.log 2>&1; echo "resnet 4 $I rc=$?"; tail -1 gpurun_out/r6_4_$I.log
done
timeout 600 $TR --nproc-per-node 4 tools/resnet_e2e.py --impl daso --mode fused > gpurun_out/r6_4_fused.log 2>&1; echo "resnet 4 fused rc=$?"; tail -1 gpurun_out/r6_4_fused.log
timeout 600 python tools/resnet_e2e.py --impl daso > gpurun_out/r6_1_daso.log 2>&1; tail -1 gpurun_out/r6_1_daso.log
timeout 600 python tools/resnet_e2e.py --impl ddp > gpurun_out/r6_1_ddp.log 2>&1; tail -1 gpurun_out/r6_1_ddp.log
