#!/bin/bash
# round 2 (session 2), 4-GPU call L: fused blocking tail with TMA bulk stores (avg_publish_tma_kernel) vs
# register stores at 2x2 and 1x4 (blocking batches), its multi-GPU parity; final default bench lines at N=2
# (2x1) and N=4 (2x2) with e2e, the N=4 reference arm; smoke with the blocking warm-up; the P-templated,
# prefetching TMA tail kernel: vcluster parity (bitwise vs register path) and its ncu capture; the N4 training
# loop on real losses (warm-up / cool-down are blocking syncs) at 2x2
O=gpurun_out/r02m4l; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 600 python -m pytest tests/test_gpu_vcluster.py -q -p no:cacheprovider -k "avg_publish or kernel_push or trace_accounting or copy_engine or blocking" > $O/pytest_vc.txt 2>&1; echo rc=$? >> $O/pytest_vc.txt
VC="python tools/vc_profile.py --topology 2x2 --B 1 --S 0 --exchange ce --steps 4"
$VC > $O/vc_blocking_plain.json 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"avg_publish" -s 8 -c 4 \
    -o $O/ncu_vc_avg_publish $VC > $O/ncu_vc_avg_publish.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --durations=5 \
  -k "(blocking_fp32_is_flat_sync and fused) or (world4_full_schedule and fused) or (copy_engine_exchange and 2-2-fused)" \
  > $O/pytest_multi.txt 2>&1; echo rc=$? >> $O/pytest_multi.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30400
b() { port=$((port+1)); timeout 400 $T --nproc-per-node 4 --master-port $port bench.py --gpus 4 --steps 200 --warmup 10 --no-e2e "$@"; }
b --B 1 --S 0 --cycles 4 > $O/b_2x2_B1S0_tma_1.json 2> $O/b_2x2_B1S0_tma_1.err
DASO_AVG_PUBLISH=ldg b --B 1 --S 0 --cycles 4 > $O/b_2x2_B1S0_ldg.json 2> $O/b_2x2_B1S0_ldg.err
b --B 1 --S 0 --cycles 4 > $O/b_2x2_B1S0_tma_2.json 2> $O/b_2x2_B1S0_tma_2.err
b --topology 1x4 --B 1 --S 0 --cycles 4 > $O/b_1x4_B1S0_tma.json 2> $O/b_1x4_B1S0_tma.err
DASO_AVG_PUBLISH=ldg b --topology 1x4 --B 1 --S 0 --cycles 4 > $O/b_1x4_B1S0_ldg.json 2> $O/b_1x4_B1S0_ldg.err
timeout 600 $T --nproc-per-node 2 --master-port 30490 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err
timeout 600 $T --nproc-per-node 4 --master-port 30491 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err
timeout 600 $T --nproc-per-node 4 --master-port 30492 bench.py --gpus 4 --impl reference > $O/bench_n4_reference.json 2> $O/bench_n4_reference.err
timeout 600 $T --nproc-per-node 4 --master-port 30493 tools/e2e_train.py --impl daso --mode fused --exchange ce --train-epochs 6 --steps-per-epoch 8 --batch 64 > $O/e2e_train_epochs.jsonl 2> $O/e2e_train_epochs.err; echo "e2e rc=$?" >> $O/smoke.txt
tail -n 2 $O/smoke.txt; tail -n 2 $O/pytest_vc.txt; tail -n 3 $O/pytest_multi.txt
for f in $O/b_*.json $O/bench_n2.json $O/bench_n4.json; do echo $f; python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline',{}); p=d['phases']
print(round(d.get('ms_per_step'),4), {k:round(v['ms_p50'],4) for k,v in (d.get('step_kinds') or {}).items()}, 'kern/step', round(p['kernel_ms'],4), 'wait', round(p['wait_ms'],4), 'exch', round(p['exch_ms'],4), 'frac', round(r.get('frac') or 0,3), 'value', round(d['value'],1), 'e2e', (d.get('e2e') or {}).get('value'))
" 2>&1 | tail -1; done
