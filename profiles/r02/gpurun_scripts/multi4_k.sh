#!/bin/bash
# round 2 (session 2), 4-GPU call K: blocking syncs with the kernel push (pack kernel stores the packed row
# into every group member's slot over NVLink) on real GPUs -- parity, and timing A/B against the copy-engine
# pushes (DASO_BLOCKING_PUSH=0) at 2x2 and 4x1; default lines 2x2 / 1x4 / 4x1
O=gpurun_out/r02m4k; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --durations=5 \
  -k "copy_engine_exchange or (blocking_fp32_is_flat_sync and fused) or (world4_full_schedule and fused) or config5" \
  > $O/pytest_multi.txt 2>&1; echo rc=$? >> $O/pytest_multi.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30300
b() { port=$((port+1)); timeout 400 $T --nproc-per-node 4 --master-port $port bench.py --gpus 4 --steps 200 --warmup 10 --no-e2e "$@"; }
b --B 1 --S 0 --cycles 4 > $O/b_2x2_B1S0_kp_1.json 2> $O/b_2x2_B1S0_kp_1.err
DASO_BLOCKING_PUSH=0 b --B 1 --S 0 --cycles 4 > $O/b_2x2_B1S0_ce.json 2> $O/b_2x2_B1S0_ce.err
b --B 1 --S 0 --cycles 4 > $O/b_2x2_B1S0_kp_2.json 2> $O/b_2x2_B1S0_kp_2.err
b --topology 4x1 --B 1 --S 0 --cycles 4 > $O/b_4x1_B1S0_kp.json 2> $O/b_4x1_B1S0_kp.err
DASO_BLOCKING_PUSH=0 b --topology 4x1 --B 1 --S 0 --cycles 4 > $O/b_4x1_B1S0_ce.json 2> $O/b_4x1_B1S0_ce.err
b --cycles 10 > $O/b_2x2_B4S1.json 2> $O/b_2x2_B4S1.err
b --topology 4x1 --cycles 10 > $O/b_4x1_B4S1.json 2> $O/b_4x1_B4S1.err
b --topology 1x4 --cycles 4 > $O/b_1x4_B4S1.json 2> $O/b_1x4_B4S1.err
tail -4 $O/pytest_multi.txt
for f in $O/b_*.json; do echo $f; python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline',{}); p=d['phases']
print(round(d.get('ms_per_step'),4), {k:round(v['ms_p50'],4) for k,v in (d.get('step_kinds') or {}).items()}, 'kern/step', round(p['kernel_ms'],4), 'wait', round(p['wait_ms'],4), 'exch', round(p['exch_ms'],4), 'frac', round(r.get('frac') or 0,3))
" 2>&1 | tail -1; done
