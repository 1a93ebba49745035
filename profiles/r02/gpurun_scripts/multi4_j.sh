#!/bin/bash
# round 2 (session 2), 4-GPU call J: fused blocking tail (OP_NOX node-tier kernel + average/re-publish
# kernel with an in-kernel end barrier, replacing K4 + peer memcpys + an NCCL barrier) -- multi-GPU parity
# and the blocking-batch timing at 2x2; P-specialised two-chunk K4 (4x1 blocking, N=1 kernels block)
O=gpurun_out/r02m4j; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "k4 or k1 or k3" > $O/pytest_kernels.txt 2>&1; echo rc=$? >> $O/pytest_kernels.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --durations=5 \
  -k "blocking_fp32_is_flat_sync or (world4_toy_config1 and fused) or (world4_full_schedule and fused) or (copy_engine_exchange and 2-2-fused) or fused_tma_path_bit_identical or config5" \
  > $O/pytest_multi.txt 2>&1; echo rc=$? >> $O/pytest_multi.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30200
b() { port=$((port+1)); timeout 400 $T --nproc-per-node 4 --master-port $port bench.py --gpus 4 --steps 200 --warmup 10 --no-e2e "$@"; }
b --B 1 --S 0 --cycles 4 > $O/b_2x2_B1S0_1.json 2> $O/b_2x2_B1S0_1.err
b --B 1 --S 0 --cycles 4 > $O/b_2x2_B1S0_2.json 2> $O/b_2x2_B1S0_2.err
b --cycles 10 > $O/b_2x2_B4S1.json 2> $O/b_2x2_B4S1.err
b --topology 4x1 --B 1 --S 0 --cycles 4 > $O/b_4x1_B1S0.json 2> $O/b_4x1_B1S0.err
timeout 600 python bench.py --no-e2e --no-cpu > $O/bench_n1.json 2> $O/bench_n1.err
tail -2 $O/pytest_kernels.txt; tail -4 $O/pytest_multi.txt
for f in $O/b_*.json $O/bench_n1.json; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline',{})
print(d.get('ms_per_step'), {k:(v['ms_p50'] if isinstance(v,dict) else v) for k,v in (d.get('step_kinds') or {}).items()}, r.get('frac'), r.get('ms_per_launch'))
k=d.get('kernels') or {}
print({n:round(v['frac'],3) for n,v in k.items()})
" 2>&1 | tail -2; done
