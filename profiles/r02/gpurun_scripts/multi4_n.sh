#!/bin/bash
# round 2 (session 2), 4-GPU call N (final library): config-2 sweep B in {1,2,4,8} (S = 1,1,1,2) and the
# blocking mode S = 0 at 2x2 and 4x1, copy-engine exchange; hidden fraction from paired cycle differences
# (sleep and GEMM stand-ins, 120 GEMM cycles per leg)
O=gpurun_out/r02m4n; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30600
b() { port=$((port+1)); timeout 400 $T --nproc-per-node 4 --master-port $port bench.py --gpus 4 --steps 200 --warmup 10 --no-e2e "$@"; }
for topo in 2x2 4x1; do
  for bs in "1 1" "2 1" "4 1" "8 2" "1 0"; do
    set -- $bs
    b --topology $topo --B $1 --S $2 --cycles 30 > $O/sweep_${topo}_B$1S$2.json 2> $O/sweep_${topo}_B$1S$2.err
  done
done
for f in $O/sweep_*.json; do echo $f; python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline',{}); o=d.get('overlap') or {}
print(round(d.get('ms_per_step'),4), {k:round(v['ms_p50'],4) for k,v in (d.get('step_kinds') or {}).items()}, 'frac', round(r.get('frac') or 0,3), 'hidden', {k:round(v['hidden_fraction'],3) for k,v in o.items() if v.get('hidden_fraction') is not None}, 'T_AG', round(list(o.values())[0]['T_AG_alone_ms'],4) if o else None, d['clocks']['sm_mhz'], d['clocks']['reasons'])
" 2>&1 | tail -1; done
