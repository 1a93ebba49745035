#!/bin/bash
# round 2 (session 2), 4-GPU call M: warp-specialised node-tier kernel with 2 / 3 / 4 shared-memory output
# buffers (DASO_PEER_OUT): can the bulk stores' smem reads stall the driver warp (and with it the load issue)?
# bitwise test on one GPU first; then 2x2 and 1x4 lines alternating
O=gpurun_out/r02m4m; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_vcluster.py -q -p no:cacheprovider -k "ws_output_buffers or peer_data_paths" > $O/pytest_vc.txt 2>&1; echo rc=$? >> $O/pytest_vc.txt
tail -n 2 $O/pytest_vc.txt
grep -q "rc=0" $O/pytest_vc.txt || exit 1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=30500
b() { port=$((port+1)); timeout 400 $T --nproc-per-node 4 --master-port $port bench.py --gpus 4 --steps 200 --warmup 10 --no-e2e --cycles 4 "$@"; }
for rep in 1 2; do
  for no in 2 4 3; do
    [ $rep = 2 ] && [ $no = 3 ] && continue
    DASO_PEER_OUT=$no b > $O/b_2x2_out${no}_$rep.json 2> $O/b_2x2_out${no}_$rep.err
    DASO_PEER_OUT=$no b --topology 1x4 > $O/b_1x4_out${no}_$rep.json 2> $O/b_1x4_out${no}_$rep.err
  done
done
for f in $O/b_*.json; do echo $f; python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline',{}); p=d['phases']
print(round(d.get('ms_per_step'),4), {k:round(v['ms_p50'],4) for k,v in (d.get('step_kinds') or {}).items()}, 'us/launch', round(r.get('ms_per_launch')*1e3,1), 'frac', round(r.get('frac') or 0,3), 'frac_p50', round(r.get('frac_at_p50_plain_step') or 0,3), d['clocks']['sm_mhz'])
" 2>&1 | tail -1; done
