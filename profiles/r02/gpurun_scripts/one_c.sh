#!/bin/bash
# round 2, 1-GPU call C: N=1 bench line; ncu launch list + full capture of the N=1 bench; ncu full capture of
# the fused node-tier kernel (warp-specialised and TMA paths) in the one-GPU virtual cluster at 1x2 and 2x2
O=gpurun_out/r02g1c; mkdir -p $O
python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?"
CMD="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-kernels"
$CMD > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_n1.csv $CMD > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
$CMD > $O/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fused_kernel \
    -s 20 -c 3 -o $O/ncu_bench_n1 $CMD > $O/ncu_full.log 2>&1; echo "full rc=$?"
for t in 1x2 2x2; do
  V="python tools/vc_profile.py --topology $t --steps 4"
  $V > $O/vc_$t.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:peer_ \
      -c 4 -o $O/ncu_vc_$t $V > $O/ncu_vc_$t.log 2>&1; echo "vc $t rc=$?"
  DASO_PEER=tma $V > $O/vc_${t}_tma.json 2>&1 && DASO_PEER=tma ncu --set full --clock-control none --import-source on \
      -k regex:peer_ -c 4 -o $O/ncu_vc_${t}_tma $V > $O/ncu_vc_${t}_tma.log 2>&1; echo "vc $t tma rc=$?"
done
ls -la $O
