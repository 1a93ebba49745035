#!/bin/bash
# round 2, 1-GPU call C: N=1 bench line; ncu launch list + full capture of the N=1 bench; ncu full capture of
# the fused node-tier kernel (warp-specialised and TMA paths) in the one-GPU virtual cluster at 1x2 and 2x2.
# Reports are exported to CSV on the box (raw metrics + source-level stalls) to stay under gpurun's 64 MiB.
O=gpurun_out/r02g1c; mkdir -p $O; S=/tmp/ncu; mkdir -p $S
python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?"
CMD="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-kernels"
$CMD > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_n1.csv $CMD > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
$CMD > $O/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fused_kernel \
    -s 20 -c 2 -o $O/ncu_bench_n1 $CMD > $O/ncu_full.log 2>&1; echo "full rc=$?"
ncu -i $O/ncu_bench_n1.ncu-rep --page raw --csv > $O/ncu_bench_n1_raw.csv 2>&1
for t in 1x2 2x2; do for p in ws tma; do
  V="python tools/vc_profile.py --topology $t --steps 3"
  DASO_PEER=$p $V > $O/vc_${t}_$p.json 2>&1 && DASO_PEER=$p ncu --set full --clock-control none --import-source on \
      -k regex:peer_ -s 2 -c 2 -o $S/ncu_vc_${t}_$p $V > $O/ncu_vc_${t}_$p.log 2>&1; echo "vc $t $p rc=$?"
  ncu -i $S/ncu_vc_${t}_$p.ncu-rep --page raw --csv > $O/ncu_vc_${t}_${p}_raw.csv 2>&1
  ncu -i $S/ncu_vc_${t}_$p.ncu-rep --page source --csv > $O/ncu_vc_${t}_${p}_source.csv 2>&1
done; done
du -sh $O; ls -la $O
