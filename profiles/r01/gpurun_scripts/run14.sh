python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke14.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke14.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest14.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest14.log
timeout 300 python bench.py > gpurun_out/bench14_n1.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench14_n1.log
timeout 300 python tools/kernel_bench.py > gpurun_out/kb14.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/kb14.json')); [print(k, round(v['us'],1), round(v['frac_of_measured_peak'],3)) for k,v in d['kernels'].items()]"
CMD="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu"
$CMD > gpurun_out/plain14.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches14.csv $CMD > gpurun_out/ncu14a.log 2>&1; echo ncu_launches=$?
$CMD > gpurun_out/plain14b.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 20 -c 5 -o gpurun_out/ncu14 $CMD > gpurun_out/ncu14b.log 2>&1; echo ncu_full=$?
