python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke24.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke24.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest24.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest24.log
timeout 300 python bench.py > gpurun_out/bench24.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench24.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['roofline']['frac'], d['roofline']['traffic'], d['clocks'], d['gpu_launches'], d['cpu_baseline']['value'])"
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench24r.log 2>&1; echo ref=$?; tail -1 gpurun_out/bench24r.log | cut -c1-300
