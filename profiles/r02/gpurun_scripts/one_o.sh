#!/bin/bash
# round 2 (session 2), 1-GPU call O: blocking syncs with the kernel push (the pack kernel stores the packed
# row into every group member's slot) through the virtual cluster: CE parity incl. all-blocking schedules,
# kernel push == copy-engine pushes bitwise, trace accounting; K3/K4 specialisations (kernel tests); N=1 line
O=gpurun_out/r02g1o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vcluster.py tests/test_gpu_kernels.py tests/test_gpu_ctx.py -q -p no:cacheprovider -x --durations=5 > $O/pytest.txt 2>&1; echo rc=$? >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 600 python bench.py --no-e2e --no-cpu > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?" >> $O/pytest.txt
tail -3 $O/pytest.txt; tail -2 $O/smoke.txt
python -c "
import json
d=json.loads(open('$O/bench_n1.json').read().strip().splitlines()[-1])
print({n:(round(v['us_mean'],1),round(v['frac'],3)) for n,v in d['kernels']['kernels'].items()})"
