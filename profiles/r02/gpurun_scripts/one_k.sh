#!/bin/bash
# round 2, 1-GPU call K: the copy-engine exchange inside the virtual cluster (parity), smoke, bench N=1
O=gpurun_out/r02g1k; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vcluster.py -q -p no:cacheprovider -x > $O/pytest_vc.txt 2>&1; echo rc=$? >> $O/pytest_vc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?" >> $O/pytest_vc.txt
tail -3 $O/pytest_vc.txt; tail -2 $O/smoke.txt
