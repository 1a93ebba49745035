#!/bin/bash
# round 2 (session 2), 1-GPU call P (re-run as Q after OP_PUSH got its own instantiations): kernel table, kernel and vcluster tests
# version slowed every pack kernel: K2 82 -> 88 us, K3+pack 106 -> 178 us); kernel table, kernel and vcluster tests
O=gpurun_out/r02g1q; mkdir -p $O
timeout 600 python bench.py --no-e2e --no-cpu --no-vcluster --steps 50 > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?" > $O/pytest.txt
python -c "
import json
d=json.loads(open('$O/bench_n1.json').read().strip().splitlines()[-1])
for n,v in d['kernels']['kernels'].items(): print(n, round(v['us_mean'],1), round(v['us_p10'],1), round(v['us_p90'],1), round(v['frac'],3))"
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_vcluster.py -q -p no:cacheprovider -x -k "not full_size" >> $O/pytest.txt 2>&1; echo rc=$? >> $O/pytest.txt
tail -3 $O/pytest.txt
