#!/bin/bash
# round 2, 1-GPU call L: virtual-cluster suite with the deferred copy-engine pushes; smoke
O=gpurun_out/r02g1l; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_vcluster.py -q -p no:cacheprovider -x --durations=8 > $O/pytest_vc.txt 2>&1; echo rc=$? >> $O/pytest_vc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
tail -12 $O/pytest_vc.txt; tail -2 $O/smoke.txt
