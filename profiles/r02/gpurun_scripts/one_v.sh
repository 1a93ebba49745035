#!/bin/bash
# round 2 (session 2), 1-GPU call V: push policy refined (the node-tier kernel also pushes for groups of P >= 3,
# where the copy engines' all-to-all reaches only 0.57 of the link); the whole virtual-cluster suite + smoke
O=gpurun_out/r02g1v; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vcluster.py tests/test_gpu_vcluster_models.py -q -p no:cacheprovider --durations=5 > $O/pytest_vc.txt 2>&1; echo rc=$? >> $O/pytest_vc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
tail -n 3 $O/pytest_vc.txt; tail -n 2 $O/smoke.txt
