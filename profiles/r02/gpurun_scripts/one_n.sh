#!/bin/bash
# round 2 (session 2), 1-GPU call N: fused blocking tail (OP_NOX node-tier kernel + average/re-publish kernel)
# through the virtual cluster vs the oracle; smoke; K4 data-movement variants (tools/k4_variants.cu)
O=gpurun_out/r02g1n; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vcluster.py tests/test_gpu_vcluster_models.py -q -p no:cacheprovider -x > $O/pytest_vc.txt 2>&1; echo rc=$? >> $O/pytest_vc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 300 ./tools/k4v > $O/k4_variants.jsonl 2>&1
timeout 300 ./tools/k4v > $O/k4_variants_2.jsonl 2>&1
tail -3 $O/pytest_vc.txt; tail -2 $O/smoke.txt; cat $O/k4_variants.jsonl
