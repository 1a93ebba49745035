#!/bin/bash
# round 2 (session 2), 1-GPU call S: push policy applied (node-tier kernel: copy-engine pushes; local pack
# kernels: kernel push); vcluster parity; smoke with the blocking warm-up; ncu --set full of the fused
# blocking pair (OP_NOX node-tier kernel + avg_publish_tma_kernel) in the one-GPU virtual cluster at 2x2
O=gpurun_out/r02g1s; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vcluster.py -q -p no:cacheprovider -k "not full_size" > $O/pytest_vc.txt 2>&1; echo rc=$? >> $O/pytest_vc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
VC="python tools/vc_profile.py --topology 2x2 --B 1 --S 0 --exchange ce --steps 4"
$VC > $O/vc_blocking_plain.json 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"avg_publish|peer_ws" -s 16 -c 8 \
    -o $O/ncu_vc_blocking $VC > $O/ncu_vc_blocking.log 2>&1
tail -n 3 $O/pytest_vc.txt; tail -n 2 $O/smoke.txt; tail -n 2 $O/ncu_vc_blocking.log
