#!/bin/bash
# round 2 (session 2), 1-GPU call R: TMA-store blocking tail (avg_publish_tma_kernel) through the virtual
# cluster (parity, ldg == tma bitwise); ncu --set full of the new/changed kernels: the fused blocking pair
# (OP_NOX node-tier kernel + average/re-publish) in the one-GPU virtual cluster at 2x2, K3 (P-specialised)
# and K4 (two-chunk) from the kernel bench
O=gpurun_out/r02g1r; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vcluster.py -q -p no:cacheprovider -x -k "not full_size" > $O/pytest_vc.txt 2>&1; echo rc=$? >> $O/pytest_vc.txt
VC="python tools/vc_profile.py --topology 2x2 --B 1 --S 0 --exchange ce --steps 4"
$VC > $O/vc_blocking_plain.json 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"avg_publish|peer_ws" -s 8 -c 4 \
    -o $O/ncu_vc_blocking $VC > $O/ncu_vc_blocking.log 2>&1
KB="python tools/kernel_bench.py --iters 2 --warmup 1 --only K3_update_merge_P2,K3_update_merge_pack_P2,K4_average_P2"
$KB > $O/kb_plain.json 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused_kernel|average_kernel" \
    -o $O/ncu_k3_k4 $KB > $O/ncu_k3_k4.log 2>&1
ls -la $O; tail -3 $O/pytest_vc.txt; tail -3 $O/ncu_vc_blocking.log $O/ncu_k3_k4.log
