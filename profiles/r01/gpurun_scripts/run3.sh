set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_k.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_k.log
DASO_KERNEL=ldg timeout 120 python tools/kernel_bench.py > gpurun_out/kb_ldg.json 2>&1; cat gpurun_out/kb_ldg.json
DASO_KERNEL=tma timeout 120 python tools/kernel_bench.py > gpurun_out/kb_tma.json 2>&1; cat gpurun_out/kb_tma.json
DASO_KERNEL=ldg timeout 120 python tools/kernel_bench.py --only K1,K3_update_merge_pack --iters 3 --warmup 1 > /dev/null 2>&1 && DASO_KERNEL=ldg timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 3 -o gpurun_out/ncu_k1_ldg python tools/kernel_bench.py --only K1,K3_update_merge_pack --iters 3 --warmup 1 > gpurun_out/ncu_ldg.log 2>&1; echo ncu1=$?
