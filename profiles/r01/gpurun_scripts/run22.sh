CMD="python tools/kernel_bench.py --iters 1 --warmup 1"
$CMD > gpurun_out/plain22.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"fused_kernel|tma_kernel" -c 20 -o gpurun_out/ncu22 $CMD > gpurun_out/ncu22.log 2>&1; echo ncu=$?
DASO_KERNEL=tma $CMD > gpurun_out/plain22b.log 2>&1 && DASO_KERNEL=tma ncu --set full --clock-control none -k regex:"tma_kernel" -c 12 -o gpurun_out/ncu22t $CMD > gpurun_out/ncu22t.log 2>&1; echo ncu_tma=$?
