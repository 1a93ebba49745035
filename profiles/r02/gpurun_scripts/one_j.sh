#!/bin/bash
# round 2, 1-GPU call J: TMA-staged K4 — bitwise test, A/B timing vs the register path
O=gpurun_out/r02g1j; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "k4" > $O/pytest_k4.txt 2>&1; echo rc=$? >> $O/pytest_k4.txt
for rep in 1 2; do for k4 in ldg tma; do DASO_K4=$k4 timeout 120 python tools/kernel_bench.py --only K4 --iters 50 > $O/k4_${k4}_$rep.json 2>&1; done; done
tail -3 $O/pytest_k4.txt
