#!/bin/bash
# round 2, 1-GPU call B: vcluster + kernel parity with the warp-specialised peer path, K4 A/B, bench N=1
O=gpurun_out/r02g1b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vcluster.py tests/test_gpu_vcluster_models.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider --durations=10 > $O/pytest.txt 2>&1; echo rc=$? >> $O/pytest.txt
for k4 in one two one two; do DASO_K4=$k4 timeout 120 python tools/kernel_bench.py --only K4 --iters 50 > $O/k4_$k4.json 2>&1; cp $O/k4_$k4.json $O/k4_${k4}_$RANDOM.json; done
timeout 600 python bench.py --steps 100 --warmup 10 > $O/bench.json 2> $O/bench.err; echo bench rc=$? >> $O/pytest.txt
tail -5 $O/pytest.txt
