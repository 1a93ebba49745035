#!/bin/bash
# round 2 (session 2), 1-GPU call W (final, after the push-policy refinement): what the driver runs at round end -- build(), smoke(), pytest -m gpu
O=gpurun_out/r02g1w; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build_smoke.txt 2>&1; echo "build+smoke rc=$?" >> $O/build_smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/pytest_gpu_1gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu_1gpu.txt
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?" >> $O/pytest_gpu_1gpu.txt
timeout 600 python bench.py --impl reference > $O/bench_n1_reference.json 2> $O/bench_n1_reference.err
tail -n 3 $O/build_smoke.txt; tail -n 4 $O/pytest_gpu_1gpu.txt
