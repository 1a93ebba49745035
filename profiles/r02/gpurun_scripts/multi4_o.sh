#!/bin/bash
# round 2 (session 2), 4-GPU call O: the multi-GPU parity tests this session's changes touch that had not run
# on real GPUs with the final library (P-specialised K3 in every mode's merges, two-chunk K4, kernel push at G = 1,
# output-buffer rotation): world-4 toy (faithful / sharded), full schedules, other topologies, full-size sampled
O=gpurun_out/r02m4o; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --durations=20 \
  -k "(world4_toy_config1 and not fused) or (world4_full_schedule and not fused) or world4_other_topologies or full_size_microbench or world2_scheduled" \
  > $O/pytest_multi.txt 2>&1; echo rc=$? >> $O/pytest_multi.txt
tail -n 4 $O/pytest_multi.txt
