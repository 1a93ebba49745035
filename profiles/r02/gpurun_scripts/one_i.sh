#!/bin/bash
# round 2, 1-GPU call I: default bench line with the vcluster_2x4 block
O=gpurun_out/r02g1i; mkdir -p $O
python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?"
tail -5 $O/bench_n1.err
