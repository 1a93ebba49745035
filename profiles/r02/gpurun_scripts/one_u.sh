#!/bin/bash
# round 2 (session 2), 1-GPU call U: full-size blocking syncs through the virtual cluster (2x2 bulk-store tail with
# many tiles per CTA; 4x1 kernel push + P-specialised K4) vs the oracle, tail paths bitwise
O=gpurun_out/r02g1u; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vcluster.py -q -p no:cacheprovider --durations=5 -k "full_size_blocking" > $O/pytest_vc.txt 2>&1; echo rc=$? >> $O/pytest_vc.txt
tail -n 8 $O/pytest_vc.txt
