#!/usr/bin/env bash
# Reproduce the measurements committed under profiles/ (run on a B200 box, e.g. via gpurun).
#   bash tools/run_profiles.sh n1      # 1 GPU: bench line, kernel table, ncu launch list + full capture
#   bash tools/run_profiles.sh multi   # 4 GPUs: bench at N=2/4 in every mode and topology, NVLink probe
#   bash tools/run_profiles.sh e2e     # 4 GPUs: ResNet-50 / HMSA end-to-end training throughput
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port ${PORT:-29530}"
case "${1:-n1}" in
n1)
    python bench.py > "$OUT/bench_n1.json"
    python tools/kernel_bench.py > "$OUT/kernel_bench.json"
    CMD="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu"
    $CMD > "$OUT/plain.log" 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file "$OUT/launches_n1.csv" $CMD > "$OUT/ncu_launches.log" 2>&1
    $CMD > "$OUT/plain2.log" 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fused_kernel \
        -s 20 -c 5 -o "$OUT/ncu_bench_n1" $CMD > "$OUT/ncu_full.log" 2>&1
    ;;
multi)
    python tools/nvlink_probe.py --gpus 4 > "$OUT/nvlink_probe.json"
    for N in 2 4; do for M in fused faithful sharded; do
        $TR --nproc-per-node $N bench.py --gpus $N --mode $M > "$OUT/bench_${N}_${M}.json"
    done; done
    for T in 1x4 4x1; do for M in fused faithful; do
        $TR --nproc-per-node 4 bench.py --gpus 4 --topology $T --mode $M --no-e2e > "$OUT/bench_${T}_${M}.json"
    done; done
    for T in 4x1 2x2; do
        $TR --nproc-per-node 4 bench.py --gpus 4 --topology $T --no-e2e --compute-ms 20 > "$OUT/bench_${T}_compute20.json"
    done
    $TR --nproc-per-node 4 bench.py --gpus 4 --impl reference > "$OUT/bench_4_reference.json"
    ;;
e2e)
    for I in "daso --mode faithful" "daso --mode fused" "daso --overlap" sync ddp; do
        $TR --nproc-per-node 4 tools/e2e_train.py --impl $I >> "$OUT/e2e_resnet50.jsonl"
    done
    for I in "daso" "daso --mode fused" ddp; do
        $TR --nproc-per-node 4 tools/e2e_train.py --model hmsa --impl $I --steps 10 --warmup 3 >> "$OUT/e2e_hmsa.jsonl"
    done
    ;;
esac
