#!/bin/bash
# round 2, 4-GPU call B: the whole GPU suite on 4 GPUs; peer-path A/B (ws / tma / ldg) at 1x2, 2x2, 1x4;
# config-2 sweep lines with the alternating hidden-fraction legs; N4 training loop; HMSA e2e
O=gpurun_out/r02m4b; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 > $O/pytest_gpu_4gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu_4gpu.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=29700
run() {   # run <name> <nproc> <env...> -- <bench args>
  name=$1; np=$2; shift 2
  port=$((port+1))
  env "$@" timeout 400 $T --nproc-per-node $np --master-port $port bench.py --gpus $np --steps 200 --warmup 10 --no-e2e $BARGS > $O/$name.json 2> $O/$name.err
}
for rep in 1 2 3; do
  for p in ws tma ldg; do
    BARGS="--topology 1x2 --cycles 4" run b_1x2_${p}_$rep 2 DASO_PEER=$p
    BARGS="--cycles 4" run b_2x2_${p}_$rep 4 DASO_PEER=$p
    BARGS="--topology 1x4 --cycles 4" run b_1x4_${p}_$rep 4 DASO_PEER=$p
  done
done
for bs in "1 1" "2 1" "4 1" "8 2" "1 0"; do
  set -- $bs
  BARGS="--B $1 --S $2 --dump-steps" run sweep_2x2_B$1S$2 4 X=1
done
BARGS="--topology 4x1" run sweep_4x1_B4S1 4 X=1
BARGS="--mode faithful" run faithful_2x2_B4S1 4 X=1
timeout 600 $T --nproc-per-node 4 --master-port 29800 tools/e2e_train.py --model resnet50 --train-epochs 6 --steps-per-epoch 8 --mode fused > $O/e2e_train_epochs_fused.jsonl 2> $O/e2e_train_epochs_fused.err
timeout 600 $T --nproc-per-node 4 --master-port 29801 tools/e2e_train.py --model resnet50 --train-epochs 6 --steps-per-epoch 8 --mode faithful --overlap > $O/e2e_train_epochs_overlap.jsonl 2> $O/e2e_train_epochs_overlap.err
timeout 600 $T --nproc-per-node 4 --master-port 29802 tools/e2e_train.py --model hmsa --mode fused --steps 10 --warmup 3 > $O/e2e_hmsa_2x2_fused.json 2> $O/e2e_hmsa_2x2_fused.err
ls $O | wc -l
