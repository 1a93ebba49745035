cp paper_2104_05588_b200/libdaso.so /tmp/libdaso_new.so
for rep in 1 2; do
for V in new prev; do
  if [ $V = prev ]; then cp paper_2104_05588_b200/libdaso_prev.so paper_2104_05588_b200/libdaso.so; else cp /tmp/libdaso_new.so paper_2104_05588_b200/libdaso.so; fi
  timeout 120 python tools/kernel_bench.py --only K1,K2,K4,pack > gpurun_out/kb25_$V.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/kb25_$V.json')); print('$V', {k: round(v['us'],1) for k,v in d['kernels'].items()})"
done; done
cp /tmp/libdaso_new.so paper_2104_05588_b200/libdaso.so
