#!/bin/bash
# token-chunk (R > sequences) validation on a 2-GPU box + a few bench points
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-tok}
S=gpurun_out/summary_$TAG.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_parity.py -k "tok or stack" -q -p no:cacheprovider > gpurun_out/pytest1_$TAG.log 2>&1; echo "pytest tok rc=$?" >> $S
timeout 900 python -m pytest tests/test_gpu_multi.py -k "2" -q -p no:cacheprovider > gpurun_out/pytest2_$TAG.log 2>&1; echo "pytest multi rc=$?" >> $S
for R in 4 8; do
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config c2 --R $R --no-cpu-baseline > gpurun_out/bench_c2_${TAG}_R${R}.json 2> gpurun_out/bench_c2_${TAG}_R${R}.err
  echo "bench c2 R$R rc=$?" >> $S
done
for R in 2 4 8; do
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config dsv2s --R $R --steps 20 --no-cpu-baseline > gpurun_out/bench_dsv2s_${TAG}_R${R}.json 2> gpurun_out/bench_dsv2s_${TAG}_R${R}.err
  echo "bench dsv2s R$R rc=$?" >> $S
done
cat $S; tail -n 15 gpurun_out/pytest1_$TAG.log; tail -n 5 gpurun_out/pytest2_$TAG.log
for f in gpurun_out/bench_*_${TAG}_*.json; do python -c "
import json
f='$f'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]
  print(f.split('/')[-1], round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s', d['roofline']['kernel'], round(d['roofline']['frac'],3))
except Exception as ex: print(f, 'ERR', ex)
"; done
