#!/bin/bash
# stack API check on a 2-GPU box: stack/chain parity tests (1 GPU + P=2), then bench
# stack vs per-block at N=1 and N=2 for c2/c3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-st}
S=gpurun_out/summary_$TAG.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_parity.py -k "stack" -q -p no:cacheprovider > gpurun_out/pytest1_$TAG.log 2>&1; echo "pytest stack rc=$?" >> $S
timeout 900 python -m pytest tests/test_gpu_multi.py -k "2" -q -p no:cacheprovider > gpurun_out/pytest2_$TAG.log 2>&1; echo "pytest multi rc=$?" >> $S
P=29800
for c in c2 c3; do
  for api in "" "--per-block"; do
    a=${api:-"--stack"}; a=${a#--}
    CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config $c $api --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}_${a}_n1.json 2> gpurun_out/bench_${c}_${TAG}_${a}_n1.err
    echo "bench $c $a n1 rc=$?" >> $S
    P=$((P+1))
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --config $c $api > gpurun_out/bench_${c}_${TAG}_${a}_n2.json 2> gpurun_out/bench_${c}_${TAG}_${a}_n2.err
    echo "bench $c $a n2 rc=$?" >> $S
  done
done
cat $S; tail -n 3 gpurun_out/pytest1_$TAG.log gpurun_out/pytest2_$TAG.log
for f in gpurun_out/bench_*_${TAG}_*.json; do python -c "
import json
f='$f'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]; e=d.get('exposed_comm') or {}
  print(f.split('/')[-1], round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s', 'e2e', round(d['e2e']['value']), 'exposed_ms', e.get('exposed_ms'))
except Exception as ex: print(f, 'ERR', ex)
"; done
