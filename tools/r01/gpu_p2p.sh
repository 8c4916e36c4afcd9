#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-p}
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -x > gpurun_out/pytest_multi_$TAG.log 2>&1; echo "pytest multi rc=$?"; tail -n 15 gpurun_out/pytest_multi_$TAG.log | grep -vE "^\s*$" | tail -8
P=29950
for c in c2 c3 c4; do for a in p2p nccl; do
  extra=""; [ $c = c4 ] && extra="--steps 10 --warmup 3"
  P=$((P+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --config $c --a2a $a $extra > gpurun_out/bench_${c}_${a}_${TAG}_n$N.json 2> gpurun_out/bench_${c}_${a}_${TAG}_n$N.err
  python -c "
import json
f='gpurun_out/bench_${c}_${a}_${TAG}_n$N.json'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]; e=d.get('exposed_comm') or {}
  print('$c $a n$N', round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s exposed_ms', e.get('exposed_ms'), 'frac', e.get('frac_of_comm'))
except Exception as ex: print(f, 'ERR', ex)
"
done; done
