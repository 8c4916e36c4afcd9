#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-m}
N=$(nvidia-smi -L | wc -l)
S=gpurun_out/summary_${TAG}_n$N.txt; echo "gpus=$N" > $S
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_multi_${TAG}_n$N.log 2>&1; echo "pytest multi rc=$?" >> $S
P=29500
for c in c2 c3 c4; do
  extra=""; [ $c = c4 ] && extra="--steps 10 --warmup 3"
  P=$((P+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --config $c $extra --profile-json gpurun_out/prof_${c}_${TAG}_n$N.json > gpurun_out/bench_${c}_${TAG}_n$N.json 2> gpurun_out/bench_${c}_${TAG}_n$N.err; echo "bench $c rc=$?" >> $S
done
cat $S; tail -n 3 gpurun_out/pytest_multi_${TAG}_n$N.log
for c in c2 c3 c4; do python -c "
import json
f='gpurun_out/bench_${c}_${TAG}_n$N.json'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]; print(f, round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s', d['roofline']['kernel'], round(d['roofline']['frac'],3), json.dumps(d.get('exposed_comm')))
except Exception as e: print(f, 'ERR', e)
"; done
