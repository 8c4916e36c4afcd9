#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-sch}
N=$(nvidia-smi -L | wc -l)
S=gpurun_out/summary_${TAG}.txt; echo "gpus=$N" > $S
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $S
P=29800
for sch in flowmoe flowmoe_ar flowmoe_at pipe_moe vanilla_ep; do
  for c in c2 c3; do
    P=$((P+1))
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --config $c --schedule $sch --compute-streams 1 --no-cpu-baseline > gpurun_out/abl_${c}_${sch}_${TAG}.json 2> gpurun_out/abl_${c}_${sch}_${TAG}.err
    echo "abl $c $sch rc=$?" >> $S
  done
done
cat $S; tail -n 3 gpurun_out/pytest_$TAG.log
for f in gpurun_out/abl_*_${TAG}.json; do python -c "
import json
f='$f'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]; e=d.get('exposed_comm') or {}
  print(f.split('/')[-1], round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s exposed_ms', e.get('exposed_ms'), 'comm_ms', e.get('comm_busy_ms'))
except Exception as ex: print(f, 'ERR', ex)
"; done
