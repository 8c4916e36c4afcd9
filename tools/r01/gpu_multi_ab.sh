#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-mab}
N=$(nvidia-smi -L | wc -l)
P=29600
run() {  # name, env, args...
  local name=$1; shift; local envs=$1; shift
  P=$((P+1))
  env $envs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@" > gpurun_out/bench_${TAG}_${name}_n$N.json 2> gpurun_out/bench_${TAG}_${name}_n$N.err
  python -c "
import json
f='gpurun_out/bench_${TAG}_${name}_n$N.json'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]; e=d.get('exposed_comm') or {}; print('$name', round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s exposed', round(e.get('exposed_ms',0),3), 'comm_busy', round(e.get('comm_busy_ms',0),3), 'frac', e.get('frac_of_comm'))
except Exception as ex: print('$name', 'ERR', ex)
"
}
for c in c2 c3; do
  run ${c}_lanesR "X=1" --config $c
  run ${c}_lanes1 "X=1" --config $c --compute-streams 1
  run ${c}_lanes2 "X=1" --config $c --compute-streams 2
  run ${c}_LL "NCCL_PROTO=LL" --config $c
  run ${c}_lanes1_LL "NCCL_PROTO=LL" --config $c --compute-streams 1
done
