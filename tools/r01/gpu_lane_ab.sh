#!/bin/bash
# 2-GPU box: P=2 parity, then N=2 benches with the peer-memory A2A on the chunk lanes
# (default) vs on the A2A stream (FLOWMOE_P2P_A2A_STREAM=1), c2 and c3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-la}
S=gpurun_out/summary_$TAG.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_multi.py -k "2" -q -p no:cacheprovider > gpurun_out/pytest2_$TAG.log 2>&1; echo "pytest multi rc=$?" >> $S
P=29900
for rep in 1 2; do
for mode in lane stream; do
  for c in c2 c3; do
    P=$((P+1))
    if [ $mode = stream ]; then E="FLOWMOE_P2P_A2A_STREAM=1"; else E="FLOWMOE_P2P_A2A_STREAM="; fi
    env $E timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --config $c --trace-iters 10 > gpurun_out/bench_${c}_${TAG}_${mode}_$rep.json 2> gpurun_out/bench_${c}_${TAG}_${mode}_$rep.err
    echo "$c $mode rc=$?" >> $S
  done
done
done
cat $S; tail -2 gpurun_out/pytest2_$TAG.log
for f in gpurun_out/bench_*_${TAG}_*.json; do python -c "
import json
f='$f'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]; e=d.get('exposed_comm') or {}
  print(f.split('/')[-1], round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s exposed', e.get('exposed_ms'), e.get('frac_of_comm'))
except Exception as ex: print(f, 'ERR', ex)
"; done
