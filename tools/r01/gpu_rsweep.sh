#!/bin/bash
# pipelining degree R on B200: c2/c3 at N=1 and N=4 (4-GPU box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/rsweep
O=gpurun_out/rsweep
P=29800
for c in c3 c2; do
  RS="1 2 4 8"; [ $c = c2 ] && RS="1 2 4"
  for R in $RS; do
    CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --config $c --R $R --no-cpu-baseline --trace-iters 0 --steps 50 > $O/${c}_R${R}_n1.json 2>/dev/null
    P=$((P+1))
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --config $c --R $R --no-cpu-baseline --trace-iters 10 --steps 50 > $O/${c}_R${R}_n4.json 2>/dev/null
  done
done
for f in $O/*.json; do python -c "
import json
f='$f'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]; e=d.get('exposed_comm') or {}
  print(f.split('/')[-1], round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s exposed', e.get('exposed_ms'), e.get('frac_of_comm'))
except Exception as ex: print(f, 'ERR', ex)
"; done
