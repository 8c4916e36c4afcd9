#!/bin/bash
# Table 6 analogue on B200 (N=4, one 4-GPU box): the five scheduling policies on the same
# kernels, c2 (R=4) and c3 (R=4), peer-memory A2A, compute lanes = R
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/table6
O=gpurun_out/table6
P=29870
for c in c2 c3; do
  for sch in vanilla_ep pipe_moe flowmoe_at flowmoe_ar flowmoe; do
    P=$((P+1))
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --config $c --R 4 --schedule $sch --no-cpu-baseline --trace-iters 10 --steps 50 > $O/${c}_${sch}.json 2>/dev/null
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
