#!/bin/bash
# Table 6 analogue on the final code (N = visible GPUs): the five scheduling policies on the
# same kernels at dsv2s (R=2, the bench default) and c3 (R=4), peer-memory A2A.
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/r02/table6_n$N; mkdir -p $O
P=29870
for spec in "dsv2s:2" "c3:4"; do
  c=${spec%%:*}; R=${spec#*:}
  for sch in vanilla_ep pipe_moe flowmoe_at flowmoe_ar flowmoe; do
    P=$((P+1))
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
      bench.py --gpus $N --config $c --R $R --schedule $sch --no-cpu-baseline --trace-iters 10 --steps 30 --trace-dir /tmp \
      > $O/${c}_${sch}.json 2> $O/${c}_${sch}.err
    echo "$c $sch rc=$?"
  done
done
for f in $O/*.json; do python -c "
import json
f='$f'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]; e=d.get('exposed_comm') or {}
  print(f.split('/')[-1], round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s exposed_ms', e.get('exposed_ms'), 'frac', e.get('frac_of_comm'))
except Exception as ex: print(f, 'ERR', ex)
"; done
