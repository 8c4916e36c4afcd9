#!/bin/bash
# Pipelining degree R at N = visible GPUs on the final code (dsv2s: R = 1, 2, 4 whole-sequence
# chunks; the FLOWMOE schedule).
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/r02/rsweep_n$N; mkdir -p $O
P=29910
for R in 1 2 4; do
  P=$((P+1))
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
    bench.py --gpus $N --config dsv2s --R $R --no-cpu-baseline --trace-iters 10 --steps 30 --trace-dir /tmp \
    > $O/dsv2s_R$R.json 2> $O/dsv2s_R$R.err
  echo "R=$R rc=$?"; python -c "
import json
d=[json.loads(l) for l in open('$O/dsv2s_R$R.json') if l.startswith('{')][0]; e=d.get('exposed_comm') or {}
print('dsv2s R=$R', round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s exposed/comm', e.get('frac_of_comm'))
"
done
