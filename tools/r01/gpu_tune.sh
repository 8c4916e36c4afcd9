#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for c in c4 c3; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29911 tools/tune_sp.py --config $c --out gpurun_out/tune_${c}_n$N.json > gpurun_out/tune_${c}_n$N.log 2>&1
  echo "tune $c rc=$?"
  tail -c 1500 gpurun_out/tune_${c}_n$N.json
  echo
done
