#!/bin/bash
# BO tuner for S_p (Theorem 2 trade-off) at N = visible GPUs on the final code, dsv2s.
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/r02/tune_n$N; mkdir -p $O
for c in ${CONFIGS:-dsv2s}; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29931 \
    tools/tune_sp.py --config $c --out $O/tune_$c.json > $O/tune_$c.log 2>&1
  echo "tune $c rc=$?"; tail -c 1800 $O/tune_$c.json; echo
done
