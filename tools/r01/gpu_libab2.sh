#!/bin/bash
# A/B of library builds at N=2 (2-GPU box): build/ab/lib_*.so vs the in-tree build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-lab2}
P=29700
[ -n "$PYTEST" ] && { timeout 900 python -m pytest tests/test_gpu_multi.py -k "2" -q -p no:cacheprovider > gpurun_out/pytest2_$TAG.log 2>&1; echo "pytest multi rc=$?"; tail -2 gpurun_out/pytest2_$TAG.log; }
for rep in 1 2; do
for lib in build/ab/lib_*.so cur ${EXTRA}; do
  n=$(basename $lib .so)
  for c in c2 c3; do
    P=$((P+1))
    if [ $lib = cur ]; then L="FLOWMOE_X=";
    elif [ $lib = cur_ikw ]; then L="FLOWMOE_P2P_INKERNEL_WAIT=1";
    else L="FLOWMOE_LIB=$PWD/$lib"; fi
    env $L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --config $c --trace-iters 0 > gpurun_out/bench_${c}_${TAG}_${n}_$rep.json 2> gpurun_out/bench_${c}_${TAG}_${n}_$rep.err
  done
done
done
for f in gpurun_out/bench_*_${TAG}_*.json; do python -c "
import json
f='$f'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]
  print(f.split('/')[-1], round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s')
except Exception as ex: print(f, 'ERR', ex)
"; done
