#!/bin/bash
# A/B of library builds on one box: build/ab/lib_*.so vs the in-tree build; c2/c3/c4 benches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-lab}
S=gpurun_out/summary_$TAG.txt; : > $S
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_multi.py -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $S; tail -3 gpurun_out/pytest_$TAG.log >> $S
for rep in 1 2; do
for lib in build/ab/lib_*.so cur; do
  n=$(basename $lib .so)
  for c in c2 c3 c4; do
    extra=""; [ $c = c4 ] && extra="--steps 10 --warmup 3"
    if [ $lib = cur ]; then L=""; else L="FLOWMOE_LIB=$PWD/$lib"; fi
    env $L timeout 600 python bench.py --config $c $extra --no-cpu-baseline --trace-iters 0 --profile-json gpurun_out/prof_${c}_${TAG}_${n}_$rep.json > gpurun_out/bench_${c}_${TAG}_${n}_$rep.json 2> gpurun_out/bench_${c}_${TAG}_${n}_$rep.err
    echo "$n $c rep$rep rc=$?" >> $S
  done
done
done
cat $S
for f in gpurun_out/bench_*_${TAG}_*.json; do python -c "
import json
f='$f'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]
  print(f.split('/')[-1], round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s')
except Exception as ex: print(f, 'ERR', ex)
"; done
