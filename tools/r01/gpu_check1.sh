#!/bin/bash
# 1-GPU: full pytest -m gpu (single-GPU files), bench c2/c3/c4 with per-kernel profiles
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-k}
S=gpurun_out/summary_$TAG.txt; : > $S
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_multi.py > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $S
for c in c2 c3 c4; do
  extra=""; [ $c = c4 ] && extra="--steps 10 --warmup 3"
  timeout 900 python bench.py --config $c $extra --profile-json gpurun_out/prof_${c}_${TAG}.json > gpurun_out/bench_${c}_${TAG}.json 2> gpurun_out/bench_${c}_${TAG}.err
  echo "bench $c rc=$?" >> $S
done
cat $S; tail -n 25 gpurun_out/pytest_$TAG.log
for f in gpurun_out/bench_*_${TAG}.json; do python -c "
import json
f='$f'
try:
  d=[json.loads(l) for l in open(f) if l.startswith('{')][0]
  print(f.split('/')[-1], round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s', d['roofline']['kernel'], round(d['roofline']['frac'],3))
except Exception as ex: print(f, 'ERR', ex)
"; done
