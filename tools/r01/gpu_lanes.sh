#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-l1}
S=gpurun_out/summary_$TAG.txt; : > $S
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $S
for c in c2 c3 c4; do
  extra=""; [ $c = c4 ] && extra="--steps 10 --warmup 3"
  [ $c != c2 ] && extra="$extra --no-cpu-baseline"
  timeout 900 python bench.py --config $c $extra --profile-json gpurun_out/prof_${c}_$TAG.json > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "bench $c rc=$?" >> $S
  timeout 900 python bench.py --config $c $extra --no-cpu-baseline --compute-streams 1 --trace-iters 0 > gpurun_out/bench_${c}_${TAG}_1s.json 2> /dev/null; echo "bench $c 1stream rc=$?" >> $S
done
cat $S; tail -n 5 gpurun_out/pytest_$TAG.log
for f in gpurun_out/bench_*_$TAG*.json; do python -c "
import json
try:
  d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s', d['roofline']['kernel'], round(d['roofline']['frac'],3), d.get('timeline',{}).get('idle_ms'))
except Exception as e: print('$f', 'ERR', e)
"; done
