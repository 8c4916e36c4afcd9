#!/bin/bash
# parity + A/B bench (PDL on/off) for c2, c3, c4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ab}
S=gpurun_out/summary_$TAG.txt
: > $S
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $S
for c in c2 c3 c4; do
  extra=""; [ $c = c4 ] && extra="--steps 10 --warmup 3"
  [ $c != c2 ] && extra="$extra --no-cpu-baseline"
  timeout 900 python bench.py --config $c $extra --profile-json gpurun_out/prof_${c}_$TAG.json > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "bench $c rc=$?" >> $S
  FLOWMOE_NO_PDL=1 timeout 900 python bench.py --config $c $extra --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}_nopdl.json 2>&1; echo "bench $c nopdl rc=$?" >> $S
done
cat $S; tail -n 5 gpurun_out/pytest_$TAG.log
for c in c2 c3 c4; do for f in gpurun_out/bench_${c}_$TAG.json gpurun_out/bench_${c}_${TAG}_nopdl.json; do python -c "
import json,sys
try:
  d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s', d['roofline']['kernel'], round(d['roofline']['frac'],3))
except Exception as e: print('$f', 'ERR', e)
"; done; done
